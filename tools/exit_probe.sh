# Exit-time crash bisection (run under gpurun).
gcc -shared -fPIC -o /tmp/segv.so tools/segv_trace.c -ldl
PRODUCT="from paper_1802_08032_b200 import quest, circuits as C
e = quest.Env(); q = quest.QuregHandle(e, 14); C.apply_circuit(q, C.layered_random_circuit(14, 3, 1)); print(q.calcTotalProb()); q.destroy(); e.destroy()"
ORC="import oracle; from paper_1802_08032_b200 import circuits as C; from tests.harness import to_oracle_ops
print(oracle.orc_run(14, to_oracle_ops(C.layered_random_circuit(14, 3, 1)))[:1])"
for v in plain fh preload fh_preload; do
  n=0
  for i in 1 2 3 4 5 6; do
    case $v in
      plain) timeout 120 python -c "$PRODUCT
$ORC" > /tmp/p.log 2>&1;;
      fh) PYTHONFAULTHANDLER=1 timeout 120 python -X faulthandler -c "$PRODUCT
$ORC" > /tmp/p.log 2>&1;;
      preload) LD_PRELOAD=/tmp/segv.so timeout 120 python -c "$PRODUCT
$ORC" > /tmp/p.log 2>&1;;
      fh_preload) LD_PRELOAD=/tmp/segv.so PYTHONFAULTHANDLER=1 timeout 120 python -X faulthandler -c "$PRODUCT
$ORC" > /tmp/p.log 2>&1;;
    esac
    rc=$?; [ $rc -ne 0 ] && { n=$((n+1)); cp /tmp/p.log /tmp/fail_$v.log; }
  done
  echo "$v: $n/6 failed"
  [ -f /tmp/fail_$v.log ] && grep -v "^$" /tmp/fail_$v.log | tail -30
done
