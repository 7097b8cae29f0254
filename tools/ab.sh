# A/B of the default build against a variant on the same box (JIT on in both;
# the variant's JIT gets VAROPTS): VAR=x VAROPTS="-DFOO=1" bash tools/ab.sh
one() { timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_gate'], d['roofline']['avg_launch_ms'], d['config']['passes_per_step'], d['check']['norm_error_after_timed_steps'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for r in 1 2; do
echo "base"; one
echo "$VAR"; QGPU_LIB=paper_1802_08032_b200/_lib/libqgpu_$VAR.so QGPU_JIT_OPTS="$VAROPTS" one
done
