# A/B of the default build against a variant (both interpreter and JIT):
#   VAR=lanecp VAROPTS="-DQGPU_LANE_COPIES=1" bash tools/ab.sh
one() { timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_gate'], d['roofline']['avg_launch_ms'], d['config']['passes_per_step'], d['check'], d['clocks']['sm_mhz'])"; }
echo "base jit";   one
echo "base interp"; QGPU_JIT=off one
echo "$VAR jit";   QGPU_LIB=paper_1802_08032_b200/_lib/libqgpu_$VAR.so QGPU_JIT_OPTS="$VAROPTS" one
echo "$VAR interp"; QGPU_LIB=paper_1802_08032_b200/_lib/libqgpu_$VAR.so QGPU_JIT=off one
