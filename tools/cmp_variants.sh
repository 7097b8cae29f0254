# Compare library variants on the bench (under gpurun): VARIANTS="rb4 x" bash tools/cmp_variants.sh
for v in base $VARIANTS; do
  if [ $v = base ]; then L=paper_1802_08032_b200/_lib/libqgpu.so; else L=paper_1802_08032_b200/_lib/libqgpu_$v.so; fi
  echo "== $v"
  QGPU_LIB=$L timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_gate'], d['roofline']['avg_launch_ms'], d['config']['passes_per_step'])"
  if [ -n "$PARITY" ]; then QGPU_LIB=$L timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2; fi
done
