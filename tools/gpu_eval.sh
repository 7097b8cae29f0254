#!/bin/bash
# Quick GPU evaluation of one or more libqgpu builds (run under gpurun):
#   tools/gpu_eval.sh [lib.so ...]   (default: the in-tree build)
# For each: the GPU parity tests, the bench's 30-qubit pass time, per-op costs.
libs=("$@"); [ ${#libs[@]} -eq 0 ] && libs=(paper_1802_08032_b200/_lib/libqgpu.so)
for lib in "${libs[@]}"; do
  echo "=== $lib"
  export QGPU_LIB=$PWD/$lib
  timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
  timeout 300 python bench.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/gate', d['ms_per_gate'], 'pass ms', d['roofline']['avg_launch_ms'], 'GB/s', d['value'], 'frac', d['roofline']['frac'])"
  [ -n "$OPCOSTS" ] && timeout 400 python tools/op_costs.py 2>&1 | tail -12
done
