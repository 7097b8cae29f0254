#!/bin/bash
# ncu --set full of chosen k_tile_jit passes of the bench circuit's step
# (30 qubits, depth 20, seed 12345; the k-th k_tile_jit launch of a
# QGPU_JIT=sync process is pass k of step 0). Run on the GPU box:
#   bash tools/prof_passes.sh OUTDIR PASS [PASS ...]
set -e
OUT=$1; shift
mkdir -p "$OUT"
export QGPU_JIT=sync
for i in "$@"; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tile_jit \
    --launch-skip "$i" --launch-count 1 -f -o "$OUT/pass_$i" \
    python tools/heavy_passes.py --steps 1 > "$OUT/ncu_$i.log" 2>&1 || echo "ncu $i failed" >> "$OUT/failed.txt"
done
