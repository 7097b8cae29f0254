#!/bin/bash
# ncu --set full of the three longest k_tile_jit passes of the bench circuit
# (30 qubits, depth 20, seed 12345). Run on the GPU box from the repo root:
#   bash tools/prof_heavy.sh OUTDIR
set -e
OUT=${1:-gpurun_out/heavy}
mkdir -p "$OUT"
export QGPU_JIT=sync
python tools/heavy_passes.py --steps 2 --out "$OUT/passes.json" > "$OUT/passes.txt"
# the three longest passes and the median one
IDX=$(python -c "import json,sys; r=json.load(open('$OUT/passes.json'))['rows']; print(' '.join(str(x['pass']) for x in r[:3] + [r[len(r) // 2]]))")
echo "top passes: $IDX" >> "$OUT/passes.txt"
for i in $IDX; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tile_jit \
    --launch-skip "$i" --launch-count 1 -f -o "$OUT/pass_$i" \
    python tools/heavy_passes.py --steps 1 > "$OUT/ncu_$i.log" 2>&1 || echo "ncu $i failed" >> "$OUT/passes.txt"
done
