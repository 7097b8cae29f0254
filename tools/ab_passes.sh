#!/bin/bash
# A/B of tile-pass code-generation variants on the bench circuit (30 qubits):
# per-step pass time for each variant (tools/heavy_passes.py, JIT sync).
#   bash tools/ab_passes.sh OUTDIR "NAME1:ENV1" "NAME2:ENV2" ...
OUT=$1; shift
mkdir -p "$OUT"
for v in "$@"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs QGPU_JIT=sync python tools/heavy_passes.py --steps 3 --out "$OUT/$name.json" > "$OUT/$name.txt" 2>&1
  echo "$name [$envs]: $(head -1 "$OUT/$name.txt")"
done
