#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck of the tile pass on the
# GPU box: JIT kernels (sync compiles) and the interpreter, circuit order and
# the default ordering. bash tools/sanitize_all.sh OUTDIR [QUBITS]
OUT=${1:-gpurun_out/sanitize}; Q=${2:-16}
mkdir -p "$OUT"
for tool in racecheck synccheck memcheck; do
  for mode in sync off; do
    for order in "" "--reorder"; do
      tag="${tool}_${mode}${order:+_reorder}"
      QGPU_JIT=$mode timeout 900 compute-sanitizer --tool $tool --print-limit 20 \
        python tools/sanitize_run.py --qubits $Q $order > "$OUT/$tag.txt" 2>&1
      echo "$tag rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' "$OUT/$tag.txt" | tail -1)"
    done
  done
done
