#!/bin/bash
# A/B of environment knobs on the bench circuit, same box, round robin:
#   REPS=2 bash tools/ab_env.sh OUTDIR "A=1" "A=0" ["A=2" ...]
# Each variant runs bench.py (no side measurements) REPS times; the JSON
# lines land in OUTDIR/<variant>_<rep>.json, one summary line per run.
OUT=$1; shift
mkdir -p "$OUT"
for r in $(seq 1 "${REPS:-2}"); do
  for v in "$@"; do
    tag=$(echo "$v" | tr ' =/' '_-_' | tail -c 48)
    env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-c5 --no-single --no-exact-side \
      > "$OUT/${tag}_$r.json" 2> "$OUT/${tag}_$r.err"
    python -c "import json,sys; d=json.load(open('$OUT/${tag}_$r.json')); print('$v', d['ms_per_step'], d['config']['passes_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
  done
done
