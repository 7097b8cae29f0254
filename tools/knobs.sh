for cfg in ${CFGS:-"7 8" "7 2" "7 3" "7 1"}; do set -- $cfg
 echo "targets=$1 phases=$2"; QGPU_TILE_TARGETS=$1 QGPU_TILE_PHASES=$2 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_gate'], d['roofline']['avg_launch_ms'], d['config']['passes_per_step'], d['clocks'])"
done
