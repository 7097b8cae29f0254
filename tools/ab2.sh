one() { timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_gate'], d['roofline']['avg_launch_ms'], d['config']['passes_per_step'], d['check'], d['clocks']['sm_mhz'])"; }
echo "base jit"; one
for ph in 2 3; do echo "rb4 jit phases=$ph"; QGPU_TILE_PHASES=$ph QGPU_LIB=paper_1802_08032_b200/_lib/libqgpu_rb4.so one; done
QGPU_LIB=paper_1802_08032_b200/_lib/libqgpu_rb4.so timeout 300 python tools/sweep.py --kinds RY,RZ --counts 16,32 --targets 5,6,7
QGPU_LIB=paper_1802_08032_b200/_lib/libqgpu_rb4.so timeout 300 python tools/jit_check.py 16,20 3
