# Round measurement bundle (run under gpurun): bench line, reference arm,
# ncu launch list + one --set full capture of a mid-circuit tile pass.
set -x
mkdir -p gpurun_out
TAG=${TAG:-cur}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo ref=$?
TAG=$TAG bash tools/gpu_prof.sh
