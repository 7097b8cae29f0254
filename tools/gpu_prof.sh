# ncu captures of the hot kernel (run under gpurun): launch list + one --set full
set -x
mkdir -p gpurun_out
TAG=${TAG:-cur}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline $BENCH_ARGS > gpurun_out/launch_bench_$TAG.log 2>&1; echo launches=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tile -s 75 -c 1 \
  -o gpurun_out/tile_$TAG python bench.py --steps 1 --warmup 1 --no-cpu-baseline $BENCH_ARGS > gpurun_out/full_$TAG.log 2>&1; echo full=$?
tail -5 gpurun_out/full_$TAG.log
