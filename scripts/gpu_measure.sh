# Full measurement pass: bench (with the reference CPU baseline), reference arm,
# ncu launch list of the bench command, one full ncu capture of the raster kernel.
# usage: bash scripts/gpu_measure.sh <tag>
set -x
TAG=${1:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_$TAG.txt
lscpu | head -20 > gpurun_out/cpu_$TAG.txt
timeout 1800 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.log 2> gpurun_out/bench_$TAG.err; echo bench=$?
timeout 1200 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_$TAG.log 2>&1; echo ref=$?
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_bench_$TAG.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches_bench_$TAG.csv $CMD > gpurun_out/ncu_bench_$TAG.log 2>&1
echo launches=$?
PCMD="python scripts/profile_raster.py --config 1 --views 8"
$PCMD > gpurun_out/plain_prof_$TAG.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_raster -c 1 \
  -o gpurun_out/raster_full_$TAG $PCMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo full=$?
tail -n 2 gpurun_out/bench_$TAG.log gpurun_out/bench_ref_$TAG.log
