# usage: bash scripts/gpu_ncu.sh <tag> [profile_raster args]
set -x
TAG=$1; shift
CMD="python scripts/profile_raster.py $*"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
echo launches=$?
$CMD > gpurun_out/plain2_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_raster -c 1 -o gpurun_out/raster_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo full=$?
tail -n 3 gpurun_out/plain_$TAG.log gpurun_out/ncu_full_$TAG.log
