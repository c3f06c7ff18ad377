# usage: bash scripts/gpu_ncu_k.sh <tag> <kernel-regex> [profile_raster args]
set -x
TAG=$1; KRE=$2; shift; shift
CMD="python scripts/profile_raster.py $*"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$KRE -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo full=$?
tail -n 3 gpurun_out/plain_$TAG.log gpurun_out/ncu_$TAG.log
