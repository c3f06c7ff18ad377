# ncu --set full of one launch of kernel KREGEX in a CFG scoring call: bash scripts/gpu_ncu_kernel.sh <cfg> <kregex> <tag> [skip]
CFG=$1; K=$2; TAG=$3; SKIP=${4:-0}
PCMD="python scripts/profile_raster.py --config $CFG --views ${VIEWS:-2}"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 \
  -o gpurun_out/k_$TAG $PCMD > gpurun_out/ncu_k_$TAG.log 2>&1
echo full=$?
python scripts/ncu_summary.py gpurun_out/k_$TAG.ncu-rep gpurun_out/k_summary_$TAG.json 1 > /dev/null 2>&1; echo summary=$?
ncu -i gpurun_out/k_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/k_sass_$TAG.csv 2>/dev/null
ncu -i gpurun_out/k_$TAG.ncu-rep --page details > gpurun_out/k_details_$TAG.txt 2>/dev/null
grep -m3 "Duration" gpurun_out/k_details_$TAG.txt
