# ncu --set full of one 8-view k_raster<score> launch of config CFG (4th launch of a 15-view
# call): bash scripts/gpu_ncu_cfg.sh <cfg> <tag>
CFG=${1:-4}; TAG=${2:-cfg$CFG}
PCMD="python scripts/profile_raster.py --config $CFG --views 15"
$PCMD > gpurun_out/plain_prof_$TAG.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_raster -s 3 -c 1 \
  -o gpurun_out/raster_full_$TAG $PCMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo full=$?
python scripts/ncu_summary.py gpurun_out/raster_full_$TAG.ncu-rep gpurun_out/raster_summary_$TAG.json 8 > /dev/null 2>&1; echo summary=$?
ncu -i gpurun_out/raster_full_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/raster_sass_$TAG.csv 2>/dev/null
ncu -i gpurun_out/raster_full_$TAG.ncu-rep --page details > gpurun_out/raster_details_$TAG.txt 2>/dev/null
grep -m3 "k_raster\|Duration" gpurun_out/raster_details_$TAG.txt
