# Round-2 evidence pass: tests, smoke, bench + reference arm, launch list of the bench command,
# one ncu --set full raster capture (+ summary), every BASELINE config.
# usage: bash scripts/gpu_r02_evidence.sh <tag>
TAG=${1:-r02}
bash scripts/gpu_r02_full.sh $TAG
# the 4th raster launch of a 15-view call: sub-batches 1, 2, 4, 8 -> the 8-view launch (views 7-14)
PCMD="python scripts/profile_raster.py --config 1 --views 15"
$PCMD > gpurun_out/plain_prof_$TAG.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_raster -s 3 -c 1 \
  -o gpurun_out/raster_full_$TAG $PCMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo full=$?
python scripts/ncu_summary.py gpurun_out/raster_full_$TAG.ncu-rep gpurun_out/raster_summary_$TAG.json 8 > /dev/null 2>&1; echo summary=$?
ncu -i gpurun_out/raster_full_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/raster_sass_$TAG.csv 2>/dev/null
ncu -i gpurun_out/raster_full_$TAG.ncu-rep --page details > gpurun_out/raster_details_$TAG.txt 2>/dev/null
timeout 1500 python scripts/config_table.py --cfgs 1,2,3,4 --out gpurun_out/config_table_$TAG.json > gpurun_out/config_table_$TAG.log 2>&1; echo table=$?
tail -n 8 gpurun_out/config_table_$TAG.log
