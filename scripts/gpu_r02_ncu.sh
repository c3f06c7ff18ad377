# ncu --set full of one 8-view k_raster<score> launch (the 4th launch of a 15-view call: the
# sub-batches are 1, 2, 4, 8 views), its summary and source page.
TAG=${1:-r02}
PCMD="python scripts/profile_raster.py --config 1 --views 15"
$PCMD > gpurun_out/plain_prof_$TAG.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_raster -s 3 -c 1 \
  -o gpurun_out/raster_full_$TAG $PCMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo full=$?
python scripts/ncu_summary.py gpurun_out/raster_full_$TAG.ncu-rep gpurun_out/raster_summary_$TAG.json 8 > /dev/null 2>&1; echo summary=$?
ncu -i gpurun_out/raster_full_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/raster_sass_$TAG.csv 2>/dev/null
ncu -i gpurun_out/raster_full_$TAG.ncu-rep --page details > gpurun_out/raster_details_$TAG.txt 2>/dev/null
grep -m3 "k_raster\|Duration" gpurun_out/raster_details_$TAG.txt
