python scripts/profile_raster.py --config 4 --views 4 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02h_launch_cfg4.csv python scripts/profile_raster.py --config 4 --views 4 --repeat 2 > /dev/null 2>&1; echo ncu=$?
