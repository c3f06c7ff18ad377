python scripts/profile_raster.py --config 1 --views 8 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02i_new.csv python scripts/profile_raster.py --config 1 --views 8 --repeat 2 > /dev/null 2>&1; echo ncu=$?
SGM_B200_LIB=paper_2506_00225_b200/_lib/libsgm_b200_prev.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02i_prev.csv python scripts/profile_raster.py --config 1 --views 8 --repeat 2 > /dev/null 2>&1; echo ncu=$?
