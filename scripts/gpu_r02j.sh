for lib in libsgm_b200_r01 libsgm_b200; do
SGM_B200_LIB=paper_2506_00225_b200/_lib/$lib.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02j_render_$lib.csv python scripts/profile_render.py --config 1 --repeat 3 > /dev/null 2>&1; echo ncu=$?
done
