for lib in libsgm_b200_r01 libsgm_b200_prev libsgm_b200; do for c in 0 1; do
SGM_B200_LIB=paper_2506_00225_b200/_lib/$lib.so timeout 300 python scripts/time_render_device.py --config $c 2>&1 | head -1 | sed "s/^/$lib /"; done; done
