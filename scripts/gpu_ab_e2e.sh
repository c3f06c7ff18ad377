# A/B of the e2e step (upload + score) for two builds: bash scripts/gpu_ab_e2e.sh
for i in 1 2; do
SGM_B200_LIB=paper_2506_00225_b200/_lib/libsgm_b200_prev.so timeout 600 python scripts/time_e2e.py 2>&1 | tail -2 | sed 's/^/prev /'
timeout 600 python scripts/time_e2e.py 2>&1 | tail -2 | sed 's/^/new  /'
done
