# A/B of two builds of the library on the same box: bash scripts/gpu_ab.sh <cfgs>
for c in ${@:-1 3}; do n=64; [ $c = 4 ] && n=32; [ $c = 3 ] && n=32
for i in 1 2; do
SGM_B200_LIB=paper_2506_00225_b200/_lib/libsgm_b200_prev.so timeout 600 python scripts/time_score.py --config $c --views $n --repeat 5 2>&1 | head -1 | sed 's/^/prev /'
timeout 600 python scripts/time_score.py --config $c --views $n --repeat 5 2>&1 | head -1 | sed 's/^/new  /'
done; done
