timeout 900 python scripts/time_score.py --config 4 --views 8 --repeat 1 --dump gpurun_out/r02g_cfg4_new.npz 2>&1 | head -2
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r02g_pytest.log 2>&1; echo pytest=$?
tail -n 3 gpurun_out/r02g_pytest.log
for c in 1 3 4; do n=64; [ $c = 4 ] && n=32; [ $c = 3 ] && n=32; timeout 600 python scripts/time_score.py --config $c --views $n --repeat 3 2>&1 | head -1; done
