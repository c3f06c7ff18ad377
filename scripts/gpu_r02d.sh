timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r02d_pytest.log 2>&1; echo pytest=$?
tail -n 15 gpurun_out/r02d_pytest.log
for c in 1 3 4; do n=64; [ $c = 4 ] && n=32; [ $c = 3 ] && n=32; timeout 600 python scripts/time_score.py --config $c --views $n --repeat 3; done > gpurun_out/r02d_time.log 2>&1
cat gpurun_out/r02d_time.log
timeout 600 python scripts/split_time.py --config 1 > gpurun_out/r02d_split.log 2>&1; tail -5 gpurun_out/r02d_split.log
