timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config_scale.py tests/test_gpu_aniso.py -m gpu -q -x > gpurun_out/r02f_pytest.log 2>&1; echo pytest=$?
tail -n 3 gpurun_out/r02f_pytest.log
python scripts/profile_raster.py --config 1 --views 8 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_launch_cfg1.csv python scripts/profile_raster.py --config 1 --views 8 --repeat 2 > /dev/null 2>&1; echo ncu=$?
for c in 1 3 4; do n=64; [ $c = 4 ] && n=32; [ $c = 3 ] && n=32; timeout 600 python scripts/time_score.py --config $c --views $n --repeat 3 2>&1 | head -1; done
