set -x
nvidia-smi -L
timeout 900 python -m pytest tests/test_gpu_config_scale.py -m gpu -q -x > gpurun_out/r02a_cfgscale.log 2>&1; echo cfgscale=$?
tail -n 30 gpurun_out/r02a_cfgscale.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02a_pytest.log 2>&1; echo pytest=$?
tail -n 3 gpurun_out/r02a_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02a_bench.log 2> gpurun_out/r02a_bench.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02a_ref.log 2>&1; echo ref=$?
tail -c 3000 gpurun_out/r02a_bench.log
