timeout 600 python -m pytest tests/test_gpu_dist.py tests/test_dropin.py -m gpu -q -x > gpurun_out/r02c_dist.log 2>&1; echo dist=$?
tail -n 30 gpurun_out/r02c_dist.log
SGM_DEVICES=0,0 timeout 600 python -m pytest tests/test_dropin.py -q -x > gpurun_out/r02c_dropin2.log 2>&1; echo dropin2=$?
tail -n 5 gpurun_out/r02c_dropin2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --force-dist --no-cpu-baseline > gpurun_out/r02c_benchdist.log 2> gpurun_out/r02c_benchdist.err; echo benchdist=$?
tail -c 1500 gpurun_out/r02c_benchdist.log; tail -n 20 gpurun_out/r02c_benchdist.err
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r02c_pytest.log 2>&1; echo pytest=$?
tail -n 5 gpurun_out/r02c_pytest.log
