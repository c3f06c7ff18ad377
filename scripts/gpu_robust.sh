# Robustness: NCCL code path at N=1 via torchrun, and the large configs.
set -x
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
  --master-port 29611 bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu-baseline --force-dist \
  > gpurun_out/bench_dist.log 2>&1; echo dist=$?
timeout 1200 python scripts/run_configs.py > gpurun_out/configs.log 2>&1; echo configs=$?
tail -c 600 gpurun_out/bench_dist.log; cat gpurun_out/configs.log | tail -20
