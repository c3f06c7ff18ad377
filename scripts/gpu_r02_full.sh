# Round-2 evidence pass: GPU tests, smoke, bench + reference arm, launch list, raster ncu.
TAG=${1:-r02}
nvidia-smi -L > gpurun_out/smi_$TAG.txt
lscpu | head -20 > gpurun_out/cpu_$TAG.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest=$?
tail -n 2 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke=$?
timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.log 2> gpurun_out/bench_$TAG.err; echo bench=$?
timeout 1200 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.log 2>&1; echo ref=$?
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_bench_$TAG.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches_bench_$TAG.csv $CMD > gpurun_out/ncu_bench_$TAG.log 2>&1
echo launches=$?
tail -c 1500 gpurun_out/bench_$TAG.log; tail -c 600 gpurun_out/bench_ref_$TAG.log
