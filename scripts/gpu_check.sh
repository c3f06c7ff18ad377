# usage: bash scripts/gpu_check.sh [bench args...]
set -x
nvidia-smi -L
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/bench.log 2>&1; echo bench=$?
tail -n 3 gpurun_out/smoke.log gpurun_out/pytest_gpu.log gpurun_out/bench.log
