# Round-end evidence pass: GPU tests, smoke, bench + reference arm + launch list + raster
# ncu capture (gpu_measure.sh), every BASELINE config (config_table.py).
# usage: bash scripts/gpu_final.sh <tag>
TAG=${1:-r01}
nvidia-smi -L > gpurun_out/smi_$TAG.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest=$?
tail -n 1 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke=$?
bash scripts/gpu_measure.sh $TAG
timeout 1500 python scripts/config_table.py --cfgs 1,2,3,4 --out gpurun_out/config_table_$TAG.json > gpurun_out/config_table_$TAG.log 2>&1; echo table=$?
