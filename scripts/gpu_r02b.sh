timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r02b_pytest.log 2>&1; echo pytest=$?
tail -n 40 gpurun_out/r02b_pytest.log
