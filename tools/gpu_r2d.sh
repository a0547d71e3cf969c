timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/r2d_pytest.log 2>&1; echo pytest=$?; grep -E "passed|failed|FAILED" gpurun_out/r2d_pytest.log | tail -8
