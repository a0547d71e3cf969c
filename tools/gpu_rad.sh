set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "radiation" > gpurun_out/rad_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/rad_pytest.log
timeout 600 python tools/rad_time.py > gpurun_out/rad_time.log 2>&1; echo rad=$?
tail -4 gpurun_out/rad_time.log
