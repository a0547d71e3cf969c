set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "strips or tma_texture" > gpurun_out/st_pytest.log 2>&1; echo pytest=$?
tail -15 gpurun_out/st_pytest.log
