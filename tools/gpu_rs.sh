set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "radiation or strips or select" > gpurun_out/rs_pytest.log 2>&1; echo pytest=$?
tail -25 gpurun_out/rs_pytest.log | grep -E "passed|failed|Error|assert|error" | head
