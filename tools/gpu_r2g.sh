timeout 300 python tools/sanitize_step.py > gpurun_out/r2g_plain.log 2>&1; echo plain=$?; tail -2 gpurun_out/r2g_plain.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_step.py > gpurun_out/r2g_memcheck.log 2>&1; echo memcheck=$?; tail -4 gpurun_out/r2g_memcheck.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=12 > gpurun_out/r2g_pytest.log 2>&1; echo pytest=$?; grep -E "passed|failed|FAILED" gpurun_out/r2g_pytest.log | tail -6
