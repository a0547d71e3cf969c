set -x
timeout 900 python -m pytest tests/test_gpu_radiation.py tests/test_radiation.py tests/test_state_api.py tests/test_snapshot.py -x -q > gpurun_out/rad2_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/rad2_pytest.log
timeout 600 python tools/rad_time.py > gpurun_out/rad2_time.log 2>&1; grep "radiation event" gpurun_out/rad2_time.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/rad2_bench_c3.log 2>&1; echo bench=$?
tail -1 gpurun_out/rad2_bench_c3.log | cut -c1-250
