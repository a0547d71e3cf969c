timeout 1200 python -m pytest tests/test_radiation.py tests/test_gpu_radiation.py tests/test_gpu_cppn.py tests/test_snapshot.py tests/test_state_api.py -m gpu -q -p no:cacheprovider > gpurun_out/r2c_pytest.log 2>&1; echo pytest=$?; tail -5 gpurun_out/r2c_pytest.log
timeout 300 python tools/rad_time.py > gpurun_out/r2c_rad.log 2>&1; echo rad=$?; head -4 gpurun_out/r2c_rad.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2c_bench_c3.log 2>&1; echo bench=$?; tail -1 gpurun_out/r2c_bench_c3.log | cut -c1-400
