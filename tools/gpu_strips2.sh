set -x
timeout 900 python -m pytest tests/test_gpu_strips.py tests/test_gpu_radiation.py -x -q > gpurun_out/s_pytest.log 2>&1; echo pytest=$?
tail -8 gpurun_out/s_pytest.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or genome_sorted or tma_texture" > gpurun_out/s_pytest2.log 2>&1; echo pytest2=$?
tail -3 gpurun_out/s_pytest2.log
timeout 900 python bench.py --strips --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s_bench_strips.log 2>&1; echo strips=$?
tail -1 gpurun_out/s_bench_strips.log | cut -c1-250
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s_bench_c3.log 2>&1; echo bench=$?
tail -1 gpurun_out/s_bench_c3.log | cut -c1-250
