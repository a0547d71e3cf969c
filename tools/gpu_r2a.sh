set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; free -g | head -2; nproc
python -c "import paper_2406_09654_b200 as p; from paper_2406_09654_b200 import _lib; _lib.load(); print('lib ok')"
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/r2a_pytest.log 2>&1; echo pytest=$?; tail -25 gpurun_out/r2a_pytest.log
timeout 300 python tools/rad_time.py > gpurun_out/r2a_rad.log 2>&1; echo rad=$?; tail -40 gpurun_out/r2a_rad.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2a_bench_c3.log 2>&1; echo bench=$?; tail -2 gpurun_out/r2a_bench_c3.log
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2a_bench_c2.log 2>&1; echo bench2=$?; tail -1 gpurun_out/r2a_bench_c2.log
