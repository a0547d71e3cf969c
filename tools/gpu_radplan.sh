set -x
timeout 900 python -m pytest tests -m gpu -q -x -k "radiation or strips" > gpurun_out/rp_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/rp_pytest.log
timeout 600 python tools/rad_time.py > gpurun_out/rp_rad.log 2>&1; echo rad=$?
head -4 gpurun_out/rp_rad.log
for i in 1 2; do timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/rp_bench_c3_$i.log 2>&1; echo bench=$?; tail -1 gpurun_out/rp_bench_c3_$i.log | cut -c1-220; done
timeout 900 python bench.py --strips --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/rp_bench_strips.log 2>&1; echo strips=$?
tail -1 gpurun_out/rp_bench_strips.log | cut -c1-220
