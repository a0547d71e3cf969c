# full GPU suite + smoke + headline bench with the gather path as default
set -x
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/g5_pytest.log 2>&1; echo pytest=$?
tail -5 gpurun_out/g5_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g5_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/g5_bench_c3.log 2>&1; echo bench=$?
tail -1 gpurun_out/g5_bench_c3.log | cut -c1-1500
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g5_bench_c2.log 2>&1; echo c2=$?
tail -1 gpurun_out/g5_bench_c2.log | cut -c1-300
