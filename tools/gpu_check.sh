# quick regression pass: GPU suite, smoke, headline bench, radiation event timing
set -x
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/chk_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/chk_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/chk_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/chk_bench_c3.log 2>&1; echo bench=$?
tail -1 gpurun_out/chk_bench_c3.log | cut -c1-400
timeout 600 python tools/rad_time.py > gpurun_out/chk_rad.log 2>&1; echo rad=$?
head -4 gpurun_out/chk_rad.log
