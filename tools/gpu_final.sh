# final check at the head: full GPU suite, smoke, headline bench
set -x
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/fin_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/fin_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/fin_bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/fin_bench.log | cut -c1-300
timeout 900 python bench.py --impl reference > gpurun_out/fin_bench_ref.log 2>&1; echo ref=$?
tail -1 gpurun_out/fin_bench_ref.log | cut -c1-200
