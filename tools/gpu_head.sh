# state check at the session head: full GPU suite, smoke, headline bench, launch list
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/h_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/h_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/h_bench_c3.log 2>&1; echo bench=$?
tail -1 gpurun_out/h_bench_c3.log | cut -c1-600
timeout 300 python tools/profile_step.py --config c3 --steps 3 > gpurun_out/h_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/h_launches_c3.csv python tools/profile_step.py --config c3 --steps 3 > gpurun_out/h_ncu.log 2>&1; echo launches=$?
