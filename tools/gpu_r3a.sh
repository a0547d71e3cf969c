# spatial decided records: parity subset + config-3 bench
set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "genome_sorted or config3 or config4 or radiation or step_host or strips or cluster" > gpurun_out/r3a_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r3a_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r3a_bench_c3.log 2>&1; echo bench=$?
tail -1 gpurun_out/r3a_bench_c3.log | cut -c1-400
timeout 300 python tools/profile_step.py --config c3 --steps 3 > gpurun_out/r3a_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/r3a_launches_c3.csv python tools/profile_step.py --config c3 --steps 3 > gpurun_out/r3a_ncu.log 2>&1; echo launches=$?
