# k_direct_rows: cross-half-tile prefetch + STG.256 records
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "genome_sorted or config3 or config4 or radiation" > gpurun_out/r3b_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/r3b_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r3b_bench_c3.log 2>&1; echo bench=$?
timeout 300 python tools/profile_step.py --config c3 --steps 3 > gpurun_out/r3b_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/r3b_launches_c3.csv python tools/profile_step.py --config c3 --steps 3 > gpurun_out/r3b_ncu.log 2>&1; echo launches=$?
