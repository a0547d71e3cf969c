set -x
timeout 900 python bench.py --strips --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/s3_bench_strips50.log 2>&1; tail -1 gpurun_out/s3_bench_strips50.log | cut -c1-220
timeout 900 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/s3_bench_c3_50.log 2>&1; tail -1 gpurun_out/s3_bench_c3_50.log | cut -c1-220
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/s3_launches_strips.csv python bench.py --strips --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s3_ncu.log 2>&1; echo launches=$?
