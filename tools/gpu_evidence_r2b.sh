# round-2b evidence: headline bench (config 3, gather path), reference arm, config 2, config-4 anchor,
# launch lists of the bench commands (traffic), sanitizer attempt on small worlds
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2b_bench_c3.log 2>&1; echo bench=$?
tail -1 gpurun_out/r2b_bench_c3.log | cut -c1-400
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2b_bench_ref.log 2>&1; echo ref=$?
tail -1 gpurun_out/r2b_bench_ref.log | cut -c1-300
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 > gpurun_out/r2b_bench_c2.log 2>&1; echo c2=$?
timeout 1500 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_bench_c4.log 2>&1; echo c4=$?
tail -1 gpurun_out/r2b_bench_c4.log | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/r2b_launches_bench_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_ncu_bench.log 2>&1; echo launches=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/r2b_launches_bench_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_ncu_bench2.log 2>&1; echo launches2=$?
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_step.py > gpurun_out/r2b_memcheck.log 2>&1; echo memcheck=$?
tail -5 gpurun_out/r2b_memcheck.log
