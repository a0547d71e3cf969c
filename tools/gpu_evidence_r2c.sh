# round-2c evidence: headline bench (config 3: TMA texture + gather net), config 2, config 4, config 5 slice
# (hidden net, both layers on tcgen05); launch lists; full ncu of the config-3 pass-1 kernels
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2c_bench_c3.log 2>&1; echo bench=$?
tail -1 gpurun_out/r2c_bench_c3.log | cut -c1-300
timeout 900 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r2c_bench_c3_50.log 2>&1; echo bench50=$?
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2c_bench_c2.log 2>&1; echo c2=$?
timeout 1500 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2c_bench_c4.log 2>&1; echo c4=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/r2c_launches_bench_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2c_ncu_bench.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gs_count_tma|k_gs_scatter|k_direct_gather|k_physics_rows|k_resolve" -s 8 -c 5 -o gpurun_out/r2c_c3 python tools/profile_step.py --config c3 --steps 3 > gpurun_out/r2c_ncu_c3.log 2>&1; echo ncufull=$?
