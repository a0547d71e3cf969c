# round-2 evidence: headline bench (config 3), reference arm, config 2, config-4 anchor,
# launch list of the headline command, full ncu captures of the top pass-1 kernels
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_c3.log 2>&1; echo bench=$?
tail -1 gpurun_out/r2_bench_c3.log | cut -c1-300
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_bench_ref.log 2>&1; echo ref=$?
tail -1 gpurun_out/r2_bench_ref.log | cut -c1-300
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 > gpurun_out/r2_bench_c2.log 2>&1; echo c2=$?
timeout 1200 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_c4.log 2>&1; echo c4=$?
tail -1 gpurun_out/r2_bench_c4.log | cut -c1-300
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/r2_launches_bench_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_ncu_bench.log 2>&1; echo launches=$?
timeout 300 python tools/profile_step.py --config c3 --steps 3 > gpurun_out/r2_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_hid_sense|k_direct_rows|k_physics_rows|k_resolve" -s 4 -c 4 -o gpurun_out/r2_c3 python tools/profile_step.py --config c3 --steps 3 > gpurun_out/r2_ncu_c3.log 2>&1; echo ncufull=$?
