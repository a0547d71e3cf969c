# round-2e evidence (fused + lazy gather step): full GPU suite + smoke, headline bench (default c3), reference arm,
# strips bench on one GPU, config 2 / 4 lines, config-5 slice timing, launch lists of the bench commands,
# ncu --set full of the config-3 step kernels
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2e_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/r2e_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2e_bench_c3.log 2>&1; echo bench=$?
tail -1 gpurun_out/r2e_bench_c3.log | cut -c1-300
timeout 900 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r2e_bench_c3_50.log 2>&1; echo bench50=$?
tail -1 gpurun_out/r2e_bench_c3_50.log | cut -c1-300
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2e_bench_ref.log 2>&1; echo ref=$?
timeout 900 python bench.py --strips --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2e_bench_strips.log 2>&1; echo strips=$?
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2e_bench_c2.log 2>&1; echo c2=$?
timeout 1500 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2e_bench_c4.log 2>&1; echo c4=$?
tail -1 gpurun_out/r2e_bench_c4.log | cut -c1-300
timeout 300 python tools/profile_step.py --config c5 --width 4096 --height 4096 --steps 6 --flush --time > gpurun_out/r2e_c5.log 2>&1; echo c5=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/r2e_launches_bench_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2e_ncu_bench.log 2>&1; echo launches=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/r2e_launches_c3.csv python tools/profile_step.py --config c3 --steps 4 > gpurun_out/r2e_ncu_c3.log 2>&1; echo launches3=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_gs_rank|k_gs_scatter|k_direct_gather|k_resolve" -s 8 -c 4 -o gpurun_out/r2e_c3 python tools/profile_step.py --config c3 --steps 4 > gpurun_out/r2e_ncu_full.log 2>&1; echo ncufull=$?
