# round-2d evidence: full GPU suite + smoke, headline bench (default c3), reference arm, strips bench on one GPU,
# config 2 / 4 lines, config-5 slice timing, launch lists of the bench commands
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2d_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/r2d_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2d_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2d_bench_c3.log 2>&1; echo bench=$?
tail -1 gpurun_out/r2d_bench_c3.log | cut -c1-300
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2d_bench_ref.log 2>&1; echo ref=$?
timeout 900 python bench.py --strips --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2d_bench_strips.log 2>&1; echo strips=$?
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2d_bench_c2.log 2>&1; echo c2=$?
timeout 1500 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2d_bench_c4.log 2>&1; echo c4=$?
timeout 300 python tools/profile_step.py --config c5 --width 4096 --height 4096 --steps 6 --flush --time > gpurun_out/r2d_c5.log 2>&1; echo c5=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/r2d_launches_bench_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2d_ncu_bench.log 2>&1; echo launches=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/r2d_launches_bench_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2d_ncu_bench2.log 2>&1; echo launches2=$?
