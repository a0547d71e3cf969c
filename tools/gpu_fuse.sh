# fused gather step (physics in the net's epilogue, pass 2 on records): parity, then A/B timing and launch lists
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or genome_sorted or tma_texture" > gpurun_out/f_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/f_pytest.log
for i in 1 2; do
timeout 300 python tools/profile_step.py --config c3 --steps 12 --flush --time > gpurun_out/f_c3_fused_$i.log 2>&1; tail -2 gpurun_out/f_c3_fused_$i.log
timeout 300 python tools/profile_step.py --config c3 --steps 12 --flush --time --flags 8192 > gpurun_out/f_c3_unfused_$i.log 2>&1; tail -2 gpurun_out/f_c3_unfused_$i.log
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/f_launches_c3.csv python tools/profile_step.py --config c3 --steps 3 > gpurun_out/f_ncu.log 2>&1; echo launches=$?
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_radiation.py tests/test_gpu_step_host.py -x -q > gpurun_out/f_pytest2.log 2>&1; echo pytest2=$?
tail -3 gpurun_out/f_pytest2.log
