set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q > gpurun_out/ab_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/ab_pytest.log
for i in 1 2; do
timeout 300 python tools/profile_step.py --config c3 --steps 12 --flush --time > gpurun_out/ab_c3_$i.log 2>&1; tail -2 gpurun_out/ab_c3_$i.log
done
timeout 300 python tools/profile_step.py --config c2 --steps 12 --flush --time > gpurun_out/ab_c2.log 2>&1; tail -2 gpurun_out/ab_c2.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/ab_launches_c3.csv python tools/profile_step.py --config c3 --steps 3 > gpurun_out/ab_ncu.log 2>&1; echo launches=$?
