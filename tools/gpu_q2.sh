set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/q2_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/q2_pytest.log
timeout 300 python tools/profile_step.py --config c3 --steps 10 --flush --time 2>&1 | grep "step ms"
timeout 300 python tools/profile_step.py --config c2 --steps 20 --flush --time 2>&1 | grep "step ms"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/q2_launches_c3.csv python tools/profile_step.py --config c3 --steps 3 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/q2_launches_c2.csv python tools/profile_step.py --config c2 --steps 3 > /dev/null 2>&1
