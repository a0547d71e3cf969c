set -x
timeout 900 python -m pytest tests -m gpu -x -q -s -k "tensor_core or hidden or config5" > gpurun_out/hb3_pytest.log 2>&1; echo pytest=$?
grep -E "passed|failed|H=|Error" gpurun_out/hb3_pytest.log | head
for f in 1024 0; do timeout 300 python tools/profile_step.py --config c5 --width 4096 --height 4096 --steps 6 --flush --time --flags $f 2>&1 | grep "step ms"; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/hb3_launches.csv python tools/profile_step.py --config c5 --width 4096 --height 4096 --steps 3 --flags 1024 > /dev/null 2>&1
