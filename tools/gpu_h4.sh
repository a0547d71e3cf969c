# hidden net over the gather sort: parity + timing + launch list
set -x
timeout 1200 python -m pytest tests -m gpu -x -q -s -k "tensor_core or hidden or config5 or radiation or step_host or snapshot or state" > gpurun_out/h4_pytest.log 2>&1; echo pytest=$?
grep -E "passed|failed|H=|Error|assert" gpurun_out/h4_pytest.log | head -20
for f in 0 512 4096; do timeout 300 python tools/profile_step.py --config c5 --width 4096 --height 4096 --steps 6 --flush --time --flags $f 2>&1 | grep "step ms"; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/h4_launches_c5.csv python tools/profile_step.py --config c5 --width 4096 --height 4096 --steps 3 > gpurun_out/h4_ncu.log 2>&1; echo launches=$?
