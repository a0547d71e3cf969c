set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/h6_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/h6_pytest.log
for f in 0 1024; do timeout 300 python tools/profile_step.py --config c5 --width 4096 --height 4096 --steps 6 --flush --time --flags $f 2>&1 | grep "step ms"; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/h6_launches_c5.csv python tools/profile_step.py --config c5 --width 4096 --height 4096 --steps 3 > gpurun_out/h6_ncu.log 2>&1; echo launches=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_hid_net2" -s 1 -c 1 -o gpurun_out/h6_net2 python tools/profile_step.py --config c5 --width 4096 --height 4096 --steps 3 > gpurun_out/h6_ncufull.log 2>&1; echo ncufull=$?
