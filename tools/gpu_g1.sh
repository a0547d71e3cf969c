# gather path: parity subset + timing A/B (gather vs rows on c3; gather vs tile on c2)
set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "genome_sorted or gather or config3 or step_host or radiation" > gpurun_out/g1_pytest.log 2>&1; echo pytest=$?
tail -15 gpurun_out/g1_pytest.log
for f in 0 512; do timeout 300 python tools/profile_step.py --config c3 --steps 8 --flush --time --flags $f 2>&1 | grep "step ms"; done
for f in 0 1024; do timeout 300 python tools/profile_step.py --config c2 --steps 12 --flush --time --flags $f 2>&1 | grep "step ms"; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/g1_launches_c3.csv python tools/profile_step.py --config c3 --steps 3 > gpurun_out/g1_ncu.log 2>&1; echo launches=$?
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/g1_launches_c2.csv python tools/profile_step.py --config c2 --steps 3 --flags 1024 > gpurun_out/g1_ncu2.log 2>&1; echo launches2=$?
