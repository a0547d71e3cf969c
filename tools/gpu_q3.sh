# quick: gather-path parity subset + config-3 timing (+ optional extra flags in $FLAGS)
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "genome_sorted or gather or config3 or tc_direct" > gpurun_out/q_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/q_pytest.log
for f in 0 2048; do timeout 300 python tools/profile_step.py --config c3 --steps 10 --flush --time --flags $f 2>&1 | grep "step ms"; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/q_launches_c3.csv python tools/profile_step.py --config c3 --steps 3 --flags 2048 > gpurun_out/q_ncu.log 2>&1; echo launches=$?
