# tcgen05 direct net v2 (two accumulators, A_lo in smem): accuracy + timing
set -x
timeout 900 python -m pytest tests -m gpu -q -rxX -k "tc_direct" > gpurun_out/g7_pytest.log 2>&1; echo pytest=$?
grep -E "passed|failed|XPASS|XFAIL|rel_err|assert" gpurun_out/g7_pytest.log | head -20
for f in 2048 0; do timeout 300 python tools/profile_step.py --config c3 --steps 8 --flush --time --flags $f 2>&1 | grep "step ms"; done
for f in 3072 0; do timeout 300 python tools/profile_step.py --config c2 --steps 12 --flush --time --flags $f 2>&1 | grep "step ms"; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/g7_launches_c3.csv python tools/profile_step.py --config c3 --steps 3 --flags 2048 > gpurun_out/g7_ncu.log 2>&1; echo launches=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_direct_tc" -s 1 -c 1 -o gpurun_out/g7_tc python tools/profile_step.py --config c3 --steps 3 --flags 2048 > gpurun_out/g7_ncufull.log 2>&1; echo ncufull=$?
