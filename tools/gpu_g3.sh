# tcgen05 issue cost / A-in-TMEM layout microbenches; gather path with vectorised sort + dynamic runs
set -x
./tools/microbench/tc_issue > gpurun_out/g3_tc_issue.log 2>&1; echo issue=$?
./tools/microbench/tc_tmem_a > gpurun_out/g3_tc_tmem_a.log 2>&1; echo tmema=$?
timeout 900 python -m pytest tests -m gpu -x -q -k "genome_sorted or gather or config3" > gpurun_out/g3_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/g3_pytest.log
for f in 0 512; do timeout 300 python tools/profile_step.py --config c3 --steps 8 --flush --time --flags $f 2>&1 | grep "step ms"; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/g3_launches_c3.csv python tools/profile_step.py --config c3 --steps 3 > gpurun_out/g3_ncu.log 2>&1; echo launches=$?
