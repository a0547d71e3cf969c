# gather path with atomic-free scatter and per-lane rotation
set -x
timeout 900 python -m pytest tests -m gpu -x -q -s -k "tc_direct or genome_sorted or gather or config3" > gpurun_out/g11_pytest.log 2>&1; echo pytest=$?
grep -E "passed|failed|tcgen05" gpurun_out/g11_pytest.log
for f in 4096 0 2048; do timeout 300 python tools/profile_step.py --config c3 --steps 8 --flush --time --flags $f 2>&1 | grep "step ms"; done
for f in 5120; do timeout 300 python tools/profile_step.py --config c2 --steps 12 --flush --time --flags $f 2>&1 | grep "step ms"; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/g11_launches_c3.csv python tools/profile_step.py --config c3 --steps 3 --flags 4096 > gpurun_out/g11_ncu.log 2>&1; echo launches=$?
