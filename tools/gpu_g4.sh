# tcgen05 direct net: parity + timing A/B on config 3 and config 2
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "tc_direct or genome_sorted or gather" > gpurun_out/g4_pytest.log 2>&1; echo pytest=$?
tail -30 gpurun_out/g4_pytest.log | grep -v "^\s*$" | tail -25
for f in 2048 0 512; do timeout 300 python tools/profile_step.py --config c3 --steps 8 --flush --time --flags $f 2>&1 | grep "step ms"; done
for f in 3072 1024 0; do timeout 300 python tools/profile_step.py --config c2 --steps 12 --flush --time --flags $f 2>&1 | grep "step ms"; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/g4_launches_c3.csv python tools/profile_step.py --config c3 --steps 3 --flags 2048 > gpurun_out/g4_ncu.log 2>&1; echo launches=$?
