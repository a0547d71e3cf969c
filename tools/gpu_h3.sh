# hidden net with layer 2 on tcgen05 (k_hid_net2): parity + timing + ncu
set -x
timeout 900 python -m pytest tests -m gpu -x -q -s -k "tensor_core or hidden or config5 or radiation" > gpurun_out/h3_pytest.log 2>&1; echo pytest=$?
grep -E "passed|failed|H=|Error" gpurun_out/h3_pytest.log | head -20
for f in 0 4096; do timeout 300 python tools/profile_step.py --config c5 --width 4096 --height 4096 --steps 6 --flush --time --flags $f 2>&1 | grep "step ms"; done
