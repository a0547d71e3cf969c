set -x
for b in 1048576 4194304 16777216; do EVO_HG_BAND=$b timeout 300 python tools/profile_step.py --config c5 --width 4096 --height 4096 --steps 5 --flush --time --flags 1024 2>&1 | grep "step ms"; done
timeout 300 python tools/profile_step.py --config c5 --width 4096 --height 4096 --steps 5 --flush --time --flags 0 2>&1 | grep "step ms"
