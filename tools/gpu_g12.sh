# full ncu of the FFMA gather net and the tcgen05 net on config 3 (L1 / writeback / latency split)
set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_direct_gather|k_direct_tc" -s 1 -c 1 -o gpurun_out/g12_ffma python tools/profile_step.py --config c3 --steps 3 > gpurun_out/g12_a.log 2>&1; echo a=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_direct_gather|k_direct_tc" -s 1 -c 1 -o gpurun_out/g12_tc python tools/profile_step.py --config c3 --steps 3 --flags 2048 > gpurun_out/g12_b.log 2>&1; echo b=$?
