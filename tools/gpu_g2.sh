# full ncu capture of the gather path's kernels on config 3
set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_direct_gather|k_gs_count|k_gs_scatter" -s 3 -c 3 -o gpurun_out/g2_c3 python tools/profile_step.py --config c3 --steps 3 > gpurun_out/g2_ncu.log 2>&1; echo ncufull=$?
