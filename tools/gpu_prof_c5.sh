# ncu capture of the hidden-layer kernels on a config-5-shaped 4096^2 world
python tools/profile_step.py --config c5 --width 4096 --height 4096 --steps 2 > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_hid_sense|k_hid_net" -s 2 -c 2 -o gpurun_out/prof_c5 python tools/profile_step.py --config c5 --width 4096 --height 4096 --steps 2 > gpurun_out/ncu_c5.log 2>&1
for k in k_hid_sense k_hid_net; do ncu -i gpurun_out/prof_c5.ncu-rep --page source --csv --kernel-name regex:$k > gpurun_out/src_$k.csv 2>/dev/null; done
ncu -i gpurun_out/prof_c5.ncu-rep --page raw --csv > gpurun_out/raw_c5.csv 2>/dev/null
echo done
