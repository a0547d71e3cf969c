# full ncu capture of one k_pass1_direct launch (config c2) + SASS source view
tag=${1:-x}
python tools/profile_step.py --steps 4 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${2:-k_pass1_direct} -s 2 -c 1 -o gpurun_out/prof_$tag python tools/profile_step.py --steps 4 > gpurun_out/ncu_$tag.log 2>&1
ncu -i gpurun_out/prof_$tag.ncu-rep --page source --csv > gpurun_out/src_$tag.csv 2>/dev/null
ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/raw_$tag.csv 2>/dev/null
echo done
