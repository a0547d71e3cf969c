# A/B of library builds on config 2: ncu launch durations of pass 1 and pass 2
for lib in "$@"; do
  EVOCA_B200_LIB=$PWD/paper_2406_09654_b200/$lib ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab2_$lib.csv python tools/profile_step.py --steps 8 > /dev/null 2>&1
  for k in k_pass1 k_resolve; do
    echo $lib $k $(grep $k gpurun_out/ab2_$lib.csv | awk -F'","' '{print $(NF)}' | tr -d '"' | tail -5 | tr '\n' ' ')
  done
done
