for lib in libevoca_b200.so libevoca_b200_k2g2.so libevoca_b200_k2g4.so; do
  EVOCA_B200_LIB=$PWD/paper_2406_09654_b200/$lib ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/k2g_$lib.csv python tools/profile_step.py --steps 6 > /dev/null 2>&1
  echo $lib; grep k_resolve gpurun_out/k2g_$lib.csv | awk -F'","' '{print $(NF)}' | tail -3
done
