set -x
for lib in libevoca_b200.so libevoca_b200_nohist.so; do
EVOCA_B200_LIB=$PWD/paper_2406_09654_b200/$lib timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/nh_$lib.csv python tools/profile_step.py --config c3 --steps 3 > /dev/null 2>&1
done
