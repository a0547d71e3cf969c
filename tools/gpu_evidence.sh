# Round evidence on one B200: GPU tests, bench line, launch list of the same
# bench command, ncu --set full of both step kernels (config 2) and of the
# hidden-layer kernels (config-5 shape).  Outputs under gpurun_out/.
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ev_pytest.log 2>&1; tail -1 gpurun_out/ev_pytest.log
python bench.py --steps 50 --warmup 5 > gpurun_out/ev_bench.log 2>&1; tail -1 gpurun_out/ev_bench.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev_launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ev_ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pass1_direct|k_resolve" -s 4 -c 2 \
    -o gpurun_out/ev_c2 python tools/profile_step.py --steps 4 > gpurun_out/ev_ncu_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_hid_net|k_hid_sense" -s 2 -c 2 \
    -o gpurun_out/ev_c5 python tools/profile_step.py --config c5 --width 4096 --height 4096 --steps 2 > gpurun_out/ev_ncu_c5.log 2>&1
python tools/profile_step.py --config c5 --width 4096 --height 4096 --steps 5 --time > gpurun_out/ev_c5_time.log 2>&1
echo done
