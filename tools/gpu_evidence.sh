# Round evidence on one B200: GPU tests, bench lines (config 2 headline,
# config 3 genome-sorted path), launch list of the config-2 bench command,
# ncu --set full of the config-2 step kernels, of the config-3 genome-sorted
# kernels and of the hidden-layer kernels (config-5 shape).  Outputs under
# gpurun_out/ with prefix $1 (default ev).
P=${1:-ev}
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${P}_pytest.log 2>&1; tail -1 gpurun_out/${P}_pytest.log
python bench.py --steps 50 --warmup 5 > gpurun_out/${P}_bench.log 2>&1; tail -1 gpurun_out/${P}_bench.log
python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${P}_bench_c3.log 2>&1; tail -1 gpurun_out/${P}_bench_c3.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${P}_launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${P}_ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pass1_direct|k_resolve" -s 4 -c 2 \
    -o gpurun_out/${P}_c2 python tools/profile_step.py --steps 4 > gpurun_out/${P}_ncu_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_hid_sense|k_direct_rows|k_physics_rows|k_resolve" -s 8 -c 4 \
    -o gpurun_out/${P}_c3 python tools/profile_step.py --config c3 --steps 3 > gpurun_out/${P}_ncu_c3.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/${P}_launches_c3.csv python tools/profile_step.py --config c3 --steps 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_hid_net|k_hid_sense" -s 2 -c 2 \
    -o gpurun_out/${P}_c5 python tools/profile_step.py --config c5 --width 4096 --height 4096 --steps 2 > gpurun_out/${P}_ncu_c5.log 2>&1
python tools/profile_step.py --config c5 --width 4096 --height 4096 --steps 5 --time > gpurun_out/${P}_c5_time.log 2>&1
python tools/profile_step.py --config c3 --steps 8 --flush --time > gpurun_out/${P}_c3_time.log 2>&1
echo done
