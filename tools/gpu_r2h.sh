timeout 300 python tools/diag_engine.py > gpurun_out/r2h_diag.log 2>&1; echo diag=$?; tail -5 gpurun_out/r2h_diag.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_strips.py tests/test_radiation.py -x -q -p no:cacheprovider -m gpu > gpurun_out/r2h_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/r2h_pytest.log
for cfg in c2 c3; do timeout 300 python tools/profile_step.py --config $cfg --steps 8 --flush --time > gpurun_out/r2h_prof_$cfg.log 2>&1; echo prof$cfg=$?; tail -2 gpurun_out/r2h_prof_$cfg.log | head -1; done
export EVO_K2_TILES=1
for cfg in c2 c3; do timeout 300 python tools/profile_step.py --config $cfg --steps 8 --flush --time > gpurun_out/r2h_prof_${cfg}_tiles.log 2>&1; echo prof${cfg}tiles=$?; tail -2 gpurun_out/r2h_prof_${cfg}_tiles.log | head -1; done
unset EVO_K2_TILES
python tools/profile_step.py --config c3 --steps 3 > gpurun_out/r2h_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/r2h_launches_c3.csv python tools/profile_step.py --config c3 --steps 3 > gpurun_out/r2h_ncu.log 2>&1; echo ncu=$?
