timeout 600 python -m pytest tests/test_radiation.py -m gpu -q -s -p no:cacheprovider -k "components" > gpurun_out/r2e_pytest.log 2>&1; echo pytest=$?; grep -E "vs exact|passed|failed" gpurun_out/r2e_pytest.log | tail -5
for v in 1 2; do
  if [ $v = 1 ]; then export EVO_SENSE_V1=1; else unset EVO_SENSE_V1; fi
  timeout 300 python tools/profile_step.py --config c3 --steps 8 --flush --time > gpurun_out/r2e_prof_v$v.log 2>&1; echo prof$v=$?; tail -2 gpurun_out/r2e_prof_v$v.log
done
unset EVO_SENSE_V1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "genome_sorted or tensor_core or hidden" > gpurun_out/r2e_pytest2.log 2>&1; echo pytest2=$?; tail -1 gpurun_out/r2e_pytest2.log
python tools/profile_step.py --config c3 --steps 4 > gpurun_out/r2e_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2e_launches_c3.csv python tools/profile_step.py --config c3 --steps 4 > gpurun_out/r2e_ncu.log 2>&1; echo ncu=$?
