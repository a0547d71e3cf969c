# fused gather step: full suite, bench, ncu full capture of the fused net and the record-reading pass 2
set -x
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/f2_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/f2_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/f2_bench_c3.log 2>&1; echo bench=$?
tail -1 gpurun_out/f2_bench_c3.log | cut -c1-400
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_direct_gather|k_resolve" -s 4 -c 2 -o gpurun_out/f2_prof python tools/profile_step.py --config c3 --steps 4 > gpurun_out/f2_ncu.log 2>&1; echo ncu=$?
ncu -i gpurun_out/f2_prof.ncu-rep --page source --csv > gpurun_out/f2_src.csv 2>/dev/null
