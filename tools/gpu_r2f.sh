timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "cluster_sharded or genome_sorted" > gpurun_out/r2f_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/r2f_pytest.log
timeout 300 python tools/profile_step.py --config c3 --steps 8 --flush --time > gpurun_out/r2f_prof.log 2>&1; echo prof=$?; tail -2 gpurun_out/r2f_prof.log
timeout 300 python tools/profile_step.py --config c3 --steps 8 --flush --time --flags 256 > gpurun_out/r2f_prof_rows.log 2>&1; echo profrows=$?; tail -2 gpurun_out/r2f_prof_rows.log
timeout 900 python -m pytest tests/test_gpu_scale.py -x -q -p no:cacheprovider -k "config3" > gpurun_out/r2f_pytest2.log 2>&1; echo pytest2=$?; tail -2 gpurun_out/r2f_pytest2.log
