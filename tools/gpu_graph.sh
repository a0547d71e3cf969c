set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "evo_run_graphs or run_equals or step_equals or determinis" > gpurun_out/g_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/g_pytest.log
for cfg in c1 c2; do
timeout 300 python tools/profile_step.py --config $cfg --steps 4 --run 1000 > gpurun_out/g_${cfg}_graph.log 2>&1; grep evo_run gpurun_out/g_${cfg}_graph.log
EVO_NO_GRAPH=1 timeout 300 python tools/profile_step.py --config $cfg --steps 4 --run 1000 > gpurun_out/g_${cfg}_eager.log 2>&1; grep evo_run gpurun_out/g_${cfg}_eager.log
done
timeout 300 python tools/profile_step.py --config c3 --steps 4 --run 100 > gpurun_out/g_c3_graph.log 2>&1; grep evo_run gpurun_out/g_c3_graph.log
EVO_NO_GRAPH=1 timeout 300 python tools/profile_step.py --config c3 --steps 4 --run 100 > gpurun_out/g_c3_eager.log 2>&1; grep evo_run gpurun_out/g_c3_eager.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/g_pytest_all.log 2>&1; echo pytest_all=$?
tail -3 gpurun_out/g_pytest_all.log
