set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q > gpurun_out/ab_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/ab_pytest.log
for i in 1 2; do
timeout 300 python tools/profile_step.py --config c3 --steps 12 --flush --time > gpurun_out/ab_c3_$i.log 2>&1; tail -2 gpurun_out/ab_c3_$i.log
done
timeout 300 python tools/profile_step.py --config c2 --steps 12 --flush --time > gpurun_out/ab_c2.log 2>&1; tail -2 gpurun_out/ab_c2.log
timeout 300 python tools/profile_step.py --config c5 --width 4096 --height 4096 --steps 6 --flush --time > gpurun_out/ab_c5.log 2>&1; tail -2 gpurun_out/ab_c5.log
for i in 1 2; do
timeout 900 python bench.py --strips --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_bench_strips_$i.log 2>&1; tail -1 gpurun_out/ab_bench_strips_$i.log | cut -c1-220
done
timeout 900 python bench.py --strips --steps 40 --warmup 12 --no-cpu-baseline > gpurun_out/ab_bench_strips_3.log 2>&1; tail -1 gpurun_out/ab_bench_strips_3.log | cut -c1-220
