set -x
timeout 900 python bench.py --strips --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bs_strips.log 2>&1; echo strips=$?
tail -1 gpurun_out/bs_strips.log | cut -c1-900
tail -5 gpurun_out/bs_strips.log | grep -i error
