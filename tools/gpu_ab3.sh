set -x
for i in 1 2; do
timeout 300 python tools/profile_step.py --config c2 --steps 12 --flush --time > gpurun_out/ab_c2_tile_$i.log 2>&1; tail -2 gpurun_out/ab_c2_tile_$i.log
timeout 300 python tools/profile_step.py --config c2 --steps 12 --flush --time --flags 1024 > gpurun_out/ab_c2_gather_$i.log 2>&1; tail -2 gpurun_out/ab_c2_gather_$i.log
done
timeout 300 python tools/profile_step.py --config c1 --steps 12 --time > gpurun_out/ab_c1_tile.log 2>&1; tail -2 gpurun_out/ab_c1_tile.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/ab_launches_c2g.csv python tools/profile_step.py --config c2 --steps 3 --flags 1024 > gpurun_out/ab_ncu.log 2>&1; echo launches=$?
