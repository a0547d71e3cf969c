# config-5 net on a 4096^2 torus (4096 genomes, 45->128->13): parity subset, step time (rows form,
# round-2 layer-2-on-CUDA-cores kernel, gather form), launch list with tensor-pipe activity
set -x
timeout 900 python -m pytest tests -m gpu -x -q -s -k "tensor_core or hidden or config5" > gpurun_out/c5_pytest.log 2>&1; echo pytest=$?
for f in 0 4096; do timeout 300 python tools/profile_step.py --config c5 --width 4096 --height 4096 --steps 6 --flush --time --flags $f 2>&1 | grep "step ms"; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/c5_launches.csv python tools/profile_step.py --config c5 --width 4096 --height 4096 --steps 3 > /dev/null 2>&1
