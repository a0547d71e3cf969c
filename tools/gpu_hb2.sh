set -x
EVO_HG_CONTIG=1 EVO_HG_BAND=16777216 timeout 300 python tools/profile_step.py --config c5 --width 4096 --height 4096 --steps 5 --flush --time --flags 1024 2>&1 | grep "step ms"
EVO_HG_CONTIG=1 timeout 300 python tools/profile_step.py --config c5 --width 4096 --height 4096 --steps 5 --flush --time --flags 1024 2>&1 | grep "step ms"
EVO_HG_CONTIG=1 EVO_HG_BAND=16777216 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/hb2_launches.csv python tools/profile_step.py --config c5 --width 4096 --height 4096 --steps 3 --flags 1024 > /dev/null 2>&1
