set -x
timeout 600 python tools/rad_time.py --profile > gpurun_out/rad_prof.log 2>&1; echo rad=$?
tail -3 gpurun_out/rad_prof.log
