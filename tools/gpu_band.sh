set -x
for b in 262144 524288 1048576 2097152 4194304; do
EVO_BAND_CELLS=$b timeout 300 python tools/profile_step.py --config c3 --steps 12 --flush --time > gpurun_out/band_$b.log 2>&1; echo band=$b; tail -2 gpurun_out/band_$b.log | head -1 | cut -c100-
done
for b in 524288 1048576 2097152; do
EVO_BAND_CELLS=$b timeout 600 python tools/profile_step.py --config c4 --steps 5 --flush --time > gpurun_out/band_c4_$b.log 2>&1; echo c4 band=$b; tail -2 gpurun_out/band_c4_$b.log | head -1
done
