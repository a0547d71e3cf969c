set -x
timeout 600 python tools/rad_time.py > gpurun_out/rad_time.log 2>&1; echo rad=$?
cat gpurun_out/rad_time.log | tail -6
timeout 600 python -c "
import cProfile, pstats, sys
sys.path.insert(0,'.')
exec(open('tools/rad_time.py').read().split('for k in range(4):')[0])
import time
st.substrate.step_counter = 250
pr = cProfile.Profile(); pr.enable()
for k in range(3):
    radiation.field_radiation(st, 50*(k+5), 0.01); dev.sync()
pr.disable(); pstats.Stats(pr).sort_stats('cumtime').print_stats(25)
" > gpurun_out/rad_prof.log 2>&1; echo prof=$?
