timeout 600 python tools/e2e_bands.py c3 4 8 12 16 24 > gpurun_out/e2e_bands.log 2>&1; echo e2e=$?; cat gpurun_out/e2e_bands.log | tail -6
