# compute-sanitizer over the sanitizer workload, one tool per run (bounded)
set -x
timeout 300 python tools/sanitize_step.py > gpurun_out/san_plain.log 2>&1; echo plain=$?
tail -2 gpurun_out/san_plain.log
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_step.py > gpurun_out/san_$tool.log 2>&1; echo $tool=$?
  tail -4 gpurun_out/san_$tool.log
done
