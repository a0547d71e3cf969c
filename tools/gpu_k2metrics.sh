# k_resolve instruction count / issue / occupancy / stalls for library variants (config 2)
for lib in "$@"; do
  EVOCA_B200_LIB=$PWD/paper_2406_09654_b200/$lib ncu --kernel-name regex:k_resolve --launch-skip 3 --launch-count 1 \
    --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread,smsp__warps_issue_stalled_barrier_per_warp_active.pct,smsp__warps_issue_stalled_long_scoreboard_per_warp_active.pct,smsp__warps_issue_stalled_wait_per_warp_active.pct,smsp__warps_issue_stalled_short_scoreboard_per_warp_active.pct,smsp__cycles_active.avg,sm__cycles_elapsed.avg \
    --csv python tools/profile_step.py --steps 6 > gpurun_out/k2m_$lib.csv 2>/dev/null
done
