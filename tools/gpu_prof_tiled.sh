mkdir -p gpurun_out
FH_SORTED=1 timeout 300 python tools/time_encode.py cfg2 3 && \
FH_SORTED=1 timeout 600 ncu --metrics gpu__time_duration.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct,smsp__warp_issue_stalled_barrier_per_warp_active.pct,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -s 40 -c 30 --csv python tools/time_encode.py cfg2 3 > gpurun_out/ncu_tiled.csv 2> gpurun_out/ncu_tiled.err
echo rc=$?
