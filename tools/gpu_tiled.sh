mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "tiled or spatial" 2>&1 | tail -3
for c in cfg2 cfg4; do
  timeout 300 python tools/time_encode.py $c 10
  FH_SORTED=1 timeout 300 python tools/time_encode.py $c 10
  FH_SORTED=1 FH_FINE_ORDER=1 timeout 300 python tools/time_encode.py $c 10
  FH_SORTED=1 FH_AGG_MIN_DENSITY=4 timeout 300 python tools/time_encode.py $c 10
  FH_SORTED=1 FH_AGG_MIN_DENSITY=0.4 timeout 300 python tools/time_encode.py $c 10
done
FH_SORTED=1 timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -s 40 -c 16 --csv python tools/time_encode.py cfg2 3 > gpurun_out/ncu_tiled.csv 2> gpurun_out/ncu_tiled.err
