mkdir -p gpurun_out
FH_SORTED=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:bwd_tiled -s 1 -c 1 -o gpurun_out/bwd_tiled python tools/time_encode.py cfg2 2 > gpurun_out/ncu_bwd.log 2>&1
echo rc=$?
