# ncu of the cfg2 forward with and without the shifted table copy
cd /root/repo
FH_PAIR_SHIFT=1 python tools/time_encode.py cfg2 3 > gpurun_out/pf_plain1.log 2>&1 &&
FH_PAIR_SHIFT=3 python tools/time_encode.py cfg2 3 > gpurun_out/pf_plain3.log 2>&1 &&
FH_PAIR_SHIFT=1 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 2 -c 1 \
    -o gpurun_out/pf_fwd1 -f python tools/time_encode.py cfg2 3 > gpurun_out/pf_ncu1.log 2>&1
FH_PAIR_SHIFT=3 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 2 -c 1 \
    -o gpurun_out/pf_fwd3 -f python tools/time_encode.py cfg2 3 > gpurun_out/pf_ncu3.log 2>&1
FH_PAIR_SHIFT=1 ncu --set full --clock-control none --import-source on -k regex:bwd_kernel -s 2 -c 1 \
    -o gpurun_out/pf_bwd1 -f python tools/time_encode.py cfg2 3 > gpurun_out/pf_ncub1.log 2>&1
ls -la gpurun_out/
