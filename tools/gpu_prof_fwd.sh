# ncu of the cfg2 forward / backward (current defaults)
cd /root/repo
python tools/time_encode.py cfg2 3 > gpurun_out/pf_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 2 -c 1 \
    -o gpurun_out/pf_fwd -f python tools/time_encode.py cfg2 3 > gpurun_out/pf_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"bwd_kernel|merge_shift" -s 4 -c 2 \
    -o gpurun_out/pf_bwd -f python tools/time_encode.py cfg2 3 > gpurun_out/pf_ncub.log 2>&1
python bench.py --no-train --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/pf_bplain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"gather_levels|red_levels" -c 2 \
    -o gpurun_out/pf_mix -f python bench.py --no-train --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/pf_ncum.log 2>&1
ls gpurun_out
