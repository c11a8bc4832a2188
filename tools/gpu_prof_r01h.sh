# round-1 evidence refresh (final kernels of the session)
cd /root/repo; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r01h_bench.log 2>&1; echo bench rc=$?
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r01h_bench_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01h_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r01h_ncu_launch.log 2>&1
echo launch rc=$?
FH_OVERWRITE=1 timeout 300 python tools/time_encode.py cfg2 3 > gpurun_out/r01h_enc_plain.log 2>&1 && \
FH_OVERWRITE=1 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:fwd_kernel|bwd_kernel|merge_shift" -s 6 -c 6 -o gpurun_out/r01h_encode_cfg2 -f python tools/time_encode.py cfg2 3 > gpurun_out/r01h_ncu_enc.log 2>&1
echo enc rc=$?
FH_OVERWRITE=1 timeout 300 python tools/time_encode.py pc 2 > gpurun_out/r01h_pc_plain.log 2>&1 && \
FH_OVERWRITE=1 timeout 900 ncu --set full --clock-control none -k "regex:bwd_small|bwd_kernel" -s 4 -c 4 -o gpurun_out/r01h_encode_pc -f python tools/time_encode.py pc 2 > gpurun_out/r01h_ncu_pc.log 2>&1
echo pc rc=$?
timeout 300 python tools/time_coreset.py 2 > gpurun_out/r01h_cs_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k "regex:feature_kernel|occupancy_kernel|dilate_kernel|emit_kernel|cellrow_kernel" -s 5 -c 5 -o gpurun_out/r01h_coreset -f python tools/time_coreset.py 2 > gpurun_out/r01h_ncu_coreset.log 2>&1
echo coreset rc=$?
