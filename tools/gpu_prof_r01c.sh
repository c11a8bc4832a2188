# round-1 evidence refresh after the shifted pairs / level table / occupancy changes
cd /root/repo; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r01c_bench.log 2>&1; echo bench rc=$?
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r01c_bench_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01c_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r01c_ncu_launch.log 2>&1
echo launch rc=$?
timeout 300 python tools/time_encode.py cfg2 3 > gpurun_out/r01c_enc_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:fwd_kernel|bwd_kernel|merge_shift|bwd_small" -s 8 -c 7 -o gpurun_out/r01c_encode_cfg2 -f python tools/time_encode.py cfg2 3 > gpurun_out/r01c_ncu_enc.log 2>&1
echo enc rc=$?
timeout 300 python tools/time_encode.py cfg4 2 > gpurun_out/r01c_enc4_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k "regex:fwd_kernel|bwd_kernel" -s 12 -c 4 -o gpurun_out/r01c_encode_cfg4 -f python tools/time_encode.py cfg4 2 > gpurun_out/r01c_ncu_enc4.log 2>&1
echo enc4 rc=$?
