mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r01b_bench.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01b_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r01b_ncu_launch.log 2>&1
echo launch rc=$?
timeout 300 python tools/time_coreset.py 2 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none -k "regex:feature_kernel|occupancy_kernel|dilate_kernel|emit_kernel|cellrow_kernel" -s 5 -c 5 -o gpurun_out/r01b_coreset python tools/time_coreset.py 1 > gpurun_out/r01b_ncu_coreset.log 2>&1
echo coreset rc=$?
