# Round-1 GPU evidence: tests, smoke, bench, ncu launch list of the bench
# command, full captures of the dominant kernels.  Run under gpurun.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -5 > gpurun_out/r01_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01_smoke.log 2>&1
CMD="python bench.py --steps 20 --warmup 5"
timeout 900 $CMD > gpurun_out/r01_bench.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_bench_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r01_ncu_launch.log 2>&1
echo launch rc=$?
timeout 600 python tools/time_encode.py cfg2 2 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:fwd_kernel|bwd_kernel" -s 2 -c 2 -o gpurun_out/r01_encode_cfg2 python tools/time_encode.py cfg2 1 > gpurun_out/r01_ncu_encode.log 2>&1
echo full rc=$?
timeout 900 ncu --set full --clock-control none -k "regex:fwd_kernel|bwd_kernel" -s 6 -c 4 -o gpurun_out/r01_encode_cfg4 python tools/time_encode.py cfg4 1 > gpurun_out/r01_ncu_encode4.log 2>&1
timeout 900 ncu --set full --clock-control none -k "regex:feature_kernel|occupancy_kernel|dilate_kernel|emit_kernel" -s 5 -c 4 -o gpurun_out/r01_coreset python tools/time_coreset.py 1 > gpurun_out/r01_ncu_coreset.log 2>&1
echo done
