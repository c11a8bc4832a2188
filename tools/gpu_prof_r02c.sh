# round-2 evidence, final state: the reworked MLP train kernel (cfg4 shape,
# K0 = 64) and fused inference (cfg3, 1024 samples) under --set full, and
# the cfg3 train step's launch list.  Each program runs once without ncu first.
mkdir -p gpurun_out
timeout 300 python tools/time_train.py cfg4 3 > gpurun_out/r02c_train_cfg4_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --warp-sampling-interval 2 --clock-control none -k regex:mlp_train_kernel -s 2 -c 1 -o gpurun_out/r02c_mlp_cfg4 -f python tools/time_train.py cfg4 3 > gpurun_out/r02c_ncu_mlp.log 2>&1
echo mlp rc=$?
timeout 300 python tools/infer_once.py cfg3 1024 > gpurun_out/r02c_infer_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:infer_fused -s 3 -c 1 -o gpurun_out/r02c_infer_1024 -f python tools/infer_once.py cfg3 1024 > gpurun_out/r02c_ncu_infer.log 2>&1
echo infer rc=$?
timeout 300 python tools/time_train.py cfg3 3 > gpurun_out/r02c_train_cfg3_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02c_train_cfg3_launches.csv python tools/time_train.py cfg3 3 > gpurun_out/r02c_ncu_train3.log 2>&1
echo train3 rc=$?
for r in r02c_mlp_cfg4 r02c_infer_1024; do
  python tools/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/${r}_summary.txt 2>&1
  ncu -i gpurun_out/$r.ncu-rep --page details > gpurun_out/${r}_details.txt 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/${r}_source.csv 2>/dev/null
done
python tools/mlp_phases.py gpurun_out/r02c_mlp_cfg4_source.csv > gpurun_out/r02c_mlp_cfg4_phases.txt 2>&1
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out | head -40
# bench launch list (every kernel the default bench launches; cold-cache, serialised)
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02c_bench_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02c_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02c_ncu_launch.log 2>&1
echo launches rc=$?
