# MLP train kernel (cfg4 shape, K0 = 64) stall profile + full bench line
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/r2u_bench.log 2>&1; echo bench rc=$?
timeout 300 python tools/time_train.py cfg4 3 20 > gpurun_out/r2u_train_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --warp-sampling-interval 2 --clock-control none -k regex:mlp_train_kernel -s 2 -c 1 -o gpurun_out/r2u_mlp -f python tools/time_train.py cfg4 3 20 > gpurun_out/r2u_ncu.log 2>&1
echo mlp rc=$?
ncu -i gpurun_out/r2u_mlp.ncu-rep --page source --csv --print-source sass > gpurun_out/r2u_mlp_source.csv 2>/dev/null
ncu -i gpurun_out/r2u_mlp.ncu-rep --page raw --csv > gpurun_out/r2u_mlp_raw.csv 2>/dev/null
rm -f gpurun_out/r2u_mlp.ncu-rep
