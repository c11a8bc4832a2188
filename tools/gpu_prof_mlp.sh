# MLP train kernel (cfg4 shape, K0 = 64): parity tests, --set full capture with warp sampling
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_train_gpu.py -x -q --timeout 120 > gpurun_out/mlp_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/mlp_tests.log
timeout 300 python tools/time_train.py cfg4 3 > gpurun_out/mlp_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --warp-sampling-interval 2 --clock-control none -k regex:mlp_train_kernel -s 2 -c 1 -o gpurun_out/mlp_prof -f python tools/time_train.py cfg4 3 > gpurun_out/mlp_ncu.log 2>&1
echo prof rc=$?
ncu -i gpurun_out/mlp_prof.ncu-rep --page source --csv --print-source sass > gpurun_out/mlp_prof_source.csv 2>/dev/null
ncu -i gpurun_out/mlp_prof.ncu-rep --page raw --csv > gpurun_out/mlp_prof_raw.csv 2>/dev/null
ncu -i gpurun_out/mlp_prof.ncu-rep --page details > gpurun_out/mlp_prof_details.txt 2>/dev/null
rm -f gpurun_out/mlp_prof.ncu-rep
