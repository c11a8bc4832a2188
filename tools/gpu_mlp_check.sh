# MLP train kernel: parity tests, train-step timing, per-launch kernel times (ncu launch list)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_train_gpu.py tests/test_umma_gpu.py -x -q --timeout 120 > gpurun_out/mlp_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/mlp_tests.log
for c in cfg3 cfg4; do
  timeout 300 python tools/time_train.py $c 10 > gpurun_out/mlp_time_$c.log 2>&1; echo time $c rc=$?; tail -3 gpurun_out/mlp_time_$c.log
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mlp_train_kernel --csv --log-file gpurun_out/mlp_launch_cfg4.csv python tools/time_train.py cfg4 3 > /dev/null 2>&1; echo ncu4 rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mlp_train_kernel --csv --log-file gpurun_out/mlp_launch_cfg3.csv python tools/time_train.py cfg3 3 > /dev/null 2>&1; echo ncu3 rc=$?
grep -h mlp_train gpurun_out/mlp_launch_cfg*.csv | awk -F'","' '{print $5, $NF}' | tail -12
