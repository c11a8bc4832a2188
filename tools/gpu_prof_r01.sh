set -x
mkdir -p gpurun_out
timeout 300 python tools/time_train.py cfg3 10
timeout 300 python tools/time_train.py cfg4 5
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/bench_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo launch rc=$?
timeout 300 python tools/time_train.py cfg3 3 > gpurun_out/tt_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:mlp_train|adam_kernel|fwd_kernel|bwd_kernel" -s 8 -c 4 -o gpurun_out/prof_train_cfg3 python tools/time_train.py cfg3 3 > gpurun_out/ncu_train.log 2>&1
echo full rc=$?
