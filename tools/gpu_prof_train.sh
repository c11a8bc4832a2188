# ncu of the cfg3 train-step kernels (after the MLP gradient flush / overwrite changes)
cd /root/repo; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r01g_bench.log 2>&1; echo bench rc=$?
timeout 300 python tools/time_train.py cfg3 3 > gpurun_out/r01g_train_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k "regex:mlp_train_kernel|mlp_grad_reduce|adam_kernel|fwd_kernel|bwd_kernel|merge_shift" -s 20 -c 10 -o gpurun_out/r01g_train_cfg3 -f python tools/time_train.py cfg3 3 > gpurun_out/r01g_ncu_train.log 2>&1
echo train rc=$?
