cd /root/repo
python -m pytest tests/test_parity_gpu.py tests/test_mhe_gpu.py tests/test_stats_gpu.py tests/test_train_gpu.py -x -q 2>&1 | tail -2
for cfg in cfg2 cfg3 cfg4 pc; do FH_OVERWRITE=1 python tools/time_encode.py $cfg 20; done
