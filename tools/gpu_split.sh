cd /root/repo
python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -2
for cfg in cfg4 pc cfg2; do for sp in 0 1; do echo -n "split=$sp "; FH_BWD_SPLIT=$sp FH_OVERWRITE=1 python tools/time_encode.py $cfg 10; done; done
for mb in 24 32 40; do echo -n "split=1 mb=$mb "; FH_BWD_GROUP_MB=$mb FH_OVERWRITE=1 python tools/time_encode.py cfg4 10; done
