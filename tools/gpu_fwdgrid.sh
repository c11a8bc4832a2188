cd /root/repo
python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -1
for cfg in cfg2 cfg3 pc cfg4; do for mb in 24 32 40 48 56 69; do
  echo -n "mb=$mb "; FH_OVERWRITE=1 FH_FWD_GROUP_MB=$mb python tools/time_encode.py $cfg 20
done; done
