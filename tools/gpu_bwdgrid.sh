cd /root/repo
for cfg in cfg2 cfg3 pc; do for mb in 24 32 40 48 56 69 80; do
  echo -n "bwd_mb=$mb "; FH_BWD_GROUP_MB=$mb python tools/time_encode.py $cfg 20
done; done
