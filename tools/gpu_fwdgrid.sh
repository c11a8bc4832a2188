cd /root/repo
for cfg in cfg2 pc cfg3; do
for sh in 1 3; do for mb in 16 24 32 48 69; do
  echo -n "shift=$sh mb=$mb "; FH_PAIR_SHIFT=$sh FH_FWD_GROUP_MB=$mb python tools/time_encode.py $cfg 20
done; done; done
