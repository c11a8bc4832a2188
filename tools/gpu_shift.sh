cd /root/repo
for cfg in cfg2 cfg3 cfg4 pc; do
 echo "== $cfg xor-hash, no shift (old)"; FHASH_LIB=paper_2507_03836_b200/libfhash_xor.so FH_PAIR_SHIFT=0 python tools/time_encode.py $cfg 20
 echo "== $cfg xadd, no shift"; FH_PAIR_SHIFT=0 python tools/time_encode.py $cfg 20
 echo "== $cfg xadd + shift"; FH_PAIR_SHIFT=1 python tools/time_encode.py $cfg 20
done
