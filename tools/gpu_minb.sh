cd /root/repo
for lib in libfhash_minb4 libfhash_minb5 libfhash_minb6; do for cfg in cfg2 cfg3 cfg4 pc; do FHASH_LIB=paper_2507_03836_b200/$lib.so python tools/time_encode.py $cfg 20; done; done
