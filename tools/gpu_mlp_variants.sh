# MLP train kernel variants (FHASH_LIB): per-launch times of mlp_train_kernel at cfg4 (2^22) and cfg3 (2^18)
mkdir -p gpurun_out
for v in "$@"; do
  lib=paper_2507_03836_b200/$v
  for c in cfg4 cfg3; do
    FHASH_LIB=$PWD/$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mlp_train_kernel --csv --log-file gpurun_out/var_${v}_$c.csv python tools/time_train.py $c 12 > /dev/null 2>&1
    echo "$v $c rc=$? $(grep -h mlp_train gpurun_out/var_${v}_$c.csv | awk -F'","' '{print $NF}' | tr -d '"' | sort -n | awk '{a[NR]=$1} END {print "min", a[1], "med", a[int(NR/2)+1], "max", a[NR]}')"
  done
done
