# A/B of two library builds on the encode passes: tools/ab_encode.sh libA.so libB.so [cfg] (alternating runs)
c=${3:-cfg2}
for r in 1 2; do for v in $1 $2; do
  echo "$v $(FHASH_LIB=$PWD/paper_2507_03836_b200/$v timeout 300 python tools/time_encode.py $c 30 2>&1 | tail -1)"
done; done
