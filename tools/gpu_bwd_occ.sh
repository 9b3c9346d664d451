# reverse replay occupancy / sub-block variants: C2 iteration time
for v in base ck5 ck6 bp2 bp2c5 bp2c6 base; do
  if [ $v = base ]; then unset XG_LIB_VARIANT; else export XG_LIB_VARIANT=$v; fi
  echo "$v $(timeout 600 python tools/probe_train.py 400 2>&1 | tail -1)"
done
