# C2 training A/B of tuning builds: VARIANTS="a b new" bash tools/gpu_train_ab.sh
VARIANTS=${VARIANTS:-"old new"}
for rep in 1 2; do
for v in $VARIANTS; do
  if [ $v = new ]; then unset XG_LIB_VARIANT; else export XG_LIB_VARIANT=$v; fi
  echo "$v $(timeout 300 python tools/probe_train.py 1000 88 1000 2>/dev/null | tail -1)"
done
done
