# C4 binning chunk count at T = 4096
for v in base bc444 bc592 bc148 base; do
  if [ $v = base ]; then unset XG_LIB_VARIANT; else export XG_LIB_VARIANT=$v; fi
  echo "$v $(timeout 300 python tools/probe.py 196 1024 8 2>&1 | grep 'per view')"
done
