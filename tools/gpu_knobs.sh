# C2 knob A/B: per-kernel times (ncu launch lists inside the timed window) and iteration times
for v in base pb4 bal296 bal592; do
  vv=$v; [ $v = base ] && vv=""
  XG_LIB_VARIANT=$vv timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/knob_$v.csv python tools/probe_train.py 5 88 1000 > /dev/null 2>&1
  echo "== $v"; python tools/launch_summary.py gpurun_out/knob_$v.csv 5 | grep -E "preprocess_bwd|bin_emit_bal|bin_count_bal|k_scan|total"
done
for v in base pb4 base pb4; do
  vv=$v; [ $v = base ] && vv=""
  echo -n "$v "; XG_LIB_VARIANT=$vv timeout 300 python tools/probe_train.py 2000 88 1000 2>&1 | tail -1
done
