for mode in bucket onesweep; do
  if [ $mode = onesweep ]; then export XG_DEPTH_SORT=onesweep; else unset XG_DEPTH_SORT; fi
  ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/bin_$mode.csv python tools/prof_c3.py 1 > /dev/null 2>&1
  echo "== $mode (C3 single view, serialized)"; python tools/launch_summary.py gpurun_out/bin_$mode.csv | grep -E "k_bs|k_os|k_iota|k_scan|k_bin|k_preprocess\(|total"
  python tools/probe_train.py 200 88 1000 | tail -1
done
