# k_bin_emit instructions / duration, default build vs the XG_LIB_VARIANT=old tuning build
for v in old new; do
  if [ $v = old ]; then export XG_LIB_VARIANT=old; else unset XG_LIB_VARIANT; fi
  timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active -k regex:"k_bin_emit|k_bin_count" --launch-skip 24 -c 4 --csv python tools/prof_sweep_bin.py 3 2>/dev/null | grep -v "^==" | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; ix={k:i for i,k in enumerate(h)}
for r in rows[1:]:
    if len(r)==len(h) and r[ix['Metric Name']]!='': print('$v', r[ix['Kernel Name']][:24], r[ix['Metric Name']], r[ix['Metric Value']])
"
done
