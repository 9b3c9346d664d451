# C3 sweep: compositing footprint vs binning overlap
run() { echo "$1 $(env $2 timeout 600 python bench.py --no-cpu-baseline --no-train --no-c4 $3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['frac'],4), round(d['roofline']['kernel_ms_in_timed_region'],3))")"; }
run default "" ""
run p3 "XG_BATCH_NONPERSISTENT=0 XG_FWD_CTAS_PER_SM=3" ""
run p3prio "XG_BATCH_NONPERSISTENT=0 XG_FWD_CTAS_PER_SM=3 XG_BIN_PRIORITY=1" ""
run p2prio "XG_BATCH_NONPERSISTENT=0 XG_FWD_CTAS_PER_SM=2 XG_BIN_PRIORITY=1" ""
run p4 "XG_BATCH_NONPERSISTENT=0 XG_FWD_CTAS_PER_SM=4" ""
run prio "XG_BIN_PRIORITY=1" ""
run b16 "" "--batch 16"
run b4 "" "--batch 4"
run default "" ""
