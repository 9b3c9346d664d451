run() { echo "$1 $(env $2 timeout 600 python bench.py --no-cpu-baseline --no-train --no-c4 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['frac'],4))")"; }
run default ""
run prio "XG_BIN_PRIORITY=1"
run persistent "XG_BATCH_NONPERSISTENT=0"
run default ""
run prio "XG_BIN_PRIORITY=1"
run persistent "XG_BATCH_NONPERSISTENT=0"
