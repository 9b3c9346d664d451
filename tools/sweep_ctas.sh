#!/usr/bin/env bash
# composite fwd/bwd time vs resident CTAs per SM (persistent grid)
for k in 2 3 4 5 6 7 8 9; do
  echo "ctas_per_sm=$k"; XG_FWD_CTAS_PER_SM=$k XG_BWD_CTAS_PER_SM=$k python tools/probe.py 152 512 10 | tail -2
done
