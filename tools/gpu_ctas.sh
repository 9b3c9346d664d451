for c in 4 3 2; do echo "== fwd ctas/sm $c"; XG_FWD_CTAS_PER_SM=$c timeout 300 python tools/probe.py 152 512 10 2>&1 | tail -2 | head -1; done
for c in 4 3 2; do echo "== bwd ctas/sm $c"; XG_BWD_CTAS_PER_SM=$c timeout 300 python tools/probe.py 152 512 10 2>&1 | tail -1; done
