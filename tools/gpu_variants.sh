# time the compositing kernels of each tuning build (tools/variants.py)
for v in ${VARIANTS:-base}; do
  echo "== $v"; XG_LIB_VARIANT=$v timeout 300 python tools/probe.py 152 512 20 2>&1 | tail -2
done
