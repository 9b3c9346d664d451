for v in ${VARIANTS:-base}; do echo "== $v"; XG_LIB_VARIANT=$v timeout 300 python tools/probe.py 152 512 10 2>&1 | tail -2 | head -1; done
VARIANTS="${VARIANTS}" bash tools/gpu_c4_variants.sh
