#!/usr/bin/env bash
# Build the UNMODIFIED reference (xsplat, /root/reference/pkg) into oracle/_ref/.
#
# Test/bench infrastructure only: oracle/_ref is the CPU checker and the CPU
# baseline arm of bench.py (--impl reference, cpu_baseline kind "reference").
# It is git-ignored (never committed) but travels to the GPU box with gpurun.
# /root/reference is read-only, so the build runs from a scratch copy in /tmp;
# only the installed package lands in oracle/_ref.  The reference's own
# Cython extension (_kernels.pyx, -O3) is compiled by its own setup.py.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${XG_REFERENCE_DIR:-/root/reference/pkg}"
OUT="$HERE/_ref"
if [ ! -d "$SRC" ]; then
  echo "build_ref: $SRC absent; keeping existing $OUT" >&2
  exit 0
fi
TMP="$(mktemp -d /tmp/xg_refbuild.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$OUT"
mkdir -p "$OUT"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
  --target "$OUT" "$TMP/pkg" >/dev/null
python - "$OUT" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
from xsplat.rasterizer import available_backends
assert "compiled" in available_backends(), available_backends()
print("build_ref: xsplat built into", sys.argv[1], "backends", available_backends())
PY
# the reference's own test modules, next to the build (git-ignored, travel to
# the GPU box): tests/test_gpu_xsplat_plugin.py runs them with the "cuda"
# kernel backend registered (paper_2403_04116_b200/rasterizer/xsplat_backend.py)
rm -rf "$OUT/xsplat_tests"
cp -r "$SRC/tests" "$OUT/xsplat_tests"
echo "build_ref: reference tests copied to $OUT/xsplat_tests"
