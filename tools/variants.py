"""Tuning builds of libxgauss (development aid).  `python tools/variants.py
a=-DX,-DY b=-DZ` builds csrc/_variants/libxgauss_{a,b}.so; select one at
run time with XG_LIB_VARIANT=a."""
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2403_04116_b200 import _build  # noqa: E402

specs = {}
for arg in sys.argv[1:]:
    name, _, flags = arg.partition("=")
    specs[name] = [f[2:] if f.startswith("-D") else f for f in flags.split(",") if f]
with ThreadPoolExecutor(4) as ex:
    for name, path in zip(specs, ex.map(lambda kv: _build.build_variant(*kv), specs.items())):
        print(name, path)
