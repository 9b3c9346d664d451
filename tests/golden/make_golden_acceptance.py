"""The reference's own acceptance numbers (pkg/tests/test_acceptance.py:187-249),
measured in the build container: xsplat 0.1.0 (oracle/_ref, compiled backend,
one thread per run) trained on the ``gen-data`` defaults for 5,000 iterations
- N_f = 16 cuboid (the baseline), N_f = 1 cuboid, N_f = 16 random init - and
evaluated on the clean test views.  ~12 min on 3 cores:

    python tests/golden/make_golden_acceptance.py   # -> tests/golden/acceptance_ref.json
"""
import json
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1] / 'oracle' / '_ref'))
import numpy as np
from multiprocessing import Pool
def job(args):
    nf, init = args
    from xsplat.acui import CuboidSpec, init_alternative
    from xsplat.dataset import add_noise, make_projection_set
    from xsplat.geometry import ScannerConfig, equal_interval_angles
    from xsplat.phantom import default_phantom_primitives, make_phantom
    from xsplat.rasterizer import set_backend
    from xsplat.trainer import TrainConfig, train, evaluate
    set_backend("compiled")
    sc = ScannerConfig(1000.0, 1500.0, 64, 64, 3.0, equal_interval_angles(100))
    ext = np.full(3, 100.0)
    ph = make_phantom(default_phantom_primitives(tuple(ext)), (64,64,64), ext/64)
    ds = add_noise(make_projection_set(ph, sc), 0.03, 0)
    cloud = init_alternative(init, CuboidSpec((100.0,)*3, (64,)*3), nf, 0, basis_weights=np.ones(nf))
    t0 = time.time()
    res = train(ds, cloud, TrainConfig(iterations=5000))
    rep = evaluate(res.cloud, ds, ds.test_indices)
    rows = [(r["iteration"], r["test_psnr"]) for r in res.metrics if r["test_psnr"] is not None]
    return {"nf": nf, "init": init, "psnr": rep.psnr, "ssim": rep.ssim, "n": res.cloud.n_points, "s": time.time()-t0, "rows": rows}
if __name__ == "__main__":
    with Pool(3) as p:
        out = p.map(job, [(16, "cuboid"), (1, "cuboid"), (16, "random")])
    json.dump(out, open(HERE / 'acceptance_ref.json', 'w'), indent=1)
    for o in out: print(o["nf"], o["init"], o["psnr"], o["ssim"], o["n"], o["s"])
