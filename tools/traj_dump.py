"""Dump the engine's training rows next to the reference's (tests/golden/train.npz)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2403_04116_b200 as xg  # noqa: E402
from paper_2403_04116_b200.dataset import ProjectionSet  # noqa: E402
from paper_2403_04116_b200.trainer import TrainConfig, train  # noqa: E402

fx = dict(np.load("tests/golden/train.npz"))
FIELDS = ("positions", "rotations", "log_scales", "raw_opacities", "features")
case = sys.argv[1] if len(sys.argv) > 1 else "ssim_reset"
l_so, l_sd, w, h, pitch, n = fx["scanner"]
sc = xg.ScannerConfig(l_so, l_sd, int(w), int(h), pitch, xg.equal_interval_angles(int(n)))
ds = ProjectionSet(fx["images"], fx["clean_images"], sc, fx["train_indices"], fx["test_indices"])
cloud = xg.GaussianCloud(**{k: fx["init/" + k] for k in FIELDS}, device="cuda")
gamma, reset = fx[case + "/cfg"]
cfg = TrainConfig(iterations=300, densify_from_iter=100, densify_interval=100, densify_until_iter=300,
                  log_interval=10, eval_interval=100, gamma=float(gamma), opacity_reset_interval=int(reset))
res = train(ds, cloud, cfg)
for row, r in zip(res.metrics, fx[case + "/rows"]):
    print(f"{row['iteration']:4d} loss {row['loss']:.6f} ref {r[1]:.6f} ({row['loss'] / r[1] - 1:+.4f})  "
          f"tpsnr {row['train_psnr']:.3f} ref {r[2]:.3f}  N {row['n_points']} {int(r[5])}  "
          f"test {row['test_psnr']} ref {r[3]:.3f}")
