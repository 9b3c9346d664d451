"""The GPU training loop against the REAL reference's ``train``
(tests/golden/train.npz, make_golden_train.py): 300 iterations from the same
float32 ACUI cloud on the same float32 targets, through two density-control
events, for the default L1 objective and for gamma = 0.2 with an opacity
reset.  Logged rows (every 10 iterations: loss, train PSNR, held-out PSNR /
SSIM every 100, N) are compared one by one.

Tolerances: the engine keeps the parameters in float32 (the reference:
float64) and sums gradients with float atomics, so the two runs agree to
rounding (measured: loss within 2e-4 relative, PSNR within 0.01 dB) - until
a density-control event at which a Gaussian whose averaged screen-gradient
norm sits within that rounding of the 2e-5 threshold is cloned on one side
only.  From there the layouts differ and, because the split offsets are the
next rng.standard_normal((n_split, 2, 3)) draws, so does every later split
child: the runs become different random processes.  So rows are compared
strictly (loss 5e-3 relative, PSNR 0.05 dB, SSIM 2e-3) up to the first event
whose N differs (held-out metrics, evaluated after each row's event, up to
iteration 200), and that event's N must be within 0.5 % of the reference's; the L1 run must keep the reference's N through its first event
(measured: exactly, 1,593).  Runs use ``reproducible=True``, so the
outcome is fixed.  The
iteration-250 checkpoint (L1 run) is compared per Gaussian: median and 90th
percentile of |delta| per field.""" 

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TRAIN = Path(__file__).resolve().parent / "golden" / "train.npz"
FIELDS = ("positions", "rotations", "log_scales", "raw_opacities", "features")


@pytest.fixture(scope="module")
def fx():
    d = np.load(TRAIN)
    return {k: d[k] for k in d.files}


@pytest.mark.parametrize("case", ["l1", "ssim_reset"])
def test_trajectory_matches_reference(fx, case):
    import torch

    import paper_2403_04116_b200 as xg
    from paper_2403_04116_b200.dataset import ProjectionSet
    from paper_2403_04116_b200.trainer import TrainConfig, train

    torch.cuda.set_device(0)
    l_so, l_sd, w, h, pitch, n = fx["scanner"]
    sc = xg.ScannerConfig(l_so, l_sd, int(w), int(h), pitch, xg.equal_interval_angles(int(n)))
    ds = ProjectionSet(fx["images"], fx["clean_images"], sc, fx["train_indices"], fx["test_indices"])
    cloud = xg.GaussianCloud(**{k: fx["init/" + k] for k in FIELDS}, device="cuda")
    gamma, reset = fx[case + "/cfg"]
    cfg = TrainConfig(iterations=300, densify_from_iter=100, densify_interval=100, densify_until_iter=300,
                      log_interval=10, eval_interval=100, gamma=float(gamma), opacity_reset_interval=int(reset))
    cfg.checkpoint_iterations = (250,)
    import tempfile

    from paper_2403_04116_b200.cloudio import load_cloud

    with tempfile.TemporaryDirectory() as tmp:
        res = train(ds, cloud, cfg, out_dir=tmp, reproducible=True)  # (fixed-order sums: a fixed outcome)
        ck = load_cloud(Path(tmp) / "ckpt_000250.ply")
    ref = fx[case + "/rows"]
    assert len(res.metrics) == ref.shape[0]
    worst = {"loss": 0.0, "train_psnr": 0.0, "test_psnr": 0.0, "test_ssim": 0.0}
    diverged_at = None
    for row, r in zip(res.metrics, ref):
        it, loss, tpsnr, vpsnr, vssim, npts = r
        assert row["iteration"] == int(it)
        if row["n_points"] != int(npts):  # a density-control decision differed at this row's event
            assert abs(row["n_points"] - npts) <= 5e-3 * npts, (case, int(it), row["n_points"], int(npts))
            diverged_at = int(it)
        # loss / train PSNR of this row's view were computed before this row's event
        worst["loss"] = max(worst["loss"], abs(row["loss"] / loss - 1))
        worst["train_psnr"] = max(worst["train_psnr"], abs(row["train_psnr"] - tpsnr))
        if diverged_at is not None:
            break
        if not np.isnan(vpsnr):
            if it < 300:
                worst["test_psnr"] = max(worst["test_psnr"], abs(row["test_psnr"] - vpsnr))
                worst["test_ssim"] = max(worst["test_ssim"], abs(row["test_ssim"] - vssim))
            else:
                # held-out evaluation after the last event: even with equal N the
                # two sides may have cloned / split different members (measured
                # 0.73 dB apart)
                assert abs(row["test_psnr"] - vpsnr) < 1.5, (case, row["test_psnr"], vpsnr)
    print(f"\n[{case}] strict agreement through iteration {diverged_at or 300}: worst deviation {worst}")
    assert worst["loss"] < 5e-3 and worst["train_psnr"] < 0.05, worst
    assert worst["test_psnr"] < 0.05 and worst["test_ssim"] < 2e-3, worst
    if case == "l1":
        assert diverged_at is None or diverged_at >= 300, diverged_at
    if diverged_at is not None and diverged_at <= 250:
        return  # the checkpoint lies after the runs parted
    ck = {k: np.asarray(getattr(ck, k).cpu() if hasattr(getattr(ck, k), "cpu") else getattr(ck, k), np.float64)
          for k in FIELDS}
    # per-Gaussian max |delta|: Gaussians with near-zero gradients (most of
    # them children born at iteration 200 with zeroed moments, where Adam's
    # normalised step turns rounding-level gradient differences into
    # full-lr steps) carry the tail; the bulk follows the reference closely
    q = {}
    for k in FIELDS:
        e = np.abs(ck[k] - fx[f"{case}/ckpt250_{k}"]).reshape(ck[k].shape[0], -1).max(1)
        q[k] = np.quantile(e, [0.5, 0.9])
    print(f"[{case}] checkpoint @250 ({ck['positions'].shape[0]} Gaussians), per-field |delta| median / p90: "
          + ", ".join(f"{k} {v[0]:.2e} / {v[1]:.2e}" for k, v in q.items()))
    assert q["positions"][0] < 1e-3 and q["positions"][1] < 0.05, q
    for k in ("log_scales", "raw_opacities", "features"):
        assert q[k][0] < 5e-3 and q[k][1] < 5e-2, (k, q[k])
