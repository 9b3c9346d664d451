"""SSIM / PSNR / loss on the GPU (xg_ssim kernel) against golden vectors of
the real reference (tests/golden/make_golden_metrics.py: xsplat
metrics.py:36-124, trainer.py:109-123), plus ports of the reference's
test_metrics.py known-answer tests."""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden" / "metrics.npz"


@pytest.fixture(scope="module")
def gold():
    d = np.load(GOLD, allow_pickle=False)
    return {k: d[k] for k in d.files}


@pytest.fixture(scope="module")
def m():
    import torch

    from paper_2403_04116_b200 import metrics

    torch.cuda.set_device(0)
    return metrics


def _cases(gold):
    return [str(c) for c in gold["cases"]]


@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_ssim_value_and_gradient_match_reference(gold, m, dtype):
    import torch

    for c in _cases(gold):
        p = c + "/"
        dt = getattr(torch, dtype)
        a = torch.as_tensor(gold[p + "pred"], device="cuda").to(dt)
        b = torch.as_tensor(gold[p + "ref"], device="cuda").to(dt)
        dr = float(gold[p + "data_range"])
        if min(a.shape) < 11:
            continue
        s = m.ssim(a, b, data_range=dr)
        assert abs(s - float(gold[p + "ssim"])) < 1e-12, (c, s, float(gold[p + "ssim"]))
        s2, g = m.ssim_and_gradient(a, b, data_range=dr)
        assert s2 == s
        want = gold[p + "ssim_grad"]
        # (the gradient of identical images is pure roundoff: floor the scale
        # at the per-window weight 1 / n_windows)
        scale = max(np.abs(want).max(), 1.0 / want.size)
        assert np.abs(g.cpu().numpy() - want).max() <= 1e-10 * scale, c


def test_psnr_matches_reference(gold, m):
    for c in _cases(gold):
        p = c + "/"
        v = m.psnr(gold[p + "pred"].astype(np.float64), gold[p + "ref"].astype(np.float64),
                   data_range=float(gold[p + "data_range"]))
        want = float(gold[p + "psnr"])
        assert (v == want) if np.isinf(want) else abs(v - want) < 1e-9, c


def test_loss_matches_reference(gold):
    from paper_2403_04116_b200.trainer import loss

    for c in _cases(gold):
        p = c + "/"
        for gamma in (0.0, 0.2, 1.0):
            k = p + f"loss_{gamma}"
            if k not in gold or min(gold[p + "pred"].shape) < 11:
                continue
            v, dl = loss(gold[p + "pred"], gold[p + "ref"], gamma)
            assert abs(v - float(gold[k])) < 1e-12, (c, gamma)
            want = gold[p + f"loss_grad_{gamma}"]
            scale = max(np.abs(want).max(), 1.0 / want.size)
            assert np.abs(dl.cpu().numpy() - want).max() <= 1e-10 * scale, (c, gamma)


def test_fused_training_gradient(gold, m):
    """The float32 dl the trainer feeds the backward: -gamma dSSIM + (1 -
    gamma) sign / HW in one launch."""
    import torch

    c = "noise64/"
    a = torch.as_tensor(gold[c + "pred"], device="cuda")
    b = torch.as_tensor(gold[c + "ref"], device="cuda")
    eng = m.SsimEngine(64, 64, a.device)
    dl = torch.empty((64, 64), dtype=torch.float32, device="cuda")
    eng.run(a, b, 1.0, dl=dl, dl_ssim_scale=-0.2, dl_l1_scale=0.8 / 4096)
    want = gold[c + "loss_grad_0.2"]
    assert np.abs(dl.cpu().numpy().astype(np.float64) - want).max() <= 1e-6 * np.abs(want).max()


class TestReferencePorts:
    """test_metrics.py:104-160 of the reference."""

    def test_identical_is_one(self, m, rng):
        a = rng.uniform(size=(16, 16))
        assert m.ssim(a, a) == pytest.approx(1.0, abs=1e-12)

    def test_negative_image_less_than_one(self, m, rng):
        a = rng.uniform(0.1, 0.9, size=(16, 16))
        assert m.ssim(a, 1.0 - a) < 1.0

    def test_symmetric(self, m, rng):
        a, b = rng.uniform(size=(20, 20)), rng.uniform(size=(20, 20))
        assert m.ssim(a, b) == pytest.approx(m.ssim(b, a), abs=1e-12)

    def test_too_small_raises(self, m):
        from paper_2403_04116_b200.errors import InvalidParameterError

        with pytest.raises(InvalidParameterError):
            m.ssim(np.zeros((10, 10)), np.zeros((10, 10)))

    def test_shape_mismatch(self, m):
        from paper_2403_04116_b200.errors import InvalidParameterError

        with pytest.raises(InvalidParameterError):
            m.ssim(np.zeros((16, 16)), np.zeros((16, 17)))

    def test_scale_invariance_with_data_range(self, m, rng):
        a = rng.uniform(size=(16, 16))
        b = rng.uniform(size=(16, 16))
        assert m.ssim(10 * a, 10 * b, data_range=10.0) == pytest.approx(m.ssim(a, b), rel=1e-12)

    def test_gradient_matches_finite_differences(self, m, rng):
        a = rng.uniform(0.2, 0.8, size=(14, 14))
        b = np.clip(a + rng.normal(scale=0.05, size=(14, 14)), 0, 1)
        _, grad = m.ssim_and_gradient(a, b)
        grad = grad.cpu().numpy()
        eps = 1e-6
        for i in (0, 3, 7, 13):
            for j in (0, 6, 13):
                bump = np.zeros_like(a)
                bump[i, j] = eps
                fd = (m.ssim(a + bump, b) - m.ssim(a - bump, b)) / (2 * eps)
                assert grad[i, j] == pytest.approx(fd, rel=1e-5, abs=1e-9)

    def test_zero_at_identity(self, m, rng):
        a = rng.uniform(0.2, 0.8, size=(16, 16))
        _, grad = m.ssim_and_gradient(a, a)
        assert np.allclose(grad.cpu().numpy(), 0.0, atol=1e-12)


def test_stack_matches_per_view(m, rng):
    """evaluate()'s batched path: one launch per view, one sync - same
    numbers as per-view ssim() / psnr()."""
    import torch

    a = torch.as_tensor(rng.uniform(size=(5, 40, 52)), dtype=torch.float32, device="cuda")
    b = torch.clamp(a + 0.05 * torch.randn_like(a), 0, 1)
    b[2] = a[2]
    s, p = m.ssim_psnr_stack(a, b)
    for v in range(5):
        assert s[v] == m.ssim(a[v], b[v])
        assert p[v] == m.psnr(a[v], b[v]) or (np.isinf(p[v]) and np.isinf(m.psnr(a[v], b[v])))
