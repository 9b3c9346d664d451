"""Training-path parity: fused Adam, density control and the train loop
(pkg/tests/test_trainer.py ports + reference golden fixtures)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import random_arrays, small_scanner

pytestmark = pytest.mark.gpu

FIELDS = ("positions", "rotations", "log_scales", "raw_opacities", "features")


@pytest.fixture(scope="module")
def xg():
    import torch

    import paper_2403_04116_b200 as xg

    torch.cuda.set_device(0)
    return xg


@pytest.fixture(scope="module")
def tr():
    from paper_2403_04116_b200 import trainer

    return trainer


def np_(t):
    return t.detach().cpu().numpy()


def cloud_of(xg, arrs):
    return xg.GaussianCloud(**arrs, device="cuda")


def make_grads(tr, cloud, fill=0.0):
    from paper_2403_04116_b200.rasterizer.backward import make_gradients

    g = make_gradients(cloud.n_points, cloud.n_features, cloud.device)
    g.flat.fill_(fill)
    g.screen_norms.zero_()
    g.visible.fill_(True)
    return g


def uniform_lr(v):
    return {f: v for f in FIELDS}


class TestAdam:  # test_trainer.py:109-169
    def test_zero_gradient_is_identity(self, xg, tr, rng):
        cloud = cloud_of(xg, random_arrays(4, rng))
        before = np_(cloud.flat).copy()
        state = tr.OptimizerState(cloud)
        tr.adam_step(cloud, make_grads(tr, cloud), state, uniform_lr(1e-2), tr.TrainConfig())
        assert state.step == 1
        after = np_(cloud.flat)
        # rotations are renormalised (already unit): float32 rounding only
        assert np.allclose(after, before, atol=1e-7)

    def test_first_step_is_sign_step(self, xg, tr, rng):
        cloud = cloud_of(xg, random_arrays(3, rng))
        before = np_(cloud.positions).copy()
        state = tr.OptimizerState(cloud)
        g = make_grads(tr, cloud)
        g.positions[:] = torch_t([[0.5, -2.0, 3.0]] * 3)
        tr.adam_step(cloud, g, state, uniform_lr(1e-3), tr.TrainConfig())
        assert np.allclose(np_(cloud.positions), before - 1e-3 * np.sign(np_(g.positions)), atol=1e-5)

    def test_moments_accumulate(self, xg, tr, rng):
        cloud = cloud_of(xg, random_arrays(2, rng))
        state = tr.OptimizerState(cloud)
        g = make_grads(tr, cloud, 1.0)
        cfg = tr.TrainConfig()
        tr.adam_step(cloud, g, state, uniform_lr(1e-3), cfg)
        assert np.allclose(np_(state.exp_avg["features"]), 1 - cfg.beta1)
        assert np.allclose(np_(state.exp_avg_sq["features"]), 1 - cfg.beta2)
        tr.adam_step(cloud, g, state, uniform_lr(1e-3), cfg)
        assert state.step == 2
        assert np.allclose(np_(state.exp_avg["features"]), (1 - cfg.beta1) * (1 + cfg.beta1))

    def test_rotations_renormalized(self, xg, tr, rng):
        cloud = cloud_of(xg, random_arrays(3, rng))
        state = tr.OptimizerState(cloud)
        g = make_grads(tr, cloud)
        g.rotations.fill_(0.3)
        tr.adam_step(cloud, g, state, uniform_lr(5e-2), tr.TrainConfig())
        assert np.allclose(np.linalg.norm(np_(cloud.rotations), axis=1), 1.0, atol=1e-6)

    def test_nan_gradient_raises_naming_field(self, xg, tr, rng):
        cloud = cloud_of(xg, random_arrays(2, rng))
        before = np_(cloud.flat).copy()
        state = tr.OptimizerState(cloud)
        g = make_grads(tr, cloud, 0.1)
        g.log_scales[0, 0] = float("nan")
        with pytest.raises(xg.TrainingDivergenceError, match="log_scales"):
            tr.adam_step(cloud, g, state, uniform_lr(1e-3), tr.TrainConfig())
        # reference semantics: fields before log_scales updated, the rest not
        assert not np.allclose(np_(cloud.positions), before[:6].reshape(2, 3))
        assert np.array_equal(np_(cloud.log_scales).reshape(-1), before[14:20])

    def test_congruence_check(self, xg, tr, rng):
        state = tr.OptimizerState(cloud_of(xg, random_arrays(4, rng)))
        with pytest.raises(xg.InvalidParameterError):
            state.check_congruent(cloud_of(xg, random_arrays(5, rng)))

    def test_matches_reference_golden(self, xg, tr, golden):
        n, nf = (int(v) for v in golden["adam/n"])
        p0 = golden["adam/params0"]
        off = np.cumsum([0, 3 * n, 4 * n, 3 * n, n, nf * n])
        arrs = {f: p0[off[i]:off[i + 1]].reshape(n, -1) if f != "raw_opacities" else p0[off[i]:off[i + 1]]
                for i, f in enumerate(FIELDS)}
        cloud = cloud_of(xg, arrs)
        state = tr.OptimizerState(cloud)
        for s in range(3):
            g = make_grads(tr, cloud)
            g.flat.copy_(torch_t(golden[f"adam/grads{s}"]))
            tr.adam_step(cloud, g, state, dict(zip(FIELDS, golden[f"adam/lr{s}"])), tr.TrainConfig())
            ref = golden[f"adam/params{s + 1}"]
            assert np.allclose(np_(cloud.flat), ref, rtol=2e-6, atol=2e-6), s
            assert np.allclose(np_(state.m_flat), golden[f"adam/m{s + 1}"], rtol=2e-6, atol=1e-8), s


def torch_t(x):
    import torch

    return torch.as_tensor(np.asarray(x, dtype=np.float32), device="cuda")


class TestDensify:  # test_trainer.py:171-270
    def _setup(self, xg, tr):
        cloud = xg.GaussianCloud([[0.0, 0, 0], [10.0, 0, 0], [20.0, 0, 0], [30.0, 0, 0]],
                                 np.tile([1.0, 0, 0, 0], (4, 1)),
                                 np.log([[1.0] * 3, [20.0] * 3, [2.0] * 3, [2.0] * 3]),
                                 [xg.logit(0.5), xg.logit(0.5), xg.logit(0.001), xg.logit(0.5)],
                                 np.zeros((4, 2)), device="cuda")
        stats = tr.DensifyStats.zeros(4, "cuda")
        stats.norm_sum[:] = torch_t([1.0, 1.0, 0.0, 0.0])
        stats.obs_count[:] = 1
        stats.world_grad_sum[0] = torch_t([2.0, 0.0, 0.0])
        state = tr.OptimizerState(cloud)
        state.step = 7
        state.m_flat.fill_(0.5)
        cfg = tr.TrainConfig(densify_grad_threshold=0.5, prune_opacity_threshold=0.005)
        return cloud, state, stats, cfg

    def test_counts_layout_and_moments(self, xg, tr):
        cloud, state, stats, cfg = self._setup(xg, tr)
        nc, ns, rep = tr.densify_and_prune(cloud, state, stats, cfg, 5.0, np.random.default_rng(0))
        assert rep == {"pruned": 1, "cloned": 1, "split": 1, "n_points": 5}
        assert nc.n_points == 5 and ns.step == 7
        p = np_(nc.positions)
        assert np.array_equal(p[0], [0, 0, 0]) and np.array_equal(p[1], [30, 0, 0])
        assert np.allclose(p[2], [-0.5, 0, 0], atol=1e-6)
        assert np.allclose(np_(nc.log_scales)[3:5], np.log(20.0) - np.log(1.6), atol=1e-6)
        off = p[3:5] - np.array([10.0, 0, 0])
        assert np.all(np.linalg.norm(off, axis=1) > 0) and np.all(np.linalg.norm(off, axis=1) < 100)
        for f in FIELDS:
            m = np_(ns.exp_avg[f])
            assert np.all(m[:2] == 0.5) and np.all(m[2:] == 0.0), f

    def test_split_offsets_follow_parent_frame(self, xg, tr):
        cloud, state, stats, cfg = self._setup(xg, tr)
        q = np.array([np.cos(0.4), 0.0, np.sin(0.4), 0.0])
        cloud.rotations[1] = torch_t(q)
        nc, _, _ = tr.densify_and_prune(cloud, state, stats, cfg, 5.0, np.random.default_rng(123))
        local = np.random.default_rng(123).standard_normal((1, 2, 3)) * 20.0
        rot = xg.quaternions_to_rotations(np_(cloud.rotations)[1].astype(np.float64))
        expected = np.array([10.0, 0, 0]) + np.einsum("ij,kj->ki", rot, local[0])
        assert np.allclose(np_(nc.positions)[3:5], expected, atol=1e-4)

    def test_cap_skips_growth(self, xg, tr):
        cloud, state, stats, cfg = self._setup(xg, tr)
        cfg.max_points = 4
        with pytest.warns(UserWarning, match="cap"):
            nc, _, rep = tr.densify_and_prune(cloud, state, stats, cfg, 5.0, np.random.default_rng(0))
        assert rep["cloned"] == 0 and rep["split"] == 0 and nc.n_points == 3

    def test_prune_everything_raises(self, xg, tr):
        cloud, state, stats, cfg = self._setup(xg, tr)
        cloud.raw_opacities[:] = xg.logit(0.001)
        with pytest.raises(xg.XSplatError):
            tr.densify_and_prune(cloud, state, stats, cfg, 5.0, np.random.default_rng(0))

    def test_threshold_uses_average(self, xg, tr):
        cloud, state, stats, cfg = self._setup(xg, tr)
        stats.norm_sum[:] = torch_t([2.0, 0, 0, 0])
        stats.obs_count[:] = torch_t([10, 1, 1, 1]).int()
        _, _, rep = tr.densify_and_prune(cloud, state, stats, cfg, 5.0, np.random.default_rng(0))
        assert rep["cloned"] == 0 and rep["split"] == 0

    def test_matches_reference_golden(self, xg, tr, golden):
        p = "densify/"
        cloud = cloud_of(xg, {f: golden[p + f] for f in FIELDS})
        state = tr.OptimizerState(cloud)
        for f in FIELDS:
            state.exp_avg[f].copy_(torch_t(golden[p + "m_" + f]).reshape(state.exp_avg[f].shape))
            state.exp_avg_sq[f].copy_(torch_t(golden[p + "v_" + f]).reshape(state.exp_avg_sq[f].shape))
        stats = tr.DensifyStats(torch_t(golden[p + "norm_sum"]), torch_t(golden[p + "obs_count"]).int(),
                                torch_t(golden[p + "world_grad_sum"]))
        gthr, sthr, pthr, split, cap, seed = golden[p + "cfg"]
        cfg = tr.TrainConfig(densify_grad_threshold=gthr, prune_opacity_threshold=pthr, split_factor=split,
                             max_points=int(cap))
        nc, ns, rep = tr.densify_and_prune(cloud, state, stats, cfg, sthr, np.random.default_rng(int(seed)))
        assert [rep[k] for k in ("pruned", "cloned", "split", "n_points")] == list(golden[p + "report"])
        for f in FIELDS:
            assert np.allclose(np_(getattr(nc, f)), golden[p + "new_" + f], rtol=1e-6, atol=1e-5), f
            assert np.array_equal(np_(ns.exp_avg[f]), golden[p + "newm_" + f].astype(np.float32)), f


def self_render_dataset(xg, truth, scanner):
    from paper_2403_04116_b200.dataset import self_render

    return self_render(truth, scanner)


class TestTrainLoop:  # test_trainer.py:290-386
    def test_single_view_overfit(self, xg, tr, rng):
        sc = small_scanner(n_views=2)
        truth_a = random_arrays(3, rng, pos_scale=20.0, scale_range=(6.0, 12.0), opacity_range=(0.2, 0.4))
        ds = self_render_dataset(xg, cloud_of(xg, truth_a), sc)
        start = {k: v.copy() for k, v in truth_a.items()}
        start["positions"] = start["positions"] + rng.normal(scale=1.0, size=start["positions"].shape)
        start["features"] = start["features"] + rng.normal(scale=0.05, size=start["features"].shape)
        start["log_scales"] = start["log_scales"] + rng.normal(scale=0.05, size=start["log_scales"].shape)
        cfg = tr.TrainConfig(iterations=2000, gamma=0.0, densify_until_iter=0, eval_interval=2000, log_interval=500)
        res = tr.train(ds, cloud_of(xg, start), cfg)
        img, _ = xg.render_view(res.cloud, sc, float(sc.angles[0]))
        from paper_2403_04116_b200.metrics import psnr

        assert psnr(img.pixels, ds.images[0]) > 40.0

    def test_input_cloud_not_mutated(self, xg, tr, rng):
        sc = small_scanner(n_views=2)
        ds = self_render_dataset(xg, cloud_of(xg, random_arrays(3, rng)), sc)
        start = cloud_of(xg, random_arrays(4, rng))
        before = np_(start.positions).copy()
        tr.train(ds, start, tr.TrainConfig(iterations=5, gamma=0.0, densify_until_iter=0))
        assert np.array_equal(np_(start.positions), before)

    def test_metrics_rows(self, xg, tr, rng):
        sc = small_scanner(n_views=4)
        ds = self_render_dataset(xg, cloud_of(xg, random_arrays(3, rng)), sc)
        cfg = tr.TrainConfig(iterations=40, gamma=0.0, densify_until_iter=0, log_interval=10, eval_interval=20)
        res = tr.train(ds, cloud_of(xg, random_arrays(4, rng)), cfg)
        assert [r["iteration"] for r in res.metrics] == [10, 20, 30, 40]
        assert res.metrics[0]["test_psnr"] is None and res.metrics[1]["test_psnr"] is not None
        assert res.test_psnr_at(20) == res.metrics[1]["test_psnr"]
        assert all(r["n_points"] == 4 for r in res.metrics)

    def test_outputs_written(self, xg, tr, rng, tmp_path):
        sc = small_scanner(n_views=2)
        ds = self_render_dataset(xg, cloud_of(xg, random_arrays(3, rng)), sc)
        cfg = tr.TrainConfig(iterations=30, gamma=0.0, densify_until_iter=0, log_interval=10, eval_interval=30,
                             checkpoint_iterations=(10,))
        tr.train(ds, cloud_of(xg, random_arrays(4, rng)), cfg, out_dir=tmp_path / "a")
        for name in ("metrics.tsv", "cloud_final.ply", "ckpt_000010.ply"):
            assert (tmp_path / "a" / name).exists(), name
        from paper_2403_04116_b200.cloudio import load_cloud

        c = load_cloud(tmp_path / "a" / "cloud_final.ply", device="cuda")
        assert c.n_points == 4

    def test_densification_grows_cloud(self, xg, tr, rng):
        sc = small_scanner(32, 32, 6.0, n_views=4)
        ds = self_render_dataset(xg, cloud_of(xg, random_arrays(8, rng, pos_scale=30.0, scale_range=(8.0, 15.0))), sc)
        cfg = tr.TrainConfig(iterations=60, gamma=0.0, densify_from_iter=10, densify_interval=20,
                             densify_until_iter=60, densify_grad_threshold=1e-9, log_interval=60)
        res = tr.train(ds, cloud_of(xg, random_arrays(6, rng, pos_scale=30.0)), cfg)
        assert res.cloud.n_points > 6

    def test_logged_loss_on_density_control_steps(self, xg, tr, rng):
        """A row logged at a density-control iteration reports that step's
        loss (the fused L1 of the frame it rendered, not the resized one's);
        reproducible mode computes it by an in-order reduction - both agree."""
        sc = small_scanner(32, 32, 6.0, n_views=4)
        ds = self_render_dataset(xg, cloud_of(xg, random_arrays(8, rng, pos_scale=30.0, scale_range=(8.0, 15.0))), sc)
        start = random_arrays(6, rng, pos_scale=30.0)
        cfg = tr.TrainConfig(iterations=40, gamma=0.0, densify_from_iter=5, densify_interval=10,
                             densify_until_iter=40, densify_grad_threshold=1e-9, log_interval=10)
        a = tr.train(ds, cloud_of(xg, start), cfg)
        b = tr.train(ds, cloud_of(xg, start), cfg, reproducible=True)
        for ra, rb in zip(a.metrics, b.metrics):
            assert ra["loss"] > 0 and rb["loss"] > 0, (ra, rb)
        assert abs(a.metrics[0]["loss"] / b.metrics[0]["loss"] - 1) < 1e-5

    def test_gamma_ssim_path_runs(self, xg, tr, rng):
        sc = small_scanner(n_views=2)
        ds = self_render_dataset(xg, cloud_of(xg, random_arrays(3, rng)), sc)
        res = tr.train(ds, cloud_of(xg, random_arrays(3, rng)),
                       tr.TrainConfig(iterations=20, gamma=0.2, densify_until_iter=0, log_interval=10))
        assert np.isfinite(res.metrics[-1]["loss"])

    def test_evaluate_ground_truth(self, xg, tr, rng):
        sc = small_scanner(n_views=2)
        truth = cloud_of(xg, random_arrays(3, rng))
        ds = self_render_dataset(xg, truth, sc)
        rep = tr.evaluate(truth, ds, np.array([0, 1]))
        assert rep.psnr > 120.0 and rep.ssim > 0.999999


class TestForwardBeforeCounterRead:
    """The trainer queues the forward before it reads the binning counters;
    after an entry-buffer overflow the forward skipped itself on the device,
    the view is re-binned and the forward re-run - the step equals one with
    ample capacity."""

    def test_overflow_step_matches(self, xg, tr, rng):
        import torch

        sc = small_scanner(32, 32, 6.0, n_views=4)
        ds = self_render_dataset(xg, cloud_of(xg, random_arrays(8, rng, pos_scale=30.0, scale_range=(8.0, 15.0))), sc)
        start = random_arrays(6, rng, pos_scale=30.0, scale_range=(8.0, 15.0))
        cfg = tr.TrainConfig(iterations=10, gamma=0.0, densify_until_iter=0, log_interval=10**6,
                             eval_interval=10**6)
        a = tr.Trainer(ds, cloud_of(xg, start), cfg)
        b = tr.Trainer(ds, cloud_of(xg, start), cfg)
        fr = b.eng.frame
        for t in (a, b):
            t.step()
        # shrink b's entry buffer below what a view needs: the next step overflows
        fr.entry_capacity = 4
        fr.entry_splat = torch.empty(4, dtype=torch.int32, device="cuda")
        for t in (a, b):
            t.step()
        assert fr.entry_capacity > 4  # the overflow was seen and the view re-binned
        torch.cuda.synchronize()
        assert np.allclose(np_(a.cloud.flat), np_(b.cloud.flat), rtol=1e-5, atol=1e-7)


class TestHostTargets:
    def test_prefetched_targets_match_device_targets(self, xg, tr, rng):
        """targets_on_host (the e2e mode: pinned host targets, the next view's
        copied on a side stream during the step) trains exactly like
        HBM-resident targets."""
        import torch

        sc = small_scanner(32, 32, 6.0, n_views=6)
        ds = self_render_dataset(xg, cloud_of(xg, random_arrays(8, rng, pos_scale=30.0, scale_range=(8.0, 15.0))), sc)
        start = random_arrays(6, rng, pos_scale=30.0, scale_range=(8.0, 15.0))
        cfg = tr.TrainConfig(iterations=40, gamma=0.0, densify_until_iter=0, log_interval=10**6,
                             eval_interval=10**6)
        a = tr.Trainer(ds, cloud_of(xg, start), cfg)
        b = tr.Trainer(ds, cloud_of(xg, start), cfg, targets_on_host=True)
        for _ in range(40):
            a.step()
            b.step()
        torch.cuda.synchronize()
        assert np.allclose(np_(a.cloud.flat), np_(b.cloud.flat), rtol=1e-5, atol=1e-7)


class TestDataParallelSingleRank:
    """The data-parallel step (bucketed reduce + range Adam + renorm) on one
    rank must reproduce the single-GPU Trainer exactly (same views, same
    kernels, no collective)."""

    def test_matches_trainer(self, xg, tr, rng):
        from paper_2403_04116_b200.parallel import DataParallelTrainer

        sc = small_scanner(32, 32, 6.0, n_views=4)
        ds = self_render_dataset(xg, cloud_of(xg, random_arrays(8, rng, pos_scale=30.0, scale_range=(8.0, 15.0))), sc)
        start = random_arrays(6, rng, pos_scale=30.0)
        cfg = tr.TrainConfig(iterations=30, gamma=0.0, densify_from_iter=5, densify_interval=10,
                             densify_until_iter=30, densify_grad_threshold=1e-9, log_interval=10**6,
                             eval_interval=10**6)
        a = tr.Trainer(ds, cloud_of(xg, start), cfg)
        b = DataParallelTrainer(ds, cloud_of(xg, start), cfg, bucket_bytes=4 * 37)
        for _ in range(30):
            a.step()
            b.step()
        assert a.cloud.n_points == b.cloud.n_points > 6
        # identical up to the summation order of the backward's float atomics
        assert np.allclose(np_(a.cloud.flat), np_(b.cloud.flat), rtol=1e-4, atol=1e-6)
