"""Data-parallel training at world size 2 on the GPU: two
processes share cuda:0 over gloo (the collective is the only difference from
the NCCL node; the kernels, buckets and Adam epilogues are the product's).

* the all-reduced gradient of one DP step equals the sum of the two ranks'
  single-view gradients, and that sum equals the CPU oracle's per-view
  float64 gradients (fused L1, backward.py:21-124) summed, normwise 1e-4;
* after 30 DP steps spanning density-control events (the stats summed over
  ranks, split normals from the same PCG64 stream on both ranks) the two
  replicas hold bit-identical clouds and Adam moments;
* gamma > 0 (L1 + SSIM) and opacity resets run through the same DP step;
* the peer-memory exchange (collective="p2p", csrc/xg_dp.cu) gives the same
  bit-identical replicas as the bucketed all-reduce.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, body, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, body(rank, world)))
    except Exception as e:  # surface the failure in the parent
        q.put((rank, {"error": repr(e)}))
        raise
    finally:
        dist.destroy_process_group()


def spawn(body, world=2):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, body, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    for r in range(world):
        assert not (isinstance(out[r], dict) and "error" in out[r]), out[r]
    return out


def _scene():
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from conftest import random_arrays, small_scanner

    rng = np.random.default_rng(77)
    truth = random_arrays(10, rng, pos_scale=30.0, scale_range=(6.0, 12.0))
    start = random_arrays(8, rng, pos_scale=30.0, scale_range=(6.0, 12.0))
    return truth, start, small_scanner(32, 32, 6.0, n_views=8)


def _dataset(truth, sc):
    import paper_2403_04116_b200 as xg
    from paper_2403_04116_b200.dataset import self_render

    return self_render(xg.GaussianCloud(**truth, device="cuda"), sc)


def _grad_sum_body(rank, world):
    import torch

    import paper_2403_04116_b200 as xg
    from paper_2403_04116_b200.parallel import DataParallelTrainer, dp_views

    truth, start, sc = _scene()
    ds = _dataset(truth, sc)
    cfg = xg.trainer.TrainConfig(iterations=10, densify_until_iter=0, log_interval=10**6, eval_interval=10**6)
    dp = DataParallelTrainer(ds, xg.GaussianCloud(**start, device="cuda"), cfg)
    views = dp_views(list(dp.order), ds.train_indices, np.random.default_rng(cfg.rng_seed), world)
    # each view's gradient alone, through the same (single-view) phases
    per_view = []
    for v in views:
        dp.it = 1
        dp._render_and_backward(v, 0)
        per_view.append(dp.eng.grads.flat.clone())
    dp.it = 0
    # one DP step: this rank renders views[rank]; capture the gradient the
    # reducer delivers to the Adam epilogues
    captured = {}
    orig = dp._reducer_for

    def spy(numel):
        red = orig(numel)

        class Wrapped:
            numel = red.numel

            def __call__(self, flat, epilogue=None):
                red(flat, epilogue)
                captured["g"] = flat.clone()
        return Wrapped()

    dp._reducer_for = spy
    dp.step()
    torch.cuda.synchronize()
    return {"views": views, "reduced": captured["g"].cpu().numpy(),
            "per_view": [g.cpu().numpy() for g in per_view]}


def test_allreduced_gradient_is_sum_of_view_gradients():
    out = spawn(_grad_sum_body)
    from conftest import normwise_ok
    from oracle import oracle as orc
    from paper_2403_04116_b200.geometry import extrinsic_from_angle

    a, b = out[0], out[1]
    assert a["views"] == b["views"] and a["views"][0] != a["views"][1]
    assert np.array_equal(a["reduced"], b["reduced"])  # both ranks hold the same sum
    s = a["per_view"][0] + a["per_view"][1]
    ok, rel = normwise_ok(a["reduced"], s, 0.0, tol=1e-5)
    assert ok, rel
    # against the oracle: sum over the two views of the float64 per-view
    # gradients of the fused L1 objective
    truth, start, sc = _scene()
    import paper_2403_04116_b200 as xg
    import torch

    torch.cuda.set_device(0)
    ds = _dataset(truth, sc)
    total = None
    fields = {k: np.asarray(v, np.float32) for k, v in start.items()}
    basis = np.ones(fields["features"].shape[1], np.float32)
    for v in a["views"]:
        phi = float(ds.angles[v])
        cam = orc.camera_from_view(1000.0, 1500.0, 32, 32, 6.0, phi)
        pre = orc.preprocess(fields, basis, cam)
        binned = orc.bin_entries(pre, cam)
        img = orc.composite_fwd(pre, binned, 32, 32)["image"].astype(np.float64)
        _, dl = orc.l1_loss(img, np.asarray(ds.images[v], np.float64))
        g = orc.preprocess_bwd(fields, basis, cam, pre, orc.composite_bwd(pre, binned, 32, 32, dl))
        flat = np.concatenate([g[f].reshape(-1) for f in orc.PARAM_FIELDS])
        total = flat if total is None else total + flat
    del extrinsic_from_angle, xg
    n = start["positions"].shape[0]
    off = 0
    for f, wdt in zip(orc.PARAM_FIELDS, (3, 4, 3, 1, fields["features"].shape[1])):
        seg = slice(off, off + n * wdt)
        floor = 1e-3 * np.abs(total).max()
        ok, rel = normwise_ok(a["reduced"][seg], total[seg], floor)
        assert ok, (f, rel)
        off += n * wdt


def _replica_body(rank, world, gamma=0.0, reset=0, collective="nccl", reproducible=False):
    import torch

    import paper_2403_04116_b200 as xg
    from paper_2403_04116_b200.parallel import DataParallelTrainer

    truth, start, sc = _scene()
    ds = _dataset(truth, sc)
    cfg = xg.trainer.TrainConfig(iterations=30, gamma=gamma, densify_from_iter=5, densify_interval=10,
                                 densify_until_iter=30, densify_grad_threshold=1e-9, log_interval=10,
                                 eval_interval=10**6, opacity_reset_interval=reset)
    dp = DataParallelTrainer(ds, xg.GaussianCloud(**start, device="cuda"), cfg, bucket_bytes=4 * 37,
                             collective=collective, reproducible=reproducible)
    for _ in range(30):
        dp.step()
    torch.cuda.synchronize()
    return {"flat": dp.cloud.flat.cpu().numpy(), "m": dp.state.m_flat.cpu().numpy(),
            "v": dp.state.v_flat.cpu().numpy(), "events": dp.densify_events, "n": dp.cloud.n_points,
            "loss": [r["loss"] for r in dp.metrics]}


def test_replicas_bit_identical_across_densify():
    out = spawn(_replica_body)
    a, b = out[0], out[1]
    assert a["events"] == b["events"] >= 2 and a["n"] == b["n"] > 8
    for k in ("flat", "m", "v"):
        assert np.array_equal(a[k], b[k]), k
    # each rank logs its own view's loss: the two ranks trained on different views
    assert a["loss"] != b["loss"]


def _peer_body(rank, world):
    # (reproducible backward: the two runs' per-view gradients are then
    # bit-identical, so the two collectives see the same operands)
    return {c: _replica_body(rank, world, collective=c, reproducible=True) for c in ("nccl", "p2p")}


def test_peer_exchange_matches_allreduce_path():
    """The peer-memory step (PeerExchange: IPC-mapped buffers, reduce-scatter
    + all-gather-Adam kernels with device-side epoch waits) across density
    control: replicas bit-identical, and equal to the bucketed all-reduce
    path (at world 2 both add the same two gradients)."""
    out = spawn(_peer_body)
    a, b = out[0], out[1]
    assert a["p2p"]["events"] == a["nccl"]["events"] >= 2 and a["p2p"]["n"] == a["nccl"]["n"]
    for k in ("flat", "m", "v"):
        assert np.array_equal(a["p2p"][k], b["p2p"][k]), k
        assert np.array_equal(a["p2p"][k], a["nccl"][k]), k


def _replica_ssim_reset_body(rank, world):
    return _replica_body(rank, world, gamma=0.2, reset=12)


def test_replicas_bit_identical_ssim_and_opacity_reset():
    out = spawn(_replica_ssim_reset_body)
    a, b = out[0], out[1]
    for k in ("flat", "m", "v"):
        assert np.array_equal(a[k], b[k]), k


def _sharded_sweep_body(rank, world):
    import torch

    import paper_2403_04116_b200 as xg
    from paper_2403_04116_b200.parallel import render_sweep_sharded

    truth, start, sc = _scene()
    cloud = xg.GaussianCloud(**truth, device="cuda")
    angles = np.linspace(0.0, np.pi, 29, endpoint=False)
    full = render_sweep_sharded(cloud, sc, angles, gather=True, batch=4)
    torch.cuda.synchronize()
    return None if full is None else full.cpu().numpy()


def test_sharded_sweep_gathers_the_single_process_stack():
    """View-sharded inference (the C3 multi-GPU mode): each rank renders its
    round-robin share through the batched renderer; the stack gathered on
    rank 0 equals one process rendering every view (same kernels, bit for
    bit)."""
    out = spawn(_sharded_sweep_body)
    assert out[1] is None
    import torch

    import paper_2403_04116_b200 as xg
    from paper_2403_04116_b200.inference import SweepRenderer

    torch.cuda.set_device(0)
    truth, start, sc = _scene()
    cloud = xg.GaussianCloud(**truth, device="cuda")
    angles = np.linspace(0.0, np.pi, 29, endpoint=False)
    ref = SweepRenderer(cloud, sc, batch=4).render(angles).cpu().numpy()
    assert out[0].shape == ref.shape and np.array_equal(out[0], ref)


def test_peer_exchange_single_process_equals_trainer():
    """world = 1 (no process group): the peer-exchange kernels with one rank
    apply exactly the single-GPU Trainer's Adam (reproducible backward, so
    both see the same gradients) - 20 steps including a density event."""
    import torch

    import paper_2403_04116_b200 as xg
    from paper_2403_04116_b200.parallel import DataParallelTrainer

    torch.cuda.set_device(0)
    truth, start, sc = _scene()
    ds = _dataset(truth, sc)

    def cfg():
        return xg.trainer.TrainConfig(iterations=20, densify_from_iter=5, densify_interval=10, densify_until_iter=20,
                                      densify_grad_threshold=1e-9, log_interval=10**6, eval_interval=10**6)

    a = xg.trainer.Trainer(ds, xg.GaussianCloud(**start, device="cuda"), cfg(), reproducible=True)
    b = DataParallelTrainer(ds, xg.GaussianCloud(**start, device="cuda"), cfg(), reproducible=True, collective="p2p")
    for _ in range(20):
        a.step()
        b.step()
    torch.cuda.synchronize()
    assert a.densify_events == b.densify_events >= 1
    for x, y in ((a.cloud.flat, b.cloud.flat), (a.state.m_flat, b.state.m_flat), (a.state.v_flat, b.state.v_flat)):
        assert torch.equal(x, y)
