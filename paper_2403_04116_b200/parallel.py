"""Multi-GPU execution of the DRR path.

One process per GPU, ``torch.distributed`` for the plumbing (NCCL on the
B200 node, gloo in the CPU tests).

* Novel-view inference shards naturally: views are independent, so each
  rank renders a disjoint subset (``shard_angles``: round-robin) with no
  collective on the data path; ``render_sweep_sharded`` can optionally
  gather the stacks to rank 0.
* Data-parallel training has exactly one exchange step: every rank renders
  a distinct training view, runs the reverse composite + chain rule, and the
  flat 27N gradient is summed over ranks.  ``GradientAllReducer`` splits the
  flat buffer into buckets, issues every bucket's all-reduce asynchronously
  and runs the per-bucket epilogue (finite check + fused Adam on that
  element range, ``xg_adam_range``) as soon as that bucket has landed, so
  Adam on bucket i overlaps the reduction of bucket i+1; all ranks then
  hold bit-identical parameters.  Density statistics stay rank-local (the
  per-view screen norms are summed, not the norm of the summed gradient) and
  are all-reduced only at densify events.

Semantics (documented deviation): one DP step consumes ``world`` views of
the reference's per-epoch permutation (trainer.py:373-375) instead of one;
the step's gradient is the sum of the per-view reference gradients.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _native as nat


def world_info(group=None) -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def shard_angles(angles, rank: int, world: int) -> np.ndarray:
    """Rank r renders views r, r + world, ... (disjoint, balanced)."""
    a = np.atleast_1d(np.asarray(angles, dtype=np.float64))
    return a[rank::world]


def render_sweep_sharded(cloud, scanner, angles=None, gather: bool = False, group=None, n_streams: int = 3):
    """This rank's share of a sweep (and, with ``gather``, the full stack on
    rank 0 in the original view order)."""
    from .inference import SweepRenderer

    rank, world = world_info(group)
    if angles is None:
        angles = scanner.angles
    angles = np.atleast_1d(np.asarray(angles, dtype=np.float64))
    local = shard_angles(angles, rank, world)
    imgs = SweepRenderer(cloud, scanner, n_streams).render(local)
    if not gather or world == 1:
        return imgs
    return gather_views(imgs, len(angles), rank, world, group)


def gather_views(local: torch.Tensor, n_views: int, rank: int, world: int, group=None):
    """Reassemble round-robin shards on rank 0 (None on other ranks)."""
    h, w = local.shape[-2:]
    per = (n_views + world - 1) // world
    pad = torch.zeros((per, h, w), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == 0 else None
    dist.gather(pad, bufs, dst=0, group=group)
    if rank != 0:
        return None
    out = torch.empty((n_views, h, w), dtype=local.dtype, device=local.device)
    for r in range(world):
        cnt = len(range(r, n_views, world))
        out[r::world] = bufs[r][:cnt]
    return out


def dp_views(order: list, train_indices, rng: np.random.Generator, world: int) -> list[int]:
    """Pop ``world`` views from the shared per-epoch permutation (refilled as
    the reference does, trainer.py:373-375); every rank calls this with the
    same generator state and takes element ``rank``."""
    views = []
    for _ in range(world):
        if not order:
            order.extend(int(i) for i in rng.permutation(train_indices))
        views.append(order.pop())
    return views


class GradientAllReducer:
    """Bucketed sum all-reduce of a flat buffer with a per-bucket epilogue.

    ``epilogue(lo, hi)`` runs (stream-ordered) after elements [lo, hi) hold
    the global sum; with NCCL, ``work.wait()`` only makes the current stream
    wait, so the epilogue of bucket i is queued behind the reduction of
    bucket i while the reduction of bucket i+1 proceeds on NCCL's stream.
    """

    def __init__(self, numel: int, bucket_bytes: int = 8 << 20, group=None):
        self.numel = int(numel)
        self.group = group
        step = max(1, bucket_bytes // 4)
        self.buckets = [(lo, min(lo + step, self.numel)) for lo in range(0, self.numel, step)]

    def __call__(self, flat: torch.Tensor, epilogue=None) -> None:
        if flat.numel() != self.numel:
            raise ValueError("buffer size changed; build a new GradientAllReducer")
        if not (dist.is_available() and dist.is_initialized()):  # single process: nothing to sum
            for lo, hi in self.buckets:
                if epilogue is not None:
                    epilogue(lo, hi)
            return
        works = [dist.all_reduce(flat[lo:hi], op=dist.ReduceOp.SUM, group=self.group, async_op=True)
                 for lo, hi in self.buckets]
        for (lo, hi), wk in zip(self.buckets, works):
            wk.wait()
            if epilogue is not None:
                epilogue(lo, hi)


def allreduce_stats(stats, group=None) -> None:
    """Sum rank-local DensifyStats before a density-control event."""
    if not (dist.is_available() and dist.is_initialized()):
        return
    for t in (stats.norm_sum, stats.obs_count, stats.world_grad_sum):
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)


class DataParallelTrainer:
    """Data-parallel training: one view per rank per step, summed gradients,
    bucket-pipelined fused Adam, identical replicas."""

    def __init__(self, dataset, cloud, cfg, group=None, bucket_bytes: int = 8 << 20, targets_on_host=False):
        from .trainer import Trainer

        self.rank, self.world = world_info(group)
        self.group = group
        self.t = Trainer(dataset, cloud, cfg, targets_on_host=targets_on_host)
        self.bucket_bytes = bucket_bytes
        self._reducer = None

    @property
    def cloud(self):
        return self.t.cloud

    def _reducer_for(self, numel: int) -> GradientAllReducer:
        if self._reducer is None or self._reducer.numel != numel:
            self._reducer = GradientAllReducer(numel, self.bucket_bytes, self.group)
        return self._reducer

    def step(self) -> None:
        from .trainer import DensifyStats, densify_and_prune, position_learning_rate, _lr_array

        t = self.t
        cfg = t.cfg
        t.it += 1
        it = t.it
        views = dp_views(t.order, t.dataset.train_indices, t.rng, self.world)
        view = views[self.rank]
        eng, cloud = t.eng, t.cloud
        fr = eng.frame
        fr.preprocess(cloud, t.cams[view])
        fr.bin_async()  # the forward is queued before the counter read (Trainer.step)
        tgt = t.targets[view]
        if t.targets_on_host:
            t.tgt_bufs[0].copy_(tgt, non_blocking=True)  # (stream-ordered on the compute stream)
            tgt = t.tgt_bufs[0]
        eng.l1.zero_()
        fr.composite(target=tgt, l1_sum=eng.l1, train=True)
        if fr.finish_bin():
            eng.l1.zero_()
            fr.composite(target=tgt, l1_sum=eng.l1, train=True)
        c = fr.last_counters
        nat.raise_for_status(int(c[nat.XG_CTR_STICKY]))
        nat.raise_for_status(int(c[nat.XG_CTR_STATUS]) & ~nat.XG_ST_ENTRY_OVERFLOW)
        fr.backward(cloud, eng.acc, eng.grads.flat, eng.grads.screen_norms, eng.vis, target=tgt,
                    l1_scale=1.0 / (t.h * t.w), stats=t.stats)
        lr = _lr_array({"positions": position_learning_rate(cfg, it - 1), "rotations": cfg.lr_rotation,
                        "log_scales": cfg.lr_scaling, "raw_opacities": cfg.lr_opacity,
                        "features": cfg.lr_feature})
        t.state.step += 1
        bc1 = 1.0 - cfg.beta1**t.state.step
        bc2 = 1.0 - cfg.beta2**t.state.step
        n, nf = cloud.n_points, cloud.n_features
        # flags of the SUMMED gradient decide divergence, identically on all
        # ranks: the finite check writes its word at counters[STATUS] of the
        # pointer it gets, so hand it a base that lands on the sticky slot
        sticky = fr.counters.data_ptr() + 4 * nat.XG_CTR_STICKY
        flag_base = sticky - 4 * nat.XG_CTR_STATUS
        lib = nat.lib()
        gflat = eng.grads.flat

        def epilogue(lo, hi):
            nat.check(lib.xg_check_finite_range(gflat.data_ptr(), n, nf, lo, hi, flag_base, nat.stream()),
                      "xg_check_finite_range")
            nat.check(lib.xg_adam_range(cloud.flat.data_ptr(), gflat.data_ptr(), t.state.m_flat.data_ptr(),
                                        t.state.v_flat.data_ptr(), n, nf, lr, cfg.beta1, cfg.beta2, cfg.eps,
                                        bc1, bc2, sticky, lo, hi, nat.stream()), "xg_adam_range")

        self._reducer_for(gflat.numel())(gflat, epilogue)
        nat.check(lib.xg_adam_renorm(cloud.flat.data_ptr(), n, nf, sticky, nat.stream()), "xg_adam_renorm")
        cloud.mark_mutated()
        if cfg.densify_from_iter < it <= cfg.densify_until_iter and it % cfg.densify_interval == 0:
            nat.raise_for_status(int(fr.counters[nat.XG_CTR_STICKY].item()) & 0xFFFFFFFF)
            allreduce_stats(t.stats, self.group)
            t.cloud, t.state, _ = densify_and_prune(cloud, t.state, t.stats, cfg, t.size_threshold, t.rng)
            t.stats = DensifyStats.zeros(t.cloud.n_points, t.dev)
            eng.resize(t.cloud)
            t.densify_events += 1

