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
  and runs the per-bucket epilogue as soon as that bucket has landed: the
  finite check of the bucket, and the fused Adam (``xg_adam_range``) of
  every field whose buckets have all been checked - so Adam on the early
  fields overlaps the reduction of the later ones; all ranks then hold
  bit-identical parameters.  Density statistics stay rank-local (the
  per-view screen norms are summed, not the norm of the summed gradient) and
  are all-reduced only at densify events.

Semantics (documented deviation): one DP step consumes ``world`` views of
the reference's per-epoch permutation (trainer.py:373-375) instead of one;
the step's gradient is the sum of the per-view reference gradients.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _native as nat
from .trainer import Trainer


def world_info(group=None) -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def shard_angles(angles, rank: int, world: int) -> np.ndarray:
    """Rank r renders views r, r + world, ... (disjoint, balanced)."""
    a = np.atleast_1d(np.asarray(angles, dtype=np.float64))
    return a[rank::world]


def render_sweep_sharded(cloud, scanner, angles=None, gather: bool = False, group=None, n_streams: int = 3,
                         batch: int = 12):
    """This rank's share of a sweep (and, with ``gather``, the full stack on
    rank 0 in the original view order), through the batched renderer the
    bench measures (``batch`` views per compositing launch)."""
    from .inference import SweepRenderer

    rank, world = world_info(group)
    if angles is None:
        angles = scanner.angles
    angles = np.atleast_1d(np.asarray(angles, dtype=np.float64))
    local = shard_angles(angles, rank, world)
    imgs = SweepRenderer(cloud, scanner, n_streams, batch=max(1, min(batch, len(local)))).render(local)
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


class PeerExchange:
    """The peer-memory form of the data-parallel gradient step (K5,
    csrc/xg_dp.cu): every rank's flat gradient, exchange buffer and sync
    words mapped into this process by CUDA IPC (torch's CUDA tensor sharing,
    handles exchanged once with ``all_gather_object``), then per step two
    kernels - reduce-scatter of the gradient into the exchange buffers and
    an all-gather whose epilogue is the fused Adam - with device-side,
    epoch-counted waits instead of a collective library call.  Rebuilt when
    the gradient buffer changes (density control); the rebuild synchronises
    every rank first, so no kernel still reads the buffers it drops."""

    def __init__(self, grads: torch.Tensor, n: int, nf: int, group=None):
        from torch.multiprocessing.reductions import reduce_tensor

        self.rank, self.world = world_info(group)
        if self.world > nat.XG_PEER_MAX:
            raise ValueError(f"peer exchange supports up to {nat.XG_PEER_MAX} ranks")
        self.group = group
        self.n, self.nf = int(n), int(nf)
        slice_len = int(nat.lib().xg_peer_slice(self.n, self.nf, self.world))
        self.xbuf = torch.zeros(2 * slice_len, dtype=torch.float32, device=grads.device)
        self.sync = torch.zeros(8, dtype=torch.int32, device=grads.device)
        self.key = (grads.data_ptr(), grads.numel())
        torch.cuda.synchronize(grads.device)
        own = (grads, self.xbuf, self.sync)
        shared = [None] * self.world
        if self.world > 1:
            dist.all_gather_object(shared, [reduce_tensor(t) for t in own], group=group)
        self._peers = []  # the peer-mapped tensors, kept alive with the exchange
        pg = nat.XgPeerGroup()
        pg.rank, pg.world, pg.epoch = self.rank, self.world, 0
        for k in range(self.world):
            if k == self.rank:
                ts = own
            else:
                ts = tuple(fn(*args) for fn, args in shared[k])
                self._peers.append(ts)
            pg.grads[k], pg.xbuf[k], pg.sync[k] = (t.data_ptr() for t in ts)
        self.pg = pg
        if self.world > 1:
            dist.barrier(group=group)

    def release(self) -> None:
        torch.cuda.synchronize()
        if self.world > 1:
            dist.barrier(group=self.group)
        self._peers.clear()

    def step(self, params, exp_avg, exp_avg_sq, lr, beta1, beta2, eps, bc1, bc2, sticky_ptr: int) -> None:
        lib = nat.lib()
        self.pg.epoch += 1
        nat.check(lib.xg_peer_reduce_scatter(ctypes.byref(self.pg), self.n, self.nf, sticky_ptr, nat.stream()),
                  "xg_peer_reduce_scatter")
        nat.check(lib.xg_peer_allgather_adam(ctypes.byref(self.pg), params.data_ptr(), exp_avg.data_ptr(),
                                             exp_avg_sq.data_ptr(), self.n, self.nf, lr, beta1, beta2, eps, bc1,
                                             bc2, sticky_ptr, nat.stream()), "xg_peer_allgather_adam")


def allreduce_stats(stats, group=None) -> None:
    """Sum rank-local DensifyStats before a density-control event."""
    if not (dist.is_available() and dist.is_initialized()):
        return
    for t in (stats.norm_sum, stats.obs_count, stats.world_grad_sum):
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)


def _field_ends(n: int, nf: int) -> list[int]:
    """End offsets of the five fields in the flat [pos | rot | log_s | raw | feat] layout."""
    ends, o = [], 0
    for wdt in (3, 4, 3, 1, nf):
        o += n * wdt
        ends.append(o)
    return ends


class DataParallelTrainer(Trainer):
    """Data-parallel training: one view per rank per step, summed gradients,
    bucket-pipelined fused Adam, identical replicas.

    The iteration is ``Trainer.step``'s - the same forward / fused loss
    (L1, or L1 + SSIM when ``gamma > 0``) / reverse pass, opacity reset,
    logging, evaluation and checkpoints (rank 0 writes ``out_dir``) - with
    two phases replaced: the view schedule (``world`` views of the shared
    permutation per step, this rank's is element ``rank``) and the gradient
    application (all-reduce + Adam), plus the density statistics summed over
    ranks before each density-control event.

    Divergence semantics follow the reference's ``adam_step``
    (trainer.py:158-170): fields are checked in order, fields before the
    first non-finite one are updated, that field and every later one are
    not.  Each bucket's finite check runs as soon as it has landed; a
    field's Adam is queued once every bucket of that field (and of all
    earlier fields) has been checked, so a non-finite value in a later
    bucket of a field can never follow a partial update of it."""

    def __init__(self, dataset, cloud, cfg, group=None, bucket_bytes: int = 8 << 20, targets_on_host=False,
                 out_dir=None, verbose: bool = False, reproducible: bool = False, collective: str = "nccl"):
        if collective not in ("nccl", "p2p"):
            raise ValueError("collective must be 'nccl' (bucketed all-reduce) or 'p2p' (PeerExchange)")
        rank, world = world_info(group)
        super().__init__(dataset, cloud, cfg, out_dir=out_dir if rank == 0 else None,
                         verbose=verbose and rank == 0, targets_on_host=targets_on_host,
                         reproducible=reproducible)
        self.rank, self.world = rank, world
        self.group = group
        self.bucket_bytes = bucket_bytes
        self._reducer = None
        self.collective = collective
        self._peer = None

    @property
    def t(self):  # (round-1 API: the wrapped Trainer is now the object itself)
        return self

    def _reducer_for(self, numel: int) -> GradientAllReducer:
        if self._reducer is None or self._reducer.numel != numel:
            self._reducer = GradientAllReducer(numel, self.bucket_bytes, self.group)
        return self._reducer

    def _next_view(self) -> int:
        return dp_views(self.order, self.dataset.train_indices, self.rng, self.world)[self.rank]

    def _upcoming_view(self):
        return self.order[-1 - self.rank] if len(self.order) > self.rank else None

    def _reduce_stats(self) -> None:
        allreduce_stats(self.stats, self.group)

    def _peer_for(self, gflat: torch.Tensor, n: int, nf: int) -> PeerExchange:
        if self._peer is None or self._peer.key != (gflat.data_ptr(), gflat.numel()):
            if self._peer is not None:
                self._peer.release()
            self._peer = PeerExchange(gflat, n, nf, self.group)
        return self._peer

    def _apply_gradients(self) -> None:
        from .trainer import _lr_array

        cfg, cloud, fr = self.cfg, self.cloud, self.eng.frame
        lr = _lr_array(self._lr_table())
        self.state.step += 1
        bc1 = 1.0 - cfg.beta1**self.state.step
        bc2 = 1.0 - cfg.beta2**self.state.step
        n, nf = cloud.n_points, cloud.n_features
        # flags of the SUMMED gradient decide divergence, identically on all
        # ranks: the finite check writes its word at counters[STATUS] of the
        # pointer it gets, so hand it a base that lands on the sticky slot
        sticky = fr.counters.data_ptr() + 4 * nat.XG_CTR_STICKY
        flag_base = sticky - 4 * nat.XG_CTR_STATUS
        lib = nat.lib()
        gflat = self.eng.grads.flat
        if self.collective == "p2p":
            # reduce-scatter + all-gather with Adam as its epilogue, over peer
            # memory (PeerExchange); the global non-finite bits land in sticky
            self._peer_for(gflat, n, nf).step(cloud.flat, self.state.m_flat, self.state.v_flat, lr, cfg.beta1,
                                              cfg.beta2, cfg.eps, bc1, bc2, sticky)
            nat.check(lib.xg_adam_renorm(cloud.flat.data_ptr(), n, nf, sticky, nat.stream()), "xg_adam_renorm")
            cloud.mark_mutated()
            return
        ends = _field_ends(n, nf)
        done = [0]

        def adam(lo, hi):
            nat.check(lib.xg_adam_range(cloud.flat.data_ptr(), gflat.data_ptr(), self.state.m_flat.data_ptr(),
                                        self.state.v_flat.data_ptr(), n, nf, lr, cfg.beta1, cfg.beta2, cfg.eps,
                                        bc1, bc2, sticky, lo, hi, nat.stream()), "xg_adam_range")

        def epilogue(lo, hi):
            nat.check(lib.xg_check_finite_range(gflat.data_ptr(), n, nf, lo, hi, flag_base, nat.stream()),
                      "xg_check_finite_range")
            ready = max([e for e in ends if e <= hi], default=0)  # fields checked in full
            if ready > done[0]:
                adam(done[0], ready)
                done[0] = ready

        self._reducer_for(gflat.numel())(gflat, epilogue)
        if done[0] < gflat.numel():  # (unreachable: the last bucket ends at the last field's end)
            adam(done[0], gflat.numel())
        nat.check(lib.xg_adam_renorm(cloud.flat.data_ptr(), n, nf, sticky, nat.stream()), "xg_adam_renorm")
        cloud.mark_mutated()
