"""Cloud optimisation on the GPU: loss, fused Adam, density control, train loop.

Mirrors ``pkg/src/xsplat/trainer.py`` API for API:

* ``TrainConfig`` (defaults and validation of ``trainer.py:31-100``),
  ``position_learning_rate`` (``:103-106``), ``loss`` (``:109-123``);
* ``OptimizerState`` / ``adam_step`` (``:126-170``) - one fused kernel
  (``xg_adam``) over the flat parameter buffer, quaternion renorm included,
  with the reference's partial-update-then-raise semantics on non-finite
  gradients (``TrainingDivergenceError`` naming the field);
* ``DensifyStats`` / ``densify_and_prune`` (``:173-268``) - masks, counts and
  compaction on the device (``xg_densify_mark`` / ``xg_densify_apply``); the
  split offsets draw ``rng.standard_normal((n_split, 2, 3))`` from the
  caller's numpy generator exactly as the reference does, so a seeded run
  produces the same children;
* ``evaluate`` / ``train`` (``:284-438``) with the same view order (numpy
  permutation per epoch), logging cadence, density-control schedule,
  opacity reset, metrics.tsv and PLY checkpoints.

Inside ``train`` one iteration is: preprocess -> bin (one host sync: entry
count + status words) -> composite with the L1 sum fused and reverse
composite with the L1 pixel gradient computed on the fly, as one overlapped
pair at gamma = 0 (``xg_composite_train_pair``: the replay of each tile starts
as soon as its forward is done) -> chain rule with DensifyStats accumulated
-> fused Adam.  Non-finite gradients
are flagged on the device and surface at the next iteration's sync, before
any further update (same cloud state as the reference at the raise).
"""

from __future__ import annotations

import ctypes
import time
import warnings
from dataclasses import dataclass, fields
from pathlib import Path

import numpy as np
import torch

from . import _native as nat
from .cloudio import save_cloud
from .dataset import ProjectionSet
from .engine import Frame
from .errors import InvalidParameterError, TrainingDivergenceError, XSplatError
from .gaussians import PARAM_FIELDS, GaussianCloud, flat_size, flat_views, logit
from .geometry import camera_pod, extrinsic_from_angle, intrinsic_from_config
from .metrics import MetricReport, SsimEngine, psnr, ssim, ssim_and_gradient, ssim_psnr_stack
from .rasterizer.backward import make_gradients
from .rasterizer.frontend import RenderGradients, render


@dataclass
class TrainConfig:
    iterations: int = 20_000
    gamma: float = 0.0
    lr_position_init: float = 1.9e-4
    lr_position_final: float = 1.9e-6
    lr_feature: float = 2e-3
    lr_opacity: float = 8e-3
    lr_scaling: float = 5e-3
    lr_rotation: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-15
    densify_interval: int = 100
    densify_grad_threshold: float = 2e-5
    prune_opacity_threshold: float = 0.005
    densify_from_iter: int = 500
    densify_until_iter: int = 15_000
    split_factor: float = 1.6
    densify_size_threshold: float | None = None
    max_points: int = 500_000
    opacity_reset_interval: int = 0
    rng_seed: int = 0
    log_interval: int = 10
    eval_interval: int = 200
    checkpoint_iterations: tuple = ()

    def __post_init__(self):
        if self.iterations < 1:
            raise InvalidParameterError("iterations must be >= 1")
        if not 0.0 <= self.gamma <= 1.0:
            raise InvalidParameterError(f"gamma must be in [0, 1], got {self.gamma}")
        for name in ("lr_position_init", "lr_position_final", "lr_feature", "lr_opacity", "lr_scaling",
                     "lr_rotation"):
            if not getattr(self, name) > 0:
                raise InvalidParameterError(f"{name} must be > 0")
        if not 0 <= self.beta1 < 1 or not 0 <= self.beta2 < 1 or not self.eps > 0:
            raise InvalidParameterError("invalid Adam parameters")
        for name in ("densify_interval", "log_interval", "eval_interval"):
            if getattr(self, name) < 1:
                raise InvalidParameterError(f"{name} must be >= 1")
        if self.split_factor <= 1.0:
            raise InvalidParameterError("split_factor must be > 1")
        self.checkpoint_iterations = tuple(int(i) for i in self.checkpoint_iterations)

    def to_dict(self) -> dict:
        d = {f.name: getattr(self, f.name) for f in fields(self)}
        d["checkpoint_iterations"] = list(self.checkpoint_iterations)
        return d

    @classmethod
    def from_dict(cls, d: dict) -> "TrainConfig":
        unknown = set(d) - {f.name for f in fields(cls)}
        if unknown:
            raise InvalidParameterError(f"unknown TrainConfig keys: {sorted(unknown)}")
        return cls(**d)


def position_learning_rate(cfg: TrainConfig, t: int) -> float:
    return cfg.lr_position_init * (cfg.lr_position_final / cfg.lr_position_init) ** (t / cfg.iterations)


def _dev(x, device=None) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(dtype=torch.float64, device=device or (x.device if x.is_cuda else "cuda"))
    return torch.as_tensor(np.asarray(x, dtype=np.float64), device=device or "cuda")


def loss(rendered, target, gamma: float):
    """(1-gamma) L1 + gamma (1 - SSIM) and its pixel gradient (trainer.py:109-123)."""
    img = _dev(getattr(rendered, "pixels", rendered))
    ref = _dev(getattr(target, "pixels", target), img.device)
    if img.shape != ref.shape:
        raise InvalidParameterError(f"shape mismatch {tuple(img.shape)} vs {tuple(ref.shape)}")
    if not 0.0 <= gamma <= 1.0:
        raise InvalidParameterError(f"gamma must be in [0, 1], got {gamma}")
    diff = img - ref
    l1 = float(torch.mean(torch.abs(diff)))
    grad = (1.0 - gamma) * torch.sign(diff) / diff.numel()
    if gamma == 0.0:
        return l1, grad
    s, ds = ssim_and_gradient(img, ref)
    return (1.0 - gamma) * l1 + gamma * (1.0 - s), grad - gamma * ds


class OptimizerState:
    """Adam moments (flat buffers laid out like the cloud) + shared step."""

    def __init__(self, cloud: GaussianCloud):
        self.step = 0
        self._n, self._nf = cloud.n_points, cloud.n_features
        self.m_flat = torch.zeros(flat_size(self._n, self._nf), dtype=torch.float32, device=cloud.device)
        self.v_flat = torch.zeros_like(self.m_flat)
        self.exp_avg = flat_views(self.m_flat, self._n, self._nf)
        self.exp_avg_sq = flat_views(self.v_flat, self._n, self._nf)

    @classmethod
    def from_flat(cls, m_flat, v_flat, n, nf, step):
        obj = cls.__new__(cls)
        obj.step, obj._n, obj._nf = step, n, nf
        obj.m_flat, obj.v_flat = m_flat, v_flat
        obj.exp_avg = flat_views(m_flat, n, nf)
        obj.exp_avg_sq = flat_views(v_flat, n, nf)
        return obj

    def check_congruent(self, cloud: GaussianCloud) -> None:
        for f in PARAM_FIELDS:
            if tuple(self.exp_avg[f].shape) != tuple(getattr(cloud, f).shape):
                raise InvalidParameterError(
                    f"optimizer state for {f} has shape {tuple(self.exp_avg[f].shape)}, "
                    f"cloud has {tuple(getattr(cloud, f).shape)}")


def _grads_flat(grads: RenderGradients, cloud: GaussianCloud) -> torch.Tensor:
    fl = getattr(grads, "flat", None)
    if fl is not None and fl.numel() == cloud.flat.numel() and fl.device == cloud.device:
        # the field views must still alias the flat buffer
        if all(getattr(grads, f).data_ptr() == v.data_ptr()
               for f, v in flat_views(fl, cloud.n_points, cloud.n_features).items()):
            return fl
    parts = [torch.as_tensor(np.asarray(getattr(grads, f).cpu() if isinstance(getattr(grads, f), torch.Tensor)
                                        else getattr(grads, f)), dtype=torch.float32).reshape(-1)
             for f in PARAM_FIELDS]
    return torch.cat(parts).to(cloud.device).contiguous()


def _lr_array(lr_table: dict) -> ctypes.Array:
    return (ctypes.c_double * 5)(*[float(lr_table[f]) for f in PARAM_FIELDS])


def _adam_launch(cloud, gflat, state, lr_table, cfg, status_ptr) -> None:
    bc1 = 1.0 - cfg.beta1**state.step
    bc2 = 1.0 - cfg.beta2**state.step
    nat.check(
        nat.lib().xg_adam(cloud.flat.data_ptr(), gflat.data_ptr(), state.m_flat.data_ptr(),
                          state.v_flat.data_ptr(), cloud.n_points, cloud.n_features, _lr_array(lr_table),
                          cfg.beta1, cfg.beta2, cfg.eps, bc1, bc2, status_ptr, nat.stream()),
        "xg_adam",
    )
    cloud.mark_mutated()


def adam_step(cloud: GaussianCloud, grads: RenderGradients, state: OptimizerState, lr_table: dict,
              cfg: TrainConfig) -> None:
    """One fused Adam update in place (trainer.py:147-170)."""
    state.check_congruent(cloud)
    nat.require_cuda(cloud.flat, "cloud")
    state.step += 1
    gflat = _grads_flat(grads, cloud)
    counters = torch.zeros(nat.XG_NCOUNTERS, dtype=torch.int32, device=cloud.device)
    nat.check(nat.lib().xg_check_finite(gflat.data_ptr(), cloud.n_points, cloud.n_features,
                                        counters.data_ptr(), nat.stream()), "xg_check_finite")
    _adam_launch(cloud, gflat, state, lr_table, cfg, counters.data_ptr() + 4 * nat.XG_CTR_STATUS)
    word = int(counters[nat.XG_CTR_STATUS].item()) & 0xFFFFFFFF
    nat.raise_for_status(word)


@dataclass
class DensifyStats:
    norm_sum: torch.Tensor
    obs_count: torch.Tensor
    world_grad_sum: torch.Tensor

    @classmethod
    def zeros(cls, n: int, device=None) -> "DensifyStats":
        device = device or ("cuda" if torch.cuda.is_available() else "cpu")
        return cls(torch.zeros(n, dtype=torch.float32, device=device),
                   torch.zeros(n, dtype=torch.int32, device=device),
                   torch.zeros((n, 3), dtype=torch.float32, device=device))

    def accumulate(self, grads: RenderGradients) -> None:
        self.norm_sum += torch.as_tensor(grads.screen_norms, device=self.norm_sum.device).float()
        self.obs_count += torch.as_tensor(grads.visible, device=self.obs_count.device).to(torch.int32)
        self.world_grad_sum += torch.as_tensor(grads.positions, device=self.world_grad_sum.device).float()


def densify_and_prune(cloud: GaussianCloud, state: OptimizerState, stats: DensifyStats, cfg: TrainConfig,
                      size_threshold: float, rng: np.random.Generator):
    """Clone / split / prune (trainer.py:191-268); returns (cloud, state, report)."""
    state.check_congruent(cloud)
    nat.require_cuda(cloud.flat, "cloud")
    n, nf, dev = cloud.n_points, cloud.n_features, cloud.device
    ns = stats.norm_sum.to(dev, torch.float32).contiguous()
    oc = stats.obs_count.to(dev, torch.int32).contiguous()
    wg = stats.world_grad_sum.to(dev, torch.float32).contiguous()
    flags = torch.empty(n, dtype=torch.uint8, device=dev)
    counts = torch.zeros(4, dtype=torch.int32, device=dev)
    nat.check(nat.lib().xg_densify_mark(cloud.flat.data_ptr(), n, nf, ns.data_ptr(), oc.data_ptr(),
                                        float(cfg.densify_grad_threshold), float(size_threshold),
                                        float(cfg.prune_opacity_threshold), flags.data_ptr(), counts.data_ptr(),
                                        nat.stream()), "xg_densify_mark")
    n_prune, n_clone, n_split = (int(v) for v in counts[:3].cpu())
    allow = 1
    if n - n_prune + n_clone + n_split > cfg.max_points:
        warnings.warn(f"densification skipped: {n - n_prune + n_clone + n_split} Gaussians would exceed cap "
                      f"{cfg.max_points}", stacklevel=2)
        allow, n_clone, n_split = 0, 0, 0
    n_keep = n - n_prune - n_split
    if n_keep + n_clone + n_split == 0:
        raise XSplatError("density control pruned every Gaussian")
    n_new = n_keep + n_clone + 2 * n_split
    normals = torch.zeros(max(6 * n_split, 1), dtype=torch.float64, device=dev)
    if n_split:
        normals = torch.as_tensor(rng.standard_normal((n_split, 2, 3)), dtype=torch.float64).reshape(-1).to(dev)
    new_p = torch.empty(flat_size(n_new, nf), dtype=torch.float32, device=dev)
    new_m = torch.empty_like(new_p)
    new_v = torch.empty_like(new_p)
    scratch = torch.empty(int(nat.lib().xg_densify_scratch_bytes(n)), dtype=torch.uint8, device=dev)
    nat.check(nat.lib().xg_densify_apply(cloud.flat.data_ptr(), state.m_flat.data_ptr(), state.v_flat.data_ptr(),
                                         n, nf, flags.data_ptr(), wg.data_ptr(), normals.data_ptr(),
                                         float(np.log(cfg.split_factor)), allow, new_p.data_ptr(),
                                         new_m.data_ptr(), new_v.data_ptr(), n_new, scratch.data_ptr(),
                                         nat.stream()), "xg_densify_apply")
    new_cloud = GaussianCloud.from_flat(new_p, n_new, nf, cloud.basis_weights.clone())
    new_state = OptimizerState.from_flat(new_m, new_v, n_new, nf, state.step)
    report = {"pruned": n_prune, "cloned": n_clone, "split": n_split, "n_points": n_new}
    return new_cloud, new_state, report


@dataclass
class TrainResult:
    cloud: GaussianCloud
    metrics: list
    out_dir: Path | None = None

    def test_psnr_at(self, iteration: int):
        for row in self.metrics:
            if row["iteration"] == iteration and row.get("test_psnr") is not None:
                return row["test_psnr"]
        return None


def evaluate(cloud: GaussianCloud, dataset: ProjectionSet, indices, use_clean: bool = True) -> MetricReport:
    """Mean / per-view PSNR and SSIM of renders vs the dataset (trainer.py:284-315)."""
    from .inference import SweepRenderer

    indices = np.asarray(indices, dtype=np.int64)
    stack = dataset.clean_images if use_clean else dataset.images
    if indices.size == 0:
        return MetricReport(psnr=float("nan"), ssim=float("nan"), per_view=[])
    imgs = SweepRenderer(cloud, dataset.scanner, batch=min(12, max(1, int(indices.size)))).render(
        dataset.angles[indices])
    refs = torch.as_tensor(np.asarray(stack)[indices], device=cloud.device)
    s, p = ssim_psnr_stack(imgs, refs)  # one launch per view, one sync
    per = [{"view": int(i), "angle": float(dataset.angles[i]), "psnr": float(p[k]), "ssim": float(s[k])}
           for k, i in enumerate(indices)]
    return MetricReport(psnr=float(np.mean([v["psnr"] for v in per])),
                        ssim=float(np.mean([v["ssim"] for v in per])), per_view=per)


METRICS_HEADER = "iteration\tloss\ttrain_psnr\ttest_psnr\ttest_ssim\tn_points\n"


def _metrics_row(row: dict) -> str:
    tp = "-" if row.get("test_psnr") is None else f"{row['test_psnr']:.6f}"
    ts = "-" if row.get("test_ssim") is None else f"{row['test_ssim']:.6f}"
    return f"{row['iteration']}\t{row['loss']:.10e}\t{row['train_psnr']:.6f}\t{tp}\t{ts}\t{row['n_points']}\n"


class _IterationEngine:
    """Persistent device buffers of the training loop (one Frame, gradient,
    accumulator and loss buffers), rebuilt when density control resizes N."""

    def __init__(self, cloud: GaussianCloud, h: int, w: int):
        self.h, self.w = h, w
        self.resize(cloud)
        self.dl = torch.empty((h, w), dtype=torch.float32, device=cloud.device)  # fused loss gradient
        self.ssim = None  # SsimEngine, created on the first gamma > 0 step

    @property
    def l1(self) -> torch.Tensor:
        """The fused-L1 sum of the current frame's forward (zeroed by its preprocess)."""
        return self.frame.l1_sum

    def resize(self, cloud: GaussianCloud, capacity: int | None = None) -> None:
        n = cloud.n_points
        cap = capacity or (getattr(self, "frame", None) and self.frame.entry_capacity) or 16 * n
        self.frame = Frame(n, self.h, self.w, cloud.device, entry_capacity=cap)
        self.frame._alloc_replay()  # (a training frame from the first bin on: entry-balanced binning)
        self.grads = make_gradients(n, cloud.n_features, cloud.device)
        self.acc = torch.empty((n, 8), dtype=torch.float32, device=cloud.device)  # (zeroed by xg_composite_bwd)
        self.vis = torch.empty(n, dtype=torch.uint8, device=cloud.device)


class Trainer:
    """The train loop of trainer.py:330-438 as a resumable object: ``step()``
    runs one iteration; ``run()`` runs to ``cfg.iterations``.  ``train()``
    is ``Trainer(...).run()``."""

    def __init__(self, dataset: ProjectionSet, cloud: GaussianCloud, cfg: TrainConfig, out_dir=None,
                 verbose: bool = False, targets_on_host: bool = False, reproducible: bool = False):
        if dataset.train_indices.size < 1:
            raise InvalidParameterError("dataset has no training projections")
        nat.require_cuda(cloud.flat, "cloud")
        self.dataset, self.cfg, self.verbose = dataset, cfg, verbose
        # reproducible: gradients summed in a fixed order (Frame.backward),
        # logged losses by an in-order reduction - byte-identical runs, like
        # the reference's single-threaded loop (test_trainer.py:336-353)
        self.reproducible = bool(reproducible)
        # measurement hook: when a dict of lists, (start, end) CUDA events
        # around each iteration's forward / reverse composite launches
        self.kernel_events = None
        self.cloud = cloud.copy()
        self.dev = dev = self.cloud.device
        self.state = OptimizerState(self.cloud)
        self.rng = np.random.default_rng(cfg.rng_seed)
        self.stats = DensifyStats.zeros(self.cloud.n_points, dev)
        pos = self.cloud.positions
        span = float((pos.max(0).values - pos.min(0).values).max())
        self.size_threshold = (cfg.densify_size_threshold if cfg.densify_size_threshold is not None
                               else 0.01 * max(span, 1.0))
        sc = dataset.scanner
        intr = intrinsic_from_config(sc)
        self.h, self.w = h, w = sc.detector_height, sc.detector_width
        self.cams = {int(i): camera_pod(extrinsic_from_angle(sc, float(dataset.angles[i])), intr, (h, w))
                     for i in dataset.train_indices}
        # targets resident in HBM (default), or kept in pinned host memory and
        # copied per iteration (end-to-end measurement)
        self.targets_on_host = targets_on_host
        self.tgt_slot = 0
        if targets_on_host:
            self.targets = {int(i): torch.as_tensor(dataset.images[i], dtype=torch.float32).pin_memory()
                            for i in dataset.train_indices}
            # double-buffered: the next view's target is copied on a side
            # stream while the current step runs
            self.tgt_bufs = [torch.empty((h, w), dtype=torch.float32, device=dev) for _ in range(2)]
            self.copy_stream = torch.cuda.Stream(device=dev)
            self.tgt_ready = [torch.cuda.Event(), torch.cuda.Event()]
            self.tgt_free = [torch.cuda.Event(), torch.cuda.Event()]
            self.tgt_view = [None, None]
            self.loss_host = torch.zeros(1, dtype=torch.float64).pin_memory()
        else:
            self.targets = {int(i): torch.as_tensor(dataset.images[i], dtype=torch.float32, device=dev).contiguous()
                            for i in dataset.train_indices}
        self.out_path = Path(out_dir) if out_dir is not None else None
        self.log = None
        if self.out_path is not None:
            self.out_path.mkdir(parents=True, exist_ok=True)
            self.log = open(self.out_path / "metrics.tsv", "w")
            self.log.write(METRICS_HEADER)
        self.eng = _IterationEngine(self.cloud, h, w)
        self.metrics: list = []
        self.order: list = []
        self.it = 0
        self.t0 = time.perf_counter()
        self.densify_events = 0

    def _copy_target(self, slot: int, view: int) -> None:
        """H2D copy of a view's target into buffer ``slot`` on the side
        stream, after the buffer's previous user finished."""
        with torch.cuda.stream(self.copy_stream):
            self.copy_stream.wait_event(self.tgt_free[slot])
            self.tgt_bufs[slot].copy_(self.targets[view], non_blocking=True)
            self.tgt_ready[slot].record(self.copy_stream)
        self.tgt_view[slot] = view

    # --- one iteration, in phases (DataParallelTrainer overrides the view
    # --- choice and the gradient application) ---------------------------------
    def step(self) -> None:
        self.it += 1
        view = self._next_view()
        slot = self.tgt_slot
        tgt = self._render_and_backward(view, slot)
        self._apply_gradients()
        self._tail(tgt, slot)

    def _next_view(self) -> int:
        if not self.order:
            self.order = [int(i) for i in self.rng.permutation(self.dataset.train_indices)]
        return self.order.pop()

    def _upcoming_view(self):
        """The view the next step will train on, if known (target prefetch)."""
        return self.order[-1] if self.order else None

    def _render_and_backward(self, view: int, slot: int) -> torch.Tensor:
        """Forward with the fused L1 sum, the loss's pixel gradient and the
        reverse pass into ``eng.grads`` (+ DensifyStats); returns the target."""
        cfg, eng = self.cfg, self.eng
        h, w = self.h, self.w
        fr = eng.frame
        fr.preprocess(self.cloud, self.cams[view])
        # the forward is queued before the host reads the binning counters
        # (it skips itself on the device after an entry overflow, then runs
        # again on the re-binned lists), so the GPU never waits on the sync
        fr.bin_async()
        if self.targets_on_host:
            if self.tgt_view[slot] != view:  # not prefetched by the previous step
                self._copy_target(slot, view)
            torch.cuda.current_stream().wait_event(self.tgt_ready[slot])
            tgt = self.tgt_bufs[slot]
        else:
            tgt = self.targets[view]
        ke = self.kernel_events
        # plain L1 (gamma = 0): forward and reverse replay as one overlapped
        # pair (xg_composite_train_pair); the SSIM objective needs the whole
        # image before its pixel gradient exists, the reproducible mode its
        # own replay
        pair = cfg.gamma == 0.0 and not self.reproducible
        # (the L1 accumulator lives in the frame's counters, zeroed by preprocess)
        if pair:
            fr.train_pair(tgt, eng.l1, eng.acc, 1.0 / (h * w), events=ke["pair"] if ke is not None else None)
            if fr.finish_bin():  # (the skipped first pair added nothing)
                fr.train_pair(tgt, eng.l1, eng.acc, 1.0 / (h * w))
        else:
            fr.composite(target=tgt, l1_sum=eng.l1, train=True, events=ke["fwd"] if ke is not None else None)
            if fr.finish_bin():  # (the skipped first forward added nothing)
                fr.composite(target=tgt, l1_sum=eng.l1, train=True)
        c = fr.last_counters
        nat.raise_for_status(int(c[nat.XG_CTR_STICKY]))  # divergence of the previous step
        nat.raise_for_status(int(c[nat.XG_CTR_STATUS]) & ~nat.XG_ST_ENTRY_OVERFLOW)
        if self.targets_on_host:
            self.loss_host.copy_(eng.l1, non_blocking=True)  # the step's scalar result, to the host
        self.s_dev = None
        if pair:
            fr.backward(self.cloud, eng.acc, eng.grads.flat, eng.grads.screen_norms, eng.vis, stats=self.stats,
                        replay_done=True)
        elif cfg.gamma == 0.0:
            fr.backward(self.cloud, eng.acc, eng.grads.flat, eng.grads.screen_norms, eng.vis, target=tgt,
                        l1_scale=1.0 / (h * w), stats=self.stats, reproducible=self.reproducible,
                        events=ke["bwd"] if ke is not None else None)
        else:
            # xg_ssim writes dl = -gamma dSSIM/dI + (1 - gamma) sign(I - T) / HW
            # (trainer.py:117-123) straight into the backward's input
            if eng.ssim is None:
                eng.ssim = SsimEngine(h, w, self.dev)
            self.s_dev = eng.ssim.run(fr.image, tgt, 1.0, dl=eng.dl, dl_ssim_scale=-cfg.gamma,
                                      dl_l1_scale=(1.0 - cfg.gamma) / (h * w))
            fr.backward(self.cloud, eng.acc, eng.grads.flat, eng.grads.screen_norms, eng.vis,
                        dl_dimage=eng.dl, stats=self.stats, reproducible=self.reproducible,
                        events=ke["bwd"] if ke is not None else None)
        return tgt

    def _lr_table(self) -> dict:
        cfg = self.cfg
        return {"positions": position_learning_rate(cfg, self.it - 1), "rotations": cfg.lr_rotation,
                "log_scales": cfg.lr_scaling, "raw_opacities": cfg.lr_opacity, "features": cfg.lr_feature}

    def _apply_gradients(self) -> None:
        fr = self.eng.frame
        # (xg_preprocess_bwd ORed this step's non-finite flags into the sticky word Adam reads)
        self.state.step += 1
        _adam_launch(self.cloud, self.eng.grads.flat, self.state, self._lr_table(), self.cfg,
                     fr.counters.data_ptr() + 4 * nat.XG_CTR_STICKY)

    def _reduce_stats(self) -> None:
        """Density statistics of this process are the whole step's (DP: summed)."""

    def _tail(self, tgt: torch.Tensor, slot: int) -> None:
        """Density control, opacity reset, logging / evaluation, checkpoints
        (trainer.py:389-437) and the next target's prefetch."""
        cfg, eng, it = self.cfg, self.eng, self.it
        h, w = self.h, self.w
        fr = eng.frame
        densify_now = cfg.densify_from_iter < it <= cfg.densify_until_iter and it % cfg.densify_interval == 0
        reset_now = bool(cfg.opacity_reset_interval) and it % cfg.opacity_reset_interval == 0
        log_now = it % cfg.log_interval == 0 or it == cfg.iterations
        ckpt_now = self.out_path is not None and it in cfg.checkpoint_iterations
        if densify_now or reset_now or log_now or ckpt_now or it == cfg.iterations:
            # the reference raises inside adam_step, before any of these
            nat.raise_for_status(int(fr.counters[nat.XG_CTR_STICKY].item()) & 0xFFFFFFFF)
        if densify_now:
            self._reduce_stats()
            self.cloud, self.state, rep = densify_and_prune(self.cloud, self.state, self.stats, cfg,
                                                            self.size_threshold, self.rng)
            self.stats = DensifyStats.zeros(self.cloud.n_points, self.dev)
            eng.resize(self.cloud)
            self.densify_events += 1
            if self.verbose:
                print(f"[{it}] density control: {rep}")
        if reset_now:
            self.cloud.raw_opacities.clamp_(max=logit(0.01))
            self.state.exp_avg["raw_opacities"].zero_()
            self.state.exp_avg_sq["raw_opacities"].zero_()
        if log_now:
            if self.reproducible:  # (the fused L1 sum adds with float atomics)
                value = float((fr.image.double() - tgt.double()).abs().mean())
            else:
                value = float(fr.l1_sum.item()) / (h * w)  # (fr: this step's frame, even after a resize)
            if cfg.gamma != 0.0:
                value = (1.0 - cfg.gamma) * value + cfg.gamma * (1.0 - float(self.s_dev.item()))
            row = {"iteration": it, "loss": value, "train_psnr": psnr(fr.image, tgt), "test_psnr": None,
                   "test_ssim": None, "n_points": self.cloud.n_points}
            if it % cfg.eval_interval == 0 or it == cfg.iterations:
                rep = evaluate(self.cloud, self.dataset, self.dataset.test_indices)
                row["test_psnr"], row["test_ssim"] = rep.psnr, rep.ssim
                if self.verbose:
                    print(f"[{it}] loss {value:.5f} test PSNR {rep.psnr:.2f} dB SSIM {rep.ssim:.4f} "
                          f"N {self.cloud.n_points} ({time.perf_counter() - self.t0:.1f}s)")
            self.metrics.append(row)
            if self.log is not None:
                self.log.write(_metrics_row(row))
                self.log.flush()
        if ckpt_now:
            save_cloud(self.cloud, self.out_path / f"ckpt_{it:06d}.ply")
        if self.targets_on_host:
            # this step's target buffer is free once its kernels ran; the next
            # view's target goes into the other one now
            self.tgt_free[slot].record()
            nxt = self._upcoming_view()
            if nxt is not None:
                self._copy_target(1 - slot, nxt)
            self.tgt_slot = 1 - slot

    def close(self) -> None:
        if self.log is not None:
            self.log.close()
            self.log = None

    def run(self) -> TrainResult:
        try:
            while self.it < self.cfg.iterations:
                self.step()
        finally:
            self.close()
        if self.out_path is not None:
            save_cloud(self.cloud, self.out_path / "cloud_final.ply")
        return TrainResult(cloud=self.cloud, metrics=self.metrics, out_dir=self.out_path)


def train(dataset: ProjectionSet, cloud: GaussianCloud, cfg: TrainConfig, out_dir=None,
          verbose: bool = False, reproducible: bool = False) -> TrainResult:
    """Optimise the cloud against the training projections (trainer.py:330-438).
    ``reproducible=True`` makes runs byte-identical (fixed-order gradient
    sums; ~7 % slower per C2 iteration), as the reference's are."""
    return Trainer(dataset, cloud, cfg, out_dir, verbose, reproducible=reproducible).run()


__all__ = [
    "PARAM_FIELDS", "DensifyStats", "OptimizerState", "TrainConfig", "TrainResult", "Trainer", "adam_step",
    "densify_and_prune", "evaluate", "loss", "position_learning_rate", "train", "render",
]
