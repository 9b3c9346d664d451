"""Per-view device buffers and the stream-ordered call sequence of one render.

``Frame`` owns every buffer one view needs (per-Gaussian screen-space
records, the sorted entry list, tile ranges, image / final transmittance /
contributor counts, the binning workspace) and drives the C-ABI:

    xg_preprocess_fwd -> xg_bin_sort -> xg_composite_fwd
    xg_composite_bwd  -> xg_preprocess_bwd

Nothing here synchronises except :meth:`Frame.read_counters`.  The entry
buffer is sized from a capacity; an overflow is reported by the device
status word and the frame is re-binned with the exact size
(:meth:`Frame.ensure_binned`).
"""

from __future__ import annotations

import ctypes

import torch

from . import _native as nat
from .geometry import XgCamera

TILE_SIZE = 16


def tile_grid(h: int, w: int) -> tuple[int, int]:
    return (h + TILE_SIZE - 1) // TILE_SIZE, (w + TILE_SIZE - 1) // TILE_SIZE


class Frame:
    """Device buffers of one view for a cloud of ``n`` Gaussians."""

    def __init__(self, n: int, h: int, w: int, device, entry_capacity: int | None = None,
                 extras: bool = False):
        self.n, self.h, self.w = int(n), int(h), int(w)
        self.device = torch.device(device)
        nty, ntx = tile_grid(h, w)
        self.n_tiles = ntx * nty
        dev = self.device
        self.mean2d = torch.empty((n, 2), dtype=torch.float64, device=dev)
        self.coef = torch.empty((n, 4), dtype=torch.float32, device=dev)
        self.inten = torch.empty(n, dtype=torch.float32, device=dev)
        self._own_inten = self.inten
        self.rect = torch.empty((n, 4), dtype=torch.int16, device=dev)
        self.tiles_touched = torch.empty(n, dtype=torch.int32, device=dev)
        self.depth_key = torch.empty(n, dtype=torch.int64, device=dev)
        self.order = torch.empty(n, dtype=torch.int32, device=dev)
        self.tile_ranges = torch.empty((self.n_tiles, 2), dtype=torch.int64, device=dev)
        self.tile_order = torch.empty(self.n_tiles, dtype=torch.int32, device=dev)
        self.unit_cost = torch.empty(4 * self.n_tiles, dtype=torch.int32, device=dev)
        self.unit_order = torch.empty(4 * self.n_tiles, dtype=torch.int32, device=dev)
        self.counters = torch.zeros(nat.XG_NCOUNTERS, dtype=torch.int32, device=dev)
        self.image = torch.empty((h, w), dtype=torch.float32, device=dev)
        self.fwd_image = self.image
        self.t_final = torch.empty((h, w), dtype=torch.float32, device=dev)
        self.n_contrib = torch.empty((h, w), dtype=torch.int32, device=dev)
        self.extras = None
        if extras:
            self.extras = {
                "cov2d": torch.empty((n, 3), dtype=torch.float64, device=dev),
                "conic": torch.empty((n, 3), dtype=torch.float64, device=dev),
                "depth": torch.empty(n, dtype=torch.float64, device=dev),
                "t_cam": torch.empty((n, 3), dtype=torch.float64, device=dev),
                "radius": torch.empty(n, dtype=torch.float64, device=dev),
                "opacity": torch.empty(n, dtype=torch.float64, device=dev),
            }
        self.entry_capacity = 0
        self.entry_splat = None
        self.workspace = None
        self.replay_ckpt = None  # training frames only: allocated by the first tracking composite
        self.replay_items = None
        self.entry_grad = None  # reproducible backward only: per-(splat, tile) slots + offsets (bytes)
        self.set_capacity(entry_capacity if entry_capacity else max(16 * n, 1024))
        self.cam = None
        self.has_forward = False

    def set_capacity(self, cap: int) -> None:
        cap = int(cap)
        if cap <= self.entry_capacity and self.entry_splat is not None:
            return
        self.entry_capacity = cap
        # (+4 slack entries: 16 B-rounded bulk copies of a list's tail stay inside the allocation)
        self.entry_splat = torch.empty(cap + 4, dtype=torch.int32, device=self.device)
        ws = nat.lib().xg_bin_workspace_bytes(self.n, cap, self.n_tiles)
        self.workspace = torch.empty(int(ws), dtype=torch.uint8, device=self.device)
        if self.replay_ckpt is not None:
            self._alloc_replay()

    def _alloc_replay(self) -> None:
        """Checkpoints of the chunked reverse replay: (T, acc) of every pixel
        before each XG_REPLAY_CHUNK-th entry of its tile, plus the chunk list
        (include/xgauss.h, xg_splats.replay_ckpt)."""
        slots = int(nat.lib().xg_replay_slots(self.entry_capacity, self.n_tiles))
        self.replay_ckpt = torch.empty((slots, 256, 2), dtype=torch.float32, device=self.device)
        self.replay_items = torch.empty((4 * slots, 2), dtype=torch.int32, device=self.device)

    def splats_struct(self) -> nat.XgSplats:
        s = nat.XgSplats()
        s.mean2d = self.mean2d.data_ptr()
        s.coef = self.coef.data_ptr()
        s.inten = self.inten.data_ptr()
        s.rect = self.rect.data_ptr()
        s.n_tiles = self.tiles_touched.data_ptr()
        s.depth_key = self.depth_key.data_ptr()
        s.order = self.order.data_ptr()
        s.entry_splat = self.entry_splat.data_ptr()
        s.tile_ranges = self.tile_ranges.data_ptr()
        s.counters = self.counters.data_ptr()
        s.n = self.n
        s.entry_capacity = self.entry_capacity
        s.tile_order = self.tile_order.data_ptr()
        s.unit_cost = self.unit_cost.data_ptr()
        s.unit_order = self.unit_order.data_ptr()
        if self.replay_ckpt is not None:
            s.replay_ckpt = self.replay_ckpt.data_ptr()
            s.replay_items = self.replay_items.data_ptr()
            s.replay_slots = self.replay_ckpt.shape[0]
        return s

    # --- stages -------------------------------------------------------------
    def preprocess(self, cloud, cam: XgCamera, intensities: torch.Tensor | None = None,
                   invariants: torch.Tensor | None = None) -> None:
        """K1.  ``intensities`` (the cloud's precomputed [N] float32
        sigmoid(F . lambda), e.g. for a sweep) is used as this frame's
        intensity buffer instead of recomputing it per view; ``invariants``
        (``_native.view_invariants``) likewise replaces the per-view
        covariance / opacity evaluation (same numbers, computed once)."""
        if cloud.n_points != self.n:
            raise ValueError("frame was allocated for a different cloud size")
        self.cam = cam
        if intensities is not None:
            self.inten = intensities  # shared, read-only for the compositing kernels
        elif getattr(self, "_own_inten", None) is not None and self.inten is not self._own_inten:
            self.inten = self._own_inten
        cs = nat.cloud_struct(cloud, intensities, invariants)
        sp = self.splats_struct()
        ex = None
        if self.extras is not None:
            ex = nat.XgSplatExtras(**{k: v.data_ptr() for k, v in self.extras.items()})
        nat.check(
            nat.lib().xg_preprocess_fwd(
                ctypes.byref(cs), ctypes.byref(cam), ctypes.byref(sp),
                ctypes.byref(ex) if ex is not None else None, nat.stream(),
            ),
            "xg_preprocess_fwd",
        )
        self.has_forward = False

    def bin(self) -> None:
        sp = self.splats_struct()
        nat.check(
            nat.lib().xg_bin_sort(
                ctypes.byref(self.cam), ctypes.byref(sp), self.workspace.data_ptr(),
                self.workspace.numel(), nat.stream(),
            ),
            "xg_bin_sort",
        )

    def composite(self, target: torch.Tensor | None = None, l1_sum: torch.Tensor | None = None,
                  image_out: torch.Tensor | None = None, track: bool = True, train: bool = False,
                  events: list | None = None) -> None:
        """K3.  ``image_out`` (float32 [H, W], contiguous) receives the image
        instead of the frame's own buffer (e.g. a slot of a sweep stack).
        ``track=False`` (inference) skips the per-pixel final transmittance
        and contributor counts the backward needs.  ``train=True`` (the
        trainer) is the tracking forward whose n_contrib is only the reverse
        replay's start (``xg_composite_fwd_train``), not the reference's
        contributor count."""
        if track and self.replay_ckpt is None:
            self._alloc_replay()
        sp = self.splats_struct()
        img = self.image if image_out is None else image_out
        fn = "xg_composite_fwd_train" if (track and train) else "xg_composite_fwd"
        ev = None
        if events is not None:  # (measurement: CUDA events around the launch)
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
        nat.check(
            getattr(nat.lib(), fn)(
                ctypes.byref(self.cam), ctypes.byref(sp), img.data_ptr(),
                self.t_final.data_ptr() if track else None, self.n_contrib.data_ptr() if track else None,
                nat.ptr(target, "target"), nat.ptr(l1_sum, "l1_sum"), nat.stream(),
            ),
            fn,
        )
        if ev is not None:
            ev[1].record()
            events.append(ev)
        self.has_forward = track
        self.fwd_image = img  # the image the backward (fused L1, replay restarts) reads

    def train_pair(self, target: torch.Tensor, l1_sum: torch.Tensor, grad_acc: torch.Tensor, l1_scale: float,
                   events: list | None = None) -> None:
        """K3 + K4a of a training iteration with the fused L1 objective
        (``xg_composite_train_pair``): the tracking forward into the frame's
        image / t_final / n_contrib / checkpoints and the reverse replay into
        ``grad_acc``, the replay overlapping the forward's tail.  Follow with
        ``backward(..., replay_done=True)`` for the chain rule."""
        if self.replay_ckpt is None:
            self._alloc_replay()
        sp = self.splats_struct()
        ev = None
        if events is not None:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
        nat.check(
            nat.lib().xg_composite_train_pair(
                ctypes.byref(self.cam), ctypes.byref(sp), self.image.data_ptr(), self.t_final.data_ptr(),
                self.n_contrib.data_ptr(), nat.ptr(target, "target"), nat.ptr(l1_sum, "l1_sum"),
                ctypes.c_float(l1_scale), grad_acc.data_ptr(), nat.stream(),
            ),
            "xg_composite_train_pair",
        )
        if ev is not None:
            ev[1].record()
            events.append(ev)
        self.has_forward = True
        self.fwd_image = self.image

    @property
    def l1_sum(self) -> torch.Tensor:
        """The forward's fused-L1 accumulator: a float64 view of counters
        words 8-9, zeroed by every xg_preprocess_fwd (no clearing launch)."""
        return self.counters[nat.XG_CTR_L1 : nat.XG_CTR_L1 + 2].view(torch.float64)

    def read_counters(self) -> tuple[int, int, int]:
        c = self.counters.cpu().numpy().astype("int64") & 0xFFFFFFFF
        self.last_counters = c
        return int(c[nat.XG_CTR_ACTIVE]), int(c[nat.XG_CTR_ENTRIES]), int(c[nat.XG_CTR_STATUS])

    def bin_async(self) -> None:
        """bin(), then an asynchronous copy of the counters to pinned host
        memory; ``finish_bin`` waits for it.  Lets a caller queue the
        forward (which skips itself on the device after an entry overflow)
        before the host reads the entry count - no GPU idle at the sync."""
        self.bin()
        if getattr(self, "_cnt_host", None) is None:
            self._cnt_host = torch.empty(self.counters.shape, dtype=self.counters.dtype, pin_memory=True)
            self._cnt_event = torch.cuda.Event()
        self._cnt_host.copy_(self.counters, non_blocking=True)
        self._cnt_event.record()

    def finish_bin(self) -> bool:
        """Wait for ``bin_async``'s counters (kept in ``last_counters``); on an
        entry-buffer overflow re-bin with the exact capacity and return True -
        work queued in between saw the overflow flag and did nothing, so the
        caller re-runs it."""
        self._cnt_event.synchronize()
        c = self._cnt_host.numpy().astype("int64") & 0xFFFFFFFF
        self.last_counters = c
        entries, status = int(c[nat.XG_CTR_ENTRIES]), int(c[nat.XG_CTR_STATUS])
        if entries <= self.entry_capacity:
            return False
        self.set_capacity(int(entries * 1.25) + 1024)
        self.counters[nat.XG_CTR_STATUS] = status & ~nat.XG_ST_ENTRY_OVERFLOW
        self.bin()
        self.read_counters()
        return True

    def ensure_binned(self, check_status: bool = True) -> tuple[int, int, int]:
        """bin(), then one sync to read (active, entries, status); re-bin with
        the exact capacity if the entry buffer overflowed.  All eight
        counters read are kept in ``last_counters``."""
        self.bin()
        active, entries, status = self.read_counters()
        if check_status:
            nat.raise_for_status(status & ~nat.XG_ST_ENTRY_OVERFLOW)
        if entries > self.entry_capacity:
            self.set_capacity(int(entries * 1.25) + 1024)
            self.counters[nat.XG_CTR_STATUS] = status & ~nat.XG_ST_ENTRY_OVERFLOW
            self.bin()
            active, entries, status = self.read_counters()
        return active, entries, status

    def backward(self, cloud, grad_acc: torch.Tensor, grads_flat: torch.Tensor, screen_norms, visible,
                 dl_dimage: torch.Tensor | None = None, target: torch.Tensor | None = None,
                 l1_scale: float = 0.0, stats=None, kernel_grads=None, reproducible: bool = False,
                 events: list | None = None, replay_done: bool = False) -> None:
        """K4a + K4b.  ``grad_acc`` ([N, 8] float32 scratch) is zeroed by the
        library (xg_composite_bwd) or fully written (reproducible mode).
        ``reproducible`` sums each splat's per-entry gradient
        records in a fixed order (xg_composite_bwd_entries +
        xg_reduce_entry_grads) instead of with float atomics, so the result
        is identical run to run (the reference's single-threaded backward
        is); it needs this frame's tracking forward (checkpointed replay).
        ``events`` (measurement) receives a (start, end) pair of CUDA events
        recorded around the reverse-composite launch."""
        sp = self.splats_struct()
        args = (ctypes.byref(self.cam), ctypes.byref(sp), self.t_final.data_ptr(), self.n_contrib.data_ptr(),
                nat.ptr(dl_dimage, "dl_dimage"), self.fwd_image.data_ptr(),
                nat.ptr(target, "target") if dl_dimage is None else None, ctypes.c_float(l1_scale))
        if replay_done:  # (train_pair ran the reverse replay into grad_acc)
            pass
        elif reproducible:
            nb = int(nat.lib().xg_entry_grad_bytes(self.n, self.entry_capacity))
            if self.entry_grad is None or self.entry_grad.numel() < nb:
                self.entry_grad = torch.empty(nb, dtype=torch.uint8, device=self.device)
            ws = (self.entry_grad.data_ptr(), self.entry_grad.numel())
            nat.check(nat.lib().xg_composite_bwd_entries(*args, *ws, nat.stream()), "xg_composite_bwd_entries")
            nat.check(nat.lib().xg_reduce_entry_grads(ctypes.byref(self.cam), ctypes.byref(sp), *ws,
                                                      grad_acc.data_ptr(), nat.stream()), "xg_reduce_entry_grads")
        else:
            ev = None
            if events is not None:
                ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                ev[0].record()
            nat.check(nat.lib().xg_composite_bwd(*args, grad_acc.data_ptr(), nat.stream()), "xg_composite_bwd")
            if ev is not None:
                ev[1].record()
                events.append(ev)
        cs = nat.cloud_struct(cloud)
        ns = oc = wg = None
        if stats is not None:
            ns, oc, wg = stats.norm_sum.data_ptr(), stats.obs_count.data_ptr(), stats.world_grad_sum.data_ptr()
        km = kc = ki = ka = None
        if kernel_grads is not None:
            km, kc, ki, ka = (kernel_grads[k].data_ptr() for k in ("g_mean", "g_conic", "g_int", "g_alpha"))
        nat.check(
            nat.lib().xg_preprocess_bwd(
                ctypes.byref(cs), ctypes.byref(self.cam), ctypes.byref(sp), grad_acc.data_ptr(),
                grads_flat.data_ptr(), nat.ptr(screen_norms), nat.ptr(visible), ns, oc, wg, km, kc, ki,
                ka, nat.stream(),
            ),
            "xg_preprocess_bwd",
        )
