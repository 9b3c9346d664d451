"""Novel-view inference: render a sweep of cone-beam views, sync-free.

The reference renders views one at a time through ``render_view``
(``frontend.py:236-242``, ``cli.py:125-143``, ``trainer.py:284-315``).  Here a
sweep is enqueued on S CUDA streams (one ``Frame`` of buffers per stream,
round-robin over views), so the latency-bound binning kernels of one view
overlap the compositing of another; no host synchronisation happens until
the end of the sweep.  Entry buffers are sized from a probe of the first
view; per-view overflow bits are collected on the device and any
overflowed view is re-rendered with an exact-size buffer afterwards.

Multi-GPU: views are independent, so ``shard_angles`` splits a sweep over
ranks with no collective (see ``parallel.py``).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _native as nat
from .engine import Frame
from .gaussians import GaussianCloud
from .geometry import ScannerConfig, XgCamera, camera_pod, extrinsic_from_angle, intrinsic_from_config


class SweepRenderer:
    """Reusable multi-stream renderer for one cloud and one detector.

    ``batch == 1``: view i runs preprocess -> bin -> composite on stream
    i % n_streams (one ``Frame`` per stream), so the binning of later views
    overlaps the compositing of earlier ones.

    ``batch == K > 1``: K views are binned concurrently on K streams into one
    of two frame sets, then composited by ONE ``xg_composite_fwd_batch``
    launch over all their units (one heaviest-first queue, no per-view tail)
    on a composite stream, while the next K views are binned into the other
    set."""

    def __init__(self, cloud: GaussianCloud, scanner: ScannerConfig, n_streams: int = 3,
                 capacity_factor: float = 1.3, batch: int = 1):
        nat.require_cuda(cloud.flat, "cloud")
        self.cloud = cloud
        self.scanner = scanner
        self.h, self.w = scanner.detector_height, scanner.detector_width
        self.intr = intrinsic_from_config(scanner)
        self.batch = int(batch)
        if not 1 <= self.batch <= nat.XG_MAX_BATCH:
            raise ValueError(f"batch must be in [1, {nat.XG_MAX_BATCH}]")
        n = self.batch if self.batch > 1 else max(1, n_streams)
        # (high-priority binning streams measured 1-3 % slower: XG_BIN_PRIORITY=1)
        prio = -1 if (self.batch > 1 and os.environ.get("XG_BIN_PRIORITY", "0") == "1") else 0
        self.streams = [torch.cuda.Stream(device=cloud.device, priority=prio) for _ in range(n)]
        self.comp_stream = torch.cuda.Stream(device=cloud.device) if self.batch > 1 else None
        # device -> host image copies (host_out) on their own stream, so a copy
        # never holds up the next compositing launch or binning on its stream
        self.copy_stream = torch.cuda.Stream(device=cloud.device)
        self.capacity_factor = capacity_factor
        self.frames: list[Frame] = []
        self.capacity = 0
        self.kernel_launches = 0
        self._batch_ws = None

    def _probe_capacity(self, phi: float) -> int:
        fr = Frame(self.cloud.n_points, self.h, self.w, self.cloud.device)
        fr.preprocess(self.cloud, self.camera(phi))
        _, entries, status = fr.ensure_binned()
        nat.raise_for_status(status & ~nat.XG_ST_ENTRY_OVERFLOW)
        return int(entries * self.capacity_factor) + 4096

    def camera(self, phi: float):
        return camera_pod(extrinsic_from_angle(self.scanner, float(phi)), self.intr, (self.h, self.w))

    def prepare(self, angles) -> None:
        angles = np.atleast_1d(np.asarray(angles, dtype=np.float64))
        if not self.frames or self.capacity == 0:
            # (after an overflow finish() dropped the frames: keep the grown capacity)
            self.capacity = max(self.capacity, self._probe_capacity(float(angles[0])))
            n = 2 * self.batch if self.batch > 1 else len(self.streams)
            self.frames = [Frame(self.cloud.n_points, self.h, self.w, self.cloud.device,
                                 entry_capacity=self.capacity) for _ in range(n)]
        if self.batch > 1 and self._batch_ws is None:
            cam = self.camera(float(angles[0]))
            nb = nat.lib().xg_composite_batch_workspace_bytes(ctypes.byref(cam), self.batch)
            self._batch_ws = torch.empty(int(nb), dtype=torch.uint8, device=self.cloud.device)

    def render(self, angles, out: torch.Tensor | None = None, host_out: torch.Tensor | None = None,
               check: bool = True, composite_events: list | None = None) -> torch.Tensor:
        """Render every angle into ``out`` ([V, H, W] float32 on the device).
        If ``host_out`` (pinned [V, H, W]) is given, each image is also copied
        to it asynchronously.  ``composite_events`` collects (start, end, views)
        CUDA events around every compositing launch, recorded on the stream
        it runs on."""
        angles = np.atleast_1d(np.asarray(angles, dtype=np.float64))
        v = angles.shape[0]
        self.prepare(angles)
        if out is None:
            out = torch.empty((v, self.h, self.w), dtype=torch.float32, device=self.cloud.device)
        status = torch.zeros(v, dtype=torch.int32, device=self.cloud.device)
        # the intensities are view-independent (isotropic RIRF): once per sweep
        # (raises for non-finite features, as the per-view check would)
        self._inten = nat.intensities(self.cloud)
        # likewise the covariance / opacity terms of the projection
        self._inv = nat.view_invariants(self.cloud)
        if self.batch > 1:
            self._render_batched(angles, out, host_out, status, composite_events)
        else:
            self._render_streams(angles, out, host_out, status, composite_events)
        self.last_status = status  # per-view status words (device), e.g. to count overflows after check=False
        if check:
            self.finish(angles, out, host_out, status)
        return out

    def _render_streams(self, angles, out, host_out, status, composite_events) -> None:
        main = torch.cuda.current_stream()
        for s in self.streams + [self.copy_stream]:
            s.wait_stream(main)
        for i, phi in enumerate(angles):
            k = i % len(self.streams)
            st, fr = self.streams[k], self.frames[k]
            with torch.cuda.stream(st):
                fr.preprocess(self.cloud, self.camera(phi), self._inten, self._inv)
                fr.bin()
                if composite_events is not None:
                    a = torch.cuda.Event(enable_timing=True)
                    b = torch.cuda.Event(enable_timing=True)
                    a.record(st)
                    fr.composite(image_out=out[i], track=False)
                    b.record(st)
                    composite_events.append((a, b, 1))
                else:
                    fr.composite(image_out=out[i], track=False)
                # (a kernel, not copy_: a 4-byte cudaMemcpy would queue on the copy
                # engine behind the previous view's image download)
                torch.add(fr.counters[nat.XG_CTR_STATUS : nat.XG_CTR_STATUS + 1], 0, out=status[i : i + 1])
            if host_out is not None:
                self.copy_stream.wait_stream(st)
                with torch.cuda.stream(self.copy_stream):
                    host_out[i].copy_(out[i], non_blocking=True)
        for s in self.streams + [self.copy_stream]:
            main.wait_stream(s)
        self.kernel_launches = len(angles)

    def _render_batched(self, angles, out, host_out, status, composite_events) -> None:
        main = torch.cuda.current_stream()
        cs, K = self.comp_stream, self.batch
        for s in self.streams + [cs, self.copy_stream]:
            s.wait_stream(main)
        done = [None, None]  # composite-finished event per frame set
        pending = None  # (lo, hi) of the last batch whose images are not downloaded yet
        lib = nat.lib()
        for j, lo in enumerate(range(0, len(angles), K)):
            hi = min(lo + K, len(angles))
            fs = self.frames[(j % 2) * K:(j % 2) * K + K]
            for i in range(lo, hi):
                st, fr = self.streams[i - lo], fs[i - lo]
                with torch.cuda.stream(st):
                    if done[j % 2] is not None:
                        st.wait_event(done[j % 2])  # the set's previous composite read these buffers
                    fr.preprocess(self.cloud, self.camera(angles[i]), self._inten, self._inv)
                    fr.bin()
                cs.wait_stream(st)
            nv = hi - lo
            cams = (XgCamera * nv)(*[fs[i].cam for i in range(nv)])
            sps = (nat.XgSplats * nv)(*[fs[i].splats_struct() for i in range(nv)])
            imgs = (ctypes.c_void_p * nv)(*[out[lo + i].data_ptr() for i in range(nv)])
            with torch.cuda.stream(cs):
                if host_out is not None and pending is not None:
                    # the previous batch's download starts with this
                    # compositing launch (not in the binning phase before it,
                    # whose L2-resident working set the DMA would evict)
                    started = torch.cuda.Event()
                    started.record(cs)
                    self.copy_stream.wait_event(started)
                    with torch.cuda.stream(self.copy_stream):
                        host_out[pending[0]:pending[1]].copy_(out[pending[0]:pending[1]], non_blocking=True)
                    pending = None
                a = b = None
                if composite_events is not None:
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(cs)
                nat.check(lib.xg_composite_fwd_batch(cams, sps, imgs, nv, self._batch_ws.data_ptr(),
                                                     self._batch_ws.numel(), nat.stream()), "xg_composite_fwd_batch")
                if b is not None:
                    b.record(cs)
                    composite_events.append((a, b, nv))
                # the views' status words in one cat kernel (a 4-byte cudaMemcpy per
                # view would queue on the copy engine behind the image downloads
                # and hold up this stream's next compositing launch)
                torch.cat([fs[i].counters[nat.XG_CTR_STATUS : nat.XG_CTR_STATUS + 1] for i in range(nv)],
                          out=status[lo:hi])
                ev = torch.cuda.Event()
                ev.record(cs)
                done[j % 2] = ev
            if host_out is not None:
                pending = (lo, hi)  # downloaded once the next launch starts (or after the loop)
        if host_out is not None and pending is not None:
            self.copy_stream.wait_stream(cs)
            with torch.cuda.stream(self.copy_stream):
                host_out[pending[0]:pending[1]].copy_(out[pending[0]:pending[1]], non_blocking=True)
        for s in self.streams + [cs, self.copy_stream]:
            main.wait_stream(s)
        self.kernel_launches = (len(angles) + K - 1) // K

    def finish(self, angles, out, host_out, status: torch.Tensor) -> None:
        st = status.cpu().numpy().astype(np.int64) & 0xFFFFFFFF
        for word in st:
            nat.raise_for_status(int(word) & ~nat.XG_ST_ENTRY_OVERFLOW)
        bad = np.flatnonzero(st & nat.XG_ST_ENTRY_OVERFLOW)
        for i in bad:  # rare: exact-size re-render of overflowed views
            fr = Frame(self.cloud.n_points, self.h, self.w, self.cloud.device,
                       entry_capacity=self.capacity)
            fr.preprocess(self.cloud, self.camera(float(angles[i])))
            fr.ensure_binned()
            fr.composite(image_out=out[i])
            self.capacity = max(self.capacity, fr.entry_capacity)
            if host_out is not None:
                host_out[i].copy_(out[i])
        if bad.size:
            self.frames = []  # grow all frames on the next sweep


def render_sweep(cloud: GaussianCloud, scanner: ScannerConfig, angles=None, n_streams: int = 3,
                 batch: int = 12) -> torch.Tensor:
    """Render ``angles`` (default: the scanner's) into a [V, H, W] device
    stack (batches of ``batch`` views per compositing launch)."""
    if angles is None:
        angles = scanner.angles
    n = np.atleast_1d(angles).size
    return SweepRenderer(cloud, scanner, n_streams, batch=max(1, min(batch, n))).render(angles)
