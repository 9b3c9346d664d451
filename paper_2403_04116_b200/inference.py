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

import os

import numpy as np
import torch

from . import _native as nat
from .engine import Frame
from .gaussians import GaussianCloud
from .geometry import ScannerConfig, camera_pod, extrinsic_from_angle, intrinsic_from_config


class SweepRenderer:
    """Reusable multi-stream renderer for one cloud and one detector."""

    def __init__(self, cloud: GaussianCloud, scanner: ScannerConfig, n_streams: int = 3,
                 capacity_factor: float = 1.3, priority_composite: bool | None = None):
        nat.require_cuda(cloud.flat, "cloud")
        self.cloud = cloud
        self.scanner = scanner
        self.h, self.w = scanner.detector_height, scanner.detector_width
        self.intr = intrinsic_from_config(scanner)
        self.streams = [torch.cuda.Stream(device=cloud.device) for _ in range(max(1, n_streams))]
        if priority_composite is None:
            priority_composite = os.environ.get("XG_PRIORITY_COMPOSITE", "0") == "1"
        # optional: compositing on high-priority streams, so the binning of the
        # next views only fills the SMs the persistent composite leaves idle
        self.comp_streams = ([torch.cuda.Stream(device=cloud.device, priority=-1) for _ in self.streams]
                             if priority_composite else None)
        self.capacity_factor = capacity_factor
        self.frames: list[Frame] = []
        self.capacity = 0
        self.kernel_launches = 0

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
            self.capacity = self._probe_capacity(float(angles[0]))
            self.frames = [Frame(self.cloud.n_points, self.h, self.w, self.cloud.device,
                                 entry_capacity=self.capacity) for _ in self.streams]

    def render(self, angles, out: torch.Tensor | None = None, host_out: torch.Tensor | None = None,
               check: bool = True, composite_events: list | None = None) -> torch.Tensor:
        """Render every angle into ``out`` ([V, H, W] float32 on the device).
        If ``host_out`` (pinned [V, H, W]) is given, each image is also copied
        to it asynchronously on the view's stream.  ``composite_events``
        collects (start, end) CUDA events around every compositing launch,
        recorded on the stream it runs on."""
        angles = np.atleast_1d(np.asarray(angles, dtype=np.float64))
        v = angles.shape[0]
        self.prepare(angles)
        if out is None:
            out = torch.empty((v, self.h, self.w), dtype=torch.float32, device=self.cloud.device)
        status = torch.zeros(v, dtype=torch.int32, device=self.cloud.device)
        main = torch.cuda.current_stream()
        for s in self.streams:
            s.wait_stream(main)
        launches = 0
        if self.comp_streams is not None:
            for s in self.comp_streams:
                s.wait_stream(main)
        for i, phi in enumerate(angles):
            k = i % len(self.streams)
            st, fr = self.streams[k], self.frames[k]
            with torch.cuda.stream(st):
                if self.comp_streams is not None:
                    st.wait_stream(self.comp_streams[k])  # the frame's previous composite is done
                fr.preprocess(self.cloud, self.camera(phi))
                fr.bin()
            if self.comp_streams is not None:
                self.comp_streams[k].wait_stream(st)
                st = self.comp_streams[k]
            with torch.cuda.stream(st):
                if composite_events is not None:
                    a = torch.cuda.Event(enable_timing=True)
                    b = torch.cuda.Event(enable_timing=True)
                    a.record(st)
                    fr.composite(image_out=out[i], track=False)
                    b.record(st)
                    composite_events.append((a, b))
                else:
                    fr.composite(image_out=out[i], track=False)
                status[i : i + 1].copy_(fr.counters[nat.XG_CTR_STATUS : nat.XG_CTR_STATUS + 1])
                if host_out is not None:
                    host_out[i].copy_(out[i], non_blocking=True)
            launches += 1
        for s in self.streams + (self.comp_streams or []):
            main.wait_stream(s)
        self.kernel_launches = launches
        if check:
            self.finish(angles, out, host_out, status)
        return out

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


def render_sweep(cloud: GaussianCloud, scanner: ScannerConfig, angles=None, n_streams: int = 3) -> torch.Tensor:
    """Render ``angles`` (default: the scanner's) into a [V, H, W] device stack."""
    if angles is None:
        angles = scanner.angles
    return SweepRenderer(cloud, scanner, n_streams).render(angles)
