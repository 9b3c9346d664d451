"""Benchmark of the DRR hot path (BASELINE.json metric).

Default workload (N=1): C3 of BASELINE.json - 493,039 ACUI Gaussians
(cuboid G=152, interval 2, 16 features, seed 0), 512x512 cone-beam
detector (L_SO 1000, L_SD 1500, pitch 192/512 mm), a 360-view novel-view
sweep over [0, pi).  One "step" = one 360-view sweep.  Multi-GPU (torchrun)
shards views with no collective on the data path: by default the 360 views
round-robin over the N ranks (strong scaling, BASELINE configs[2]);
``--scaling weak`` gives every rank its own 360-view sweep offset by r/N of
the 0.5 degree step.  Under N > 1 the other mode is reported as well.

Further blocks on the same line: ``fwdbwd_c1`` (C1: 50k Gaussians, 256^2
forward + backward), ``stress_c4`` (C4: 1M Gaussians at 1024^2) and
``train_c2`` (C2: full training iterations; ``train_c5`` data-parallel under
torchrun), each with its roofline and, on rank 0 at N = 1, the reference's
CPU path timed in the same run.

Contract: ``python bench.py --gpus N --steps K --warmup W`` prints ONE JSON
line (rank 0); ``--impl reference`` times the reference's own CPU
implementation (xsplat built into oracle/_ref, else the oracle C port) on
the host cores for the same metric.  See DESIGN.md (Measurement).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

# (before CUDA initialises: 32 hardware work queues for the sweep's ~14
# streams - the package sets the same default on import)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "fps (512x512 cone-beam projections/s), 500k Gaussians"
VIEWS = 360
G_C3, DET = 152, 512
L_SO, L_SD = 1000.0, 1500.0
FLOP_PER_PAIR = 17  # forward composite FLOP per traversed (pixel, entry) pair


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--streams", type=int, default=4)
    ap.add_argument("--batch", type=int, default=12,  # measured: 8 -> 12 views per launch +3.5 % (C3)
                    help="views per compositing launch (xg_composite_fwd_batch); 1: one launch per view on "
                         "--streams streams")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-views", type=int, default=0, help="0 = one per worker")
    ap.add_argument("--no-train", action="store_true", help="skip the C2 training-iteration block")
    ap.add_argument("--train-iters-per-step", type=int, default=200)  # 5 steps: 1,000 timed iterations
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 (1M Gaussians, 1024^2) stress block")
    ap.add_argument("--no-c1", action="store_true", help="skip the C1 (50k Gaussians, 256^2 fwd+bwd) block")
    ap.add_argument("--no-c5", action="store_true", help="N = 1: skip the C5-size (493k) training block")
    ap.add_argument("--collective", choices=("nccl", "p2p"), default="nccl",
                    help="C5 data-parallel gradient step: bucketed NCCL all-reduce + fused Adam, or the peer-memory "
                         "reduce-scatter / all-gather-Adam kernels (parallel.PeerExchange, csrc/xg_dp.cu)")
    ap.add_argument("--scaling", choices=("strong", "weak"), default="strong",
                    help="C3 under N GPUs: the 360-view sweep sharded over them (strong, BASELINE configs[2]) "
                         "or 360 views per GPU (weak)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def sweep_angles(rank: int, world: int) -> np.ndarray:
    return (np.arange(VIEWS, dtype=np.float64) + rank / max(world, 1)) * (np.pi / VIEWS)


G_C2 = 88


def phantom_dataset(g: int, scanner):
    """Training targets exactly as the reference's pipeline makes them
    (cli.py:60-72): the default phantom primitives voxelised on
    the G^3 grid of the 100 mm ACUI cuboid, cone-beam projected at every
    angle (GPU projector, phantom.py:190-250), normalised by the global max
    and given 3 % Gaussian noise (seed 0).  Returns (dataset, seconds)."""
    import torch

    from paper_2403_04116_b200.dataset import add_noise, make_projection_set
    from paper_2403_04116_b200.phantom import default_phantom_primitives, make_phantom

    extent = np.full(3, 100.0)
    t0 = time.perf_counter()
    ph = make_phantom(default_phantom_primitives(extent), (g, g, g), extent / g)
    ds = add_noise(make_projection_set(ph, scanner), 0.03, 0)
    torch.cuda.synchronize()
    return ds, time.perf_counter() - t0


def c3_arrays():
    from paper_2403_04116_b200 import acui

    return acui.init_alternative_arrays("cuboid", acui.benchmark_spec(G_C3), 16, 0)


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._thr = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._thr = threading.Thread(target=self._run, daemon=True)
        self._thr.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._thr:
            self._thr.join(timeout=10)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 4 + i and s[4 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU baseline: the reference itself on the host cores
# ---------------------------------------------------------------------------
def _ref_available() -> bool:
    return (ROOT / "oracle" / "_ref" / "xsplat" / "rasterizer").is_dir()


_CPU_STATE = {}
G_C1, DET_C1 = 68, 256


def _cpu_init(kind: str, case: str = "C3", target=None):
    """Worker initializer: the case's float32-rounded ACUI cloud in the
    reference's (or the oracle port's) form, built once per process."""
    os.environ["OMP_NUM_THREADS"] = "1"
    from paper_2403_04116_b200 import acui

    g, det = {"C1": (G_C1, DET_C1), "C2": (G_C2, DET), "C3": (G_C3, DET), "C4": (G_C4, DET_C4)}[case]
    arrs = acui.init_alternative_arrays("cuboid", acui.benchmark_spec(g), 16, 0)
    _CPU_STATE.update(kind=kind, case=case, det=det, target=target)
    if kind == "reference":
        sys.path.insert(0, str(ROOT / "oracle" / "_ref"))
        from xsplat.gaussians import GaussianCloud
        from xsplat.geometry import ScannerConfig
        from xsplat.rasterizer import set_backend

        set_backend("compiled")
        f32 = {k: np.asarray(v, np.float32).astype(np.float64) for k, v in arrs.items()}
        _CPU_STATE["cloud"] = GaussianCloud(**f32)
        _CPU_STATE["scanner"] = ScannerConfig(L_SO, L_SD, det, det, 192.0 / det)
    else:
        _CPU_STATE["fields"] = {k: np.asarray(v, np.float32) for k, v in arrs.items()}


def _cpu_unit(phi: float) -> float:
    """One unit of the case's work on the host, timed: C3/C4 one view
    (render_view, frontend.py:236-242), C1 one forward + backward with
    dL/dI ~ N(0,1)/HW (render + render_backward, backward.py:21-124), C2 one
    full training iteration (render, loss, render_backward, DensifyStats,
    adam_step: trainer.py:372-387)."""
    st = _CPU_STATE
    det, case = st["det"], st["case"]
    t0 = time.perf_counter()
    if st["kind"] == "reference":
        from xsplat.rasterizer import render_backward, render_view

        proj, sp = render_view(st["cloud"], st["scanner"], phi)
        if case == "C1":
            render_backward(st["cloud"], sp, np.random.default_rng(0).normal(size=(det, det)) / det**2)
        elif case == "C2":
            from xsplat.trainer import DensifyStats, OptimizerState, TrainConfig, adam_step, loss

            if "opt" not in st:
                st["opt"] = (OptimizerState(st["cloud"]), DensifyStats.zeros(st["cloud"].n_points), TrainConfig())
            state, stats, cfg = st["opt"]
            _, dl = loss(proj, st["target"], cfg.gamma)
            grads = render_backward(st["cloud"], sp, dl)
            stats.accumulate(grads)
            lr = {"positions": cfg.lr_position_init, "rotations": cfg.lr_rotation, "log_scales": cfg.lr_scaling,
                  "raw_opacities": cfg.lr_opacity, "features": cfg.lr_feature}
            adam_step(st["cloud"], grads, state, lr, cfg)
    else:
        from oracle import oracle as orc

        cam = orc.camera_from_view(L_SO, L_SD, det, det, 192.0 / det, phi)
        r = orc.render(st["fields"], np.ones(16, np.float32), cam)
        if case in ("C1", "C2"):
            dl = np.random.default_rng(0).normal(size=(det, det)) / det**2
            if case == "C2":
                dl = orc.l1_loss(r["image"], st["target"])[1]
            kg = orc.composite_bwd(r["pre"], r["bin"], det, det, dl)
            orc.preprocess_bwd(st["fields"], np.ones(16, np.float32), cam, r["pre"], kg)
    return time.perf_counter() - t0


GB_PER_PROCESS = {"C1": 1.0, "C2": 3.0, "C3": 3.0, "C4": 8.0}  # peak resident set of one reference process


def cpu_workers(case: str = "C3", cap: int | None = None) -> int:
    n = os.cpu_count() or 1
    try:
        import psutil

        mem = psutil.virtual_memory().available
        n = min(n, max(1, int(mem // (GB_PER_PROCESS[case] * 2**30))))
    except Exception:
        pass
    return max(1, min(n, cap or 64))


def cpu_pool(kind: str, workers: int, case: str = "C3", target=None):
    import multiprocessing as mp

    ctx = mp.get_context("fork")
    return ctx.Pool(workers, initializer=_cpu_init, initargs=(kind, case, target))


UNIT = {"C1": ("fwd+bwd/s", "forward + backward of one 256x256 view (dL/dI ~ N(0,1)/HW)"),
        "C2": ("iters/s", "full training iteration at 512x512 (render, L1, backward, stats, Adam)"),
        "C3": ("fps", "one 512x512 view (render_view)"), "C4": ("fps", "one 1024x1024 view (render_view)")}


def cpu_baseline(case: str = "C3", units: int | None = None, target=None, angles=None) -> dict:
    """The reference itself (xsplat, compiled backend, oracle/_ref) - or the
    oracle C port where it is absent - on the host cores, timed in the same
    run: one unit of the case's work per worker process (the reference is
    single-threaded, cli.py:4-7), all workers at once; value = units / wall."""
    kind = "reference" if _ref_available() else "port"
    if case == "C2" and kind != "reference":
        return {"value": None, "unit": UNIT[case][0], "kind": kind, "note": "needs the reference (oracle/_ref)"}
    workers = cpu_workers(case, units)
    nv = units or workers
    if angles is None:
        angles = (np.arange(nv) * (np.pi / max(nv, 1)) + 0.7) % np.pi
    with cpu_pool(kind, workers, case, target) as pool:
        t0 = time.perf_counter()
        per = pool.map(_cpu_unit, [float(a) for a in angles[:nv]], chunksize=1)
        wall = time.perf_counter() - t0
    src = "xsplat compiled backend" if kind == "reference" else "oracle C port"
    return {"value": nv / wall, "unit": UNIT[case][0], "cores": workers, "kind": kind,
            "sample": f"{nv} x {UNIT[case][1]} ({src}, 1 unit per process, {workers} processes, "
                      f"OMP_NUM_THREADS=1; one unit {np.median(per):.1f} s median)",
            "unit_s_median": float(np.median(per))}


def run_reference(args) -> None:
    rank, world, _ = dist_env()
    if rank != 0:
        return
    kind = "reference" if _ref_available() else "port"
    workers = cpu_workers("C3")
    with cpu_pool(kind, workers, "C3") as pool:
        angles = [float(a) for a in sweep_angles(0, 1)[:: max(1, VIEWS // workers)][:workers]]
        for _ in range(args.warmup):
            pool.map(_cpu_unit, angles, chunksize=1)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            pool.map(_cpu_unit, angles, chunksize=1)
        wall = time.perf_counter() - t0
    value = len(angles) * args.steps / wall
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "fps", "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic ACUI cuboid cloud (seed 0), analytic cone-beam cameras",
        "config": {"workload": "C3: 493,039 Gaussians, 512x512, novel-view sweep (each step: one view per "
                               f"host worker, {len(angles)} views)", "views_per_step": len(angles)},
        "cpu_baseline": {"value": value, "unit": "fps", "cores": workers, "kind": kind,
                         "sample": f"{len(angles)} views per step, 1 view per process"},
        "e2e": {"value": value, "unit": "fps", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def fp32_peak() -> tuple[float, str]:
    """The FP32 roofline denominator: nominal 148 SM x 128 FP32 lanes x 2 FLOP
    x 1.965 GHz = 74.45 TFLOP/s (MEASURED_PEAKS.json and the profiling guide
    carry only HBM and bf16; nothing on this path is a contraction).  The
    pool's measured FFMA probe (profiles/fp32_peak.json, 72.5) is reported
    beside it as ``frac_of_measured_ffma``."""
    return 74.45, "nominal FP32: 148 SM x 128 lanes x 2 FLOP x 1.965 GHz (no driver-measured FP32 peak)"


def ffma_probe() -> float | None:
    p = ROOT / "profiles" / "fp32_peak.json"
    return float(json.loads(p.read_text())["fp32_tflops"]) if p.exists() else None


def ncu_pipes() -> dict | None:
    """Physical pipe utilisation of the compositing launch from the committed
    ncu capture (profiles/ncu_composite_fwd.json): the hardware-efficiency
    figure next to the algorithmic-work fraction."""
    p = ROOT / "profiles" / "ncu_composite_fwd.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    return {k: d[k] for k in ("fma_pipe_pct", "xu_pipe_pct", "issue_active_pct", "source") if k in d} or None


def hbm_peak() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (driver-measured copy)"
    return 7700.0, "nominal B200 HBM3e (no MEASURED_PEAKS.json)"


def dram_traffic_per_view(batched: bool) -> float | None:
    """DRAM bytes per composited view from the committed ncu capture."""
    p = ROOT / "profiles" / "ncu_composite_fwd.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["dram_bytes_per_view_batched" if batched else "dram_bytes_per_view_single"])
    return None


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    # XG_BENCH_SHARE_GPU=1 (test aid): ranks share the visible GPUs round-robin
    # and talk over gloo - exercises the multi-rank code path on one GPU;
    # its numbers are not a measurement.
    share = os.environ.get("XG_BENCH_SHARE_GPU") == "1"
    if share:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            # NCCL's communicator-init INFO lines (rank 0, to stderr: stdout
            # carries only the JSON line) - the record of nranks / transports
            if rank == 0:
                os.environ.setdefault("NCCL_DEBUG", "INFO")
                os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
                os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            t = torch.ones(1, device="cuda")
            dist.all_reduce(t)  # (creates the communicator now, so the INFO lines precede the run)
    from paper_2403_04116_b200 import _native, geometry
    from paper_2403_04116_b200.gaussians import GaussianCloud
    from paper_2403_04116_b200.inference import SweepRenderer

    arrs = c3_arrays()
    cloud = GaussianCloud(**arrs, device="cuda")
    sc = geometry.ScannerConfig(L_SO, L_SD, DET, DET, 192.0 / DET)
    # strong scaling (default, BASELINE configs[2]: the 360 views sharded
    # over the N GPUs) or weak (360 views per GPU, offset by r/N of a step)
    from paper_2403_04116_b200.parallel import shard_angles

    def angles_for(mode: str):
        return shard_angles(sweep_angles(0, 1), rank, world) if mode == "strong" else sweep_angles(rank, world)

    angles = angles_for(args.scaling)
    nloc = len(angles)
    rend = SweepRenderer(cloud, sc, n_streams=args.streams, batch=args.batch)
    out = torch.empty((VIEWS, DET, DET), dtype=torch.float32, device="cuda")
    host = torch.empty((VIEWS, DET, DET), dtype=torch.float32, pin_memory=True)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, k) -> float:
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k):
            fn()
        e1.record()
        barrier()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    # work units (untimed): traversed (pixel, entry) pairs per view, from the
    # engine's own per-pixel outputs: n_traversed = n_contrib if the pixel
    # terminated (T_final < 1e-4) else the tile's entry count.
    from paper_2403_04116_b200.engine import Frame

    fr = Frame(cloud.n_points, DET, DET, "cuda")
    traversed = []
    comp_iso = []
    ntx = (DET + 15) // 16
    yy, xx = np.meshgrid(np.arange(DET), np.arange(DET), indexing="ij")
    tile_of = torch.as_tensor((yy // 16) * ntx + xx // 16, device="cuda")
    for phi in angles[:: max(1, VIEWS // 36)]:
        fr.preprocess(cloud, rend.camera(phi))
        fr.ensure_binned()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fr.composite()
        e0.record()
        fr.composite()
        e1.record()
        torch.cuda.synchronize()
        comp_iso.append(e0.elapsed_time(e1))
        lens = (fr.tile_ranges[:, 1] - fr.tile_ranges[:, 0])[tile_of]
        nt = torch.where(fr.t_final < 1e-4, fr.n_contrib.to(torch.int64), lens)
        traversed.append(float(nt.sum().item()))
    pairs_per_view = float(np.mean(traversed))

    # device-resident sweep
    for _ in range(args.warmup):
        rend.render(angles, out=out)
    launches0 = _native.kernel_launches()
    comp_events: list = []
    step_idx = [0]

    statuses: list = []

    def step():
        # composite-kernel events on their own stream during the last timed step
        ev = comp_events if step_idx[0] == args.steps - 1 else None
        step_idx[0] += 1
        rend.render(angles, out=out, check=False, composite_events=ev)
        statuses.append(rend.last_status)

    # XG_PROFILE_TIMED=1: open the CUDA profiler range around the timed
    # region only (ncu --profile-from-start off -> the launch list of exactly
    # the timed sweep; profiles/)
    prof = os.environ.get("XG_PROFILE_TIMED") == "1"
    if prof:
        torch.cuda.profiler.start()
    with ClockSampler(local) as clk:
        ms = timed(step, args.steps)
    if prof:
        torch.cuda.profiler.stop()
    launches = _native.kernel_launches() - launches0
    # per launch: a batched launch composites nv views
    comp_ctx = float(np.mean([a.elapsed_time(b) / nv for a, b, nv in comp_events]))
    launch_views = float(np.mean([nv for _, _, nv in comp_events]))
    rend.render(angles, out=out)  # status check of a full sweep
    # end to end: images to pinned host memory every view
    for _ in range(1):
        rend.render(angles, out=out, host_out=host)
    # e2e: the cloud comes from host memory too (the reference API takes a
    # host cloud), so every step re-uploads it before rendering
    cloud_host = cloud.flat.detach().cpu().pin_memory()

    def e2e_step():
        cloud.flat.copy_(cloud_host, non_blocking=True)
        rend.render(angles, out=out, host_out=host, check=False)

    ms_e2e = timed(e2e_step, args.steps)
    overflowed = count_overflows(statuses)

    # second end-to-end figure: the reference-shaped per-view call,
    # render_view(cloud, scanner, phi) (frontend.py:236-242), image read back
    # to the host after every view - what a drop-in caller's loop costs
    from paper_2403_04116_b200.rasterizer import render_view

    rv_angles = angles[:: max(1, nloc // 36)]
    # (views round-robin over streams: render_view's entry-count sync waits
    # for its own view's binning only; each image lands in its stream's
    # pinned buffer)
    rv_streams = [torch.cuda.Stream() for _ in range(RV_STREAMS)]
    img_host = [torch.empty((DET, DET), dtype=torch.float32, pin_memory=True) for _ in rv_streams]

    def rv_step():
        main = torch.cuda.current_stream()
        cloud.flat.copy_(cloud_host, non_blocking=True)
        for st in rv_streams:
            st.wait_stream(main)
        for i, a in enumerate(rv_angles):
            with torch.cuda.stream(rv_streams[i % RV_STREAMS]):
                proj, _ = render_view(cloud, sc, float(a))
                img_host[i % RV_STREAMS].copy_(proj.pixels, non_blocking=True)
        for st in rv_streams:
            main.wait_stream(st)

    rv_step()
    ms_rv = timed(rv_step, 2)
    rv_value = len(rv_angles) * 2 * world / (ms_rv / 1e3)

    # N > 1: the other sharding mode too (same kernels, other view sets)
    other = None
    if world > 1:
        omode = "weak" if args.scaling == "strong" else "strong"
        oang = angles_for(omode)
        rend.render(oang, out=out)
        ms_o = timed(lambda: rend.render(oang, out=out, check=False), args.steps)
        rend.render(oang, out=out)
        other = {"scaling": omode, "value": len(oang) * args.steps * world / (ms_o / 1e3), "unit": "fps",
                 "views_per_step_per_gpu": len(oang), "ms_per_step": ms_o / args.steps}

    total_views = nloc * args.steps * world
    value = total_views / (ms / 1e3)
    e2e_value = total_views / (ms_e2e / 1e3)
    peak, peak_note = fp32_peak()
    comp_iso_ms = float(np.mean(comp_iso))
    achieved = FLOP_PER_PAIR * pairs_per_view / (comp_ctx * 1e-3) / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": "fps", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: ACUI cuboid cloud (BASELINE C3 generator, seed 0), analytic cameras",
        "config": {"workload": "C3: 493,039 Gaussians (G=152), 512x512 detector, 360-view novel-view sweep "
                               + ("sharded over the GPUs (strong scaling: 360 views per step in total)"
                                  if args.scaling == "strong" else "per GPU per step (weak scaling)"),
                   "views_per_step_per_gpu": nloc, "streams": args.streams,
                   "l2": "inputs larger than L2 (6M-entry lists + 1 MB images per view, 360 views/step)",
                   "views_per_composite_launch": args.batch,
                   "parallelism": f"view-sharded x{world}"},
        "e2e": {"value": e2e_value, "unit": "fps",
                "h2d_bytes_per_step": 128 * nloc + 4 * cloud.flat.numel(),
                "d2h_bytes_per_step": 4 * DET * DET * nloc,
                "note": "same sweep through SweepRenderer.render: the cloud uploaded from pinned host "
                        "memory at the start of every step, each image copied to pinned host memory, "
                        "inside the timed region; the per-view camera (128 B xg_camera) travels as "
                        "kernel parameters",
                "render_view_loop": {"value": rv_value, "unit": "fps", "views_per_step": len(rv_angles),
                                     "note": "the drop-in call per view: render_view(cloud, scanner, phi) (one "
                                             "host sync for the entry count, fresh Frame and SplatList), each "
                                             "image copied to pinned host memory, the cloud re-uploaded per step; "
                                             f"views round-robin over {RV_STREAMS} streams"}},
        "roofline": {"bound": "fp32", "kernel": "k_composite_fwd_batch" if args.batch > 1 else "k_composite_fwd",
                     "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s", "frac": achieved / peak,
                     "traffic": (dram_traffic_per_view(args.batch > 1) * launch_views
                                 if dram_traffic_per_view(args.batch > 1) else None),
                     "flop_per_unit": FLOP_PER_PAIR, "units_per_launch": pairs_per_view * launch_views,
                     "views_per_launch": launch_views,
                     "kernel_ms_in_timed_region": comp_ctx * launch_views, "kernel_ms_isolated": comp_iso_ms,
                     "peak_source": peak_note,
                     "frac_of_measured_ffma": achieved / ffma_probe() if ffma_probe() else None,
                     "work_note": "work = 17 FLOP per pair the reference's loop visits (SURVEY 8d); the kernel "
                                  "skips pairs provably below the power cut-off at every pixel of its 16x8 half "
                                  "(exact), so this is useful work per second; ncu_pipes is the hardware view",
                     "ncu_pipes": ncu_pipes()},
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
        "ms_per_view": ms / (nloc * args.steps),
        "overflowed_views_timed": overflowed,
    }
    if other is not None:
        line["other_scaling_mode"] = other
    # the same kernel against the HBM roofline (why it is not the bound):
    # DRAM bytes per launch from the committed ncu capture / live launch time
    traffic = dram_traffic_per_view(args.batch > 1)
    if traffic:
        hpk, hnote = hbm_peak()
        gbs = traffic / (comp_ctx * 1e-3) / 1e9
        line["roofline_hbm"] = {"bound": "hbm", "kernel": line["roofline"]["kernel"], "achieved": gbs, "peak": hpk,
                                "unit": "GB/s", "frac": gbs / hpk, "traffic": traffic * launch_views,
                                "peak_source": hnote,
                                "note": "DRAM traffic (ncu dram__bytes_read + write, profiles/ncu_composite_fwd.json) "
                                        "per composited view / the live per-view kernel time"}
    del rend, out, host
    torch.cuda.empty_cache()
    if not args.no_c1:
        line["fwdbwd_c1"] = c1_block(args, timed, ClockSampler, local, world, rank)
    if not args.no_c4:
        line["stress_c4"] = c4_block(args, timed, world, rank)
    if not args.no_train:
        line["train_c2" if world == 1 else "train_c5"] = train_block(args, timed, ClockSampler, local, world)
        if world == 1 and not args.no_c5:  # train iters/s vs Gaussian count (BASELINE metric): C5 at N = 1
            line["train_c5"] = train_block(args, timed, ClockSampler, local, world, c5=True)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            nv = args.cpu_sample_views or cpu_workers("C3")
            line["cpu_baseline"] = cpu_baseline("C3", nv, angles=sweep_angles(0, 1)[:: max(1, VIEWS // nv)][:nv])
        except Exception as exc:  # report, never fake
            line["cpu_baseline"] = {"value": None, "error": repr(exc)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


G_C4, DET_C4, VIEWS_C4 = 196, 1024, 8
FLOP_BWD_PAIR = 51  # reverse-composite FLOP per traversed pair


def traversed_pairs(fr) -> float:
    """Sum over pixels of the entries the reference's loop visits
    (_kernels.pyx:56-58): n_contrib where the pixel terminated (T < 1e-4),
    else its tile's whole list - from a tracking forward's own outputs."""
    import torch

    ntx = (fr.w + 15) // 16
    key = (fr.h, fr.w)
    if key not in _TILE_OF:
        yy, xx = np.meshgrid(np.arange(fr.h), np.arange(fr.w), indexing="ij")
        _TILE_OF[key] = torch.as_tensor((yy // 16) * ntx + xx // 16, device=fr.image.device)
    lens = (fr.tile_ranges[:, 1] - fr.tile_ranges[:, 0])[_TILE_OF[key]]
    return float(torch.where(fr.t_final < 1e-4, fr.n_contrib.to(torch.int64), lens).sum().item())


_TILE_OF: dict = {}


def sort_bytes(n_active: float, entries: float, n_tiles: int) -> float:
    """SURVEY.md 8(d) S2 binning bytes: E (12 + 24 P + 8) + 8 T, P 8-bit passes."""
    p = int(np.ceil((np.ceil(np.log2(max(n_tiles, 2))) + 32) / 8))
    return entries * (12 + 24 * p + 8) + 8 * n_tiles


def ev_mean_ms(pairs) -> float:
    return float(np.mean([a.elapsed_time(b) for a, b in pairs])) if pairs else float("nan")


def c4_block(args, timed, world: int, rank: int) -> dict:
    """C4 of BASELINE.json: 1,030,301 ACUI Gaussians at a 1024x1024 detector
    (binning/sort and compositing stress).  One step = 8 views (22.5 degree
    steps, offset per rank); per-stage times from CUDA events on single
    views, throughput from the multi-stream sweep with images left in HBM;
    roofline of the compositing launch (events inside the timed sweep)."""
    import torch

    from paper_2403_04116_b200 import acui, geometry
    from paper_2403_04116_b200.engine import Frame
    from paper_2403_04116_b200.gaussians import GaussianCloud
    from paper_2403_04116_b200.inference import SweepRenderer

    cloud = GaussianCloud(**acui.init_alternative_arrays("cuboid", acui.benchmark_spec(G_C4), 16, 0), device="cuda")
    sc = geometry.ScannerConfig(L_SO, L_SD, DET_C4, DET_C4, 192.0 / DET_C4)
    angles = (np.arange(VIEWS_C4) + rank / max(world, 1)) * (np.pi / VIEWS_C4)
    rend = SweepRenderer(cloud, sc, n_streams=args.streams, batch=max(1, min(args.batch, VIEWS_C4)))
    out = torch.empty((VIEWS_C4, DET_C4, DET_C4), dtype=torch.float32, device="cuda")
    fr = Frame(cloud.n_points, DET_C4, DET_C4, "cuda")
    stages = np.zeros(3)
    entries, pairs, active = [], [], []
    for phi in angles:
        cam = rend.camera(phi)
        fr.preprocess(cloud, cam)
        a_n, e_n, _ = fr.ensure_binned()
        entries.append(e_n)
        active.append(a_n)
        fr.composite()  # tracking: n_contrib / t_final for the pair count
        pairs.append(traversed_pairs(fr))
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        fr.preprocess(cloud, cam)
        ev[1].record()
        fr.bin()
        ev[2].record()
        fr.composite(track=False)
        ev[3].record()
        torch.cuda.synchronize()
        stages += [ev[i].elapsed_time(ev[i + 1]) for i in range(3)]
    stages /= VIEWS_C4
    for _ in range(args.warmup):
        rend.render(angles, out=out)
    comp_events: list = []
    statuses: list = []
    idx = [0]

    def step():
        ev = comp_events if idx[0] == args.steps - 1 else None
        idx[0] += 1
        rend.render(angles, out=out, check=False, composite_events=ev)
        statuses.append(rend.last_status)

    ms = timed(step, args.steps)
    overflowed = count_overflows(statuses)
    rend.render(angles, out=out)  # status check
    ms_view = ms / (VIEWS_C4 * args.steps)
    ppv = float(np.mean(pairs))
    comp_ms_view = float(np.mean([a.elapsed_time(b) / nv for a, b, nv in comp_events]))
    peak, note = fp32_peak()
    hpk, _ = hbm_peak()
    achieved = FLOP_PER_PAIR * ppv / (comp_ms_view * 1e-3) / 1e12
    # step roofline (1,524 us): projection bytes + binning bytes at the HBM peak, 17 FLOP per pair
    roof_s = (156 * cloud.n_points + sort_bytes(np.mean(active), np.mean(entries), (DET_C4 // 16) ** 2)) / (hpk * 1e9) \
        + FLOP_PER_PAIR * ppv / (peak * 1e12)
    blk = {"metric": "fps (1024x1024 cone-beam projections/s), 1M Gaussians",
           "value": VIEWS_C4 * args.steps * world / (ms / 1e3), "unit": "fps",
           "ms_per_view": ms_view,
           "stages_ms_isolated": {"preprocess": stages[0], "bin_sort": stages[1], "composite": stages[2]},
           "entries_per_view": float(np.mean(entries)), "traversed_pairs_per_view": ppv,
           "overflowed_views_timed": overflowed,
           "roofline": {"bound": "fp32", "kernel": "k_composite_fwd_batch_np", "achieved": achieved, "peak": peak,
                        "unit": "TFLOP/s", "frac": achieved / peak, "traffic": None, "flop_per_unit": FLOP_PER_PAIR,
                        "units_per_launch": ppv * np.mean([nv for _, _, nv in comp_events]),
                        "kernel_ms_per_view_in_timed_region": comp_ms_view, "peak_source": note},
           "step_roofline": {"roofline_ms_per_view": roof_s * 1e3, "measured_ms_per_view": ms_view,
                             "frac": roof_s * 1e3 / ms_view,
                             "model": "156 B/G projection + SURVEY 8d S2 binning bytes at the HBM peak + "
                                      "17 FLOP per traversed pair at the FP32 peak",
                             "note": "the reference algorithm's roofline, not a bound on this implementation: "
                                     "the binning writes each entry once (multisplit) instead of the model's "
                                     "radix sort of 64-bit (tile|depth) keys, and the compositing skips pairs "
                                     "below the power cut-off at every pixel of a 16x8 half - so frac can "
                                     "exceed 1"},
           "config": {"workload": f"C4: {cloud.n_points:,} ACUI Gaussians (G={G_C4}), {DET_C4}x{DET_C4} detector, "
                                  f"{VIEWS_C4} views per GPU per step", "streams": args.streams}}
    del rend, fr, cloud, out
    torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        blk["cpu_baseline"] = safe(lambda: cpu_baseline("C4", units=min(cpu_workers("C4"), 16)))
    return blk


def count_overflows(statuses) -> int:
    """Views of the timed region whose entry buffer overflowed (rendered as
    no-ops there, re-rendered after timing)."""
    from paper_2403_04116_b200 import _native

    n = 0
    for st in statuses:
        w = st.cpu().numpy().astype(np.int64) & 0xFFFFFFFF
        n += int(np.count_nonzero(w & _native.XG_ST_ENTRY_OVERFLOW))
    return n


def safe(fn) -> dict:
    try:
        return fn()
    except Exception as exc:  # report, never fake
        return {"value": None, "error": repr(exc)[:200]}


VIEWS_C1 = 16
RV_STREAMS = int(os.environ.get("XG_RV_STREAMS", "4"))  # C3 render_view loop: views in flight


def c1_block(args, timed, clock_cls, local, world: int, rank: int) -> dict:
    """C1 of BASELINE.json: 50,653 ACUI Gaussians, one 256x256
    view forward + backward with dL/dI ~ N(0,1)/HW (the case the CPU
    reference runs, frontend.py:208-233 + backward.py:21-124).  One step =
    16 views (angles offset per rank), each a full fwd + bwd.
    value: the engine path (reused buffers, no host sync but the entry
    count read the forward overlaps); e2e: the reference-shaped public API
    (``render`` + ``render_backward``) with dL/dI uploaded from pinned host
    memory and every RenderGradients field copied back to the host."""
    import torch

    from paper_2403_04116_b200 import acui, geometry
    from paper_2403_04116_b200.engine import Frame
    from paper_2403_04116_b200.gaussians import GaussianCloud
    from paper_2403_04116_b200.rasterizer import render, render_backward
    from paper_2403_04116_b200.trainer import _IterationEngine

    cloud = GaussianCloud(**acui.init_alternative_arrays("cuboid", acui.benchmark_spec(G_C1), 16, 0), device="cuda")
    d = DET_C1
    sc = geometry.ScannerConfig(L_SO, L_SD, d, d, 192.0 / d)
    intr = geometry.intrinsic_from_config(sc)
    angles = (0.7 + (np.arange(VIEWS_C1) + rank / max(world, 1)) * (np.pi / VIEWS_C1)) % np.pi
    cams = [geometry.camera_pod(geometry.extrinsic_from_angle(sc, a), intr, (d, d)) for a in angles]
    dl_host = torch.as_tensor(np.random.default_rng(0).normal(size=(d, d)) / (d * d), dtype=torch.float32).pin_memory()
    dl = dl_host.cuda()
    n_streams = int(os.environ.get("XG_C1_STREAMS", "8"))  # independent views in flight (their kernels overlap on the 148 SMs)
    engs = [_IterationEngine(cloud, d, d) for _ in range(n_streams)]
    streams = [torch.cuda.Stream() for _ in range(n_streams)]
    eng = engs[0]
    fr = eng.frame
    # work units: traversed pairs per view (exact tracking forward)
    probe = Frame(cloud.n_points, d, d, "cuda")
    pairs, entries, active = [], [], []
    for cam in cams:
        probe.preprocess(cloud, cam)
        a_n, e_n, _ = probe.ensure_binned()
        probe.composite()
        pairs.append(traversed_pairs(probe))
        entries.append(e_n)
        active.append(a_n)
    del probe
    ev = {"fwd": [], "bwd": []}
    idx = [0]

    def one(e, cam, rec):
        f = e.frame
        f.preprocess(cloud, cam)
        f.bin_async()
        f.composite(train=True, events=ev["fwd"] if rec else None)
        if f.finish_bin():
            f.composite(train=True)
        f.backward(cloud, e.acc, e.grads.flat, e.grads.screen_norms, e.vis, dl_dimage=dl,
                   events=ev["bwd"] if rec else None)

    wave = os.environ.get("XG_C1_WAVE", "1") == "1"

    def step():
        # views round-robin over the streams (each its own buffers)
        main = torch.cuda.current_stream()
        for st in streams:
            st.wait_stream(main)
        if wave:
            # waves of n_streams views: every view's binning and forward are
            # queued before the host waits for the first entry count
            for w0 in range(0, len(cams), n_streams):
                grp = list(range(w0, min(w0 + n_streams, len(cams))))
                for i in grp:
                    with torch.cuda.stream(streams[i % n_streams]):
                        f = engs[i % n_streams].frame
                        f.preprocess(cloud, cams[i])
                        f.bin_async()
                        f.composite(train=True)
                for i in grp:
                    with torch.cuda.stream(streams[i % n_streams]):
                        e = engs[i % n_streams]
                        f = e.frame
                        if f.finish_bin():
                            f.composite(train=True)
                        f.backward(cloud, e.acc, e.grads.flat, e.grads.screen_norms, e.vis, dl_dimage=dl)
        else:
            for i, cam in enumerate(cams):
                with torch.cuda.stream(streams[i % n_streams]):
                    one(engs[i % n_streams], cam, False)
        for st in streams:
            main.wait_stream(st)

    def serial_step():
        rec = idx[0] == args.steps - 1
        idx[0] += 1
        for cam in cams:
            one(eng, cam, rec)

    for _ in range(args.warmup):
        step()
        serial_step()
    idx[0] = 0
    ms_serial = timed(serial_step, args.steps)  # one view at a time: the per-unit latency, kernel events
    with clock_cls(local) as clk:
        ms = timed(step, args.steps)
    grads_host = [torch.empty(eng.grads.flat.numel(), dtype=torch.float32).pin_memory() for _ in streams]

    def e2e_step():
        # the public calls, views round-robin over the streams: render()'s
        # entry-count sync waits for its own view's binning only, not for the
        # previous view's backward
        main = torch.cuda.current_stream()
        for st in streams:
            st.wait_stream(main)
        for i, a in enumerate(angles):
            with torch.cuda.stream(streams[i % n_streams]):
                ext = geometry.extrinsic_from_angle(sc, a)
                _, sp = render(cloud, ext, intr, (d, d))
                g = render_backward(cloud, sp, dl_host.to("cuda", non_blocking=True))
                grads_host[i % n_streams].copy_(g.flat, non_blocking=True)
        for st in streams:
            main.wait_stream(st)

    for _ in range(args.warmup):
        e2e_step()
    ms_e2e = timed(e2e_step, args.steps)
    units = VIEWS_C1 * args.steps * world
    ppv = float(np.mean(pairs))
    bwd_ms, fwd_ms = ev_mean_ms(ev["bwd"]), ev_mean_ms(ev["fwd"])
    peak, note = fp32_peak()
    hpk, _ = hbm_peak()
    achieved = FLOP_BWD_PAIR * ppv / (bwd_ms * 1e-3) / 1e12
    ms_unit = ms_serial / (VIEWS_C1 * args.steps)
    roof_s = (sort_bytes(np.mean(active), np.mean(entries), (d // 16) ** 2) + (156 + 248) * cloud.n_points) \
        / (hpk * 1e9) + (FLOP_PER_PAIR + FLOP_BWD_PAIR) * ppv / (peak * 1e12)
    blk = {"metric": "fwd+bwd/s (256x256 view, 50k Gaussians)", "value": units / (ms / 1e3), "unit": "fwd+bwd/s",
           "ms_per_unit": ms / (VIEWS_C1 * args.steps),
           "latency_ms_single_view": ms_unit,
           "concurrency": f"{n_streams} views in flight on {n_streams} streams (own buffers each), issued in "
                          "waves (every view's binning + forward queued before the host reads an entry count); "
                          "latency_ms_single_view: one view at a time",
           "e2e": {"value": units / (ms_e2e / 1e3), "unit": "fwd+bwd/s", "h2d_bytes_per_step": 4 * d * d * VIEWS_C1,
                   "d2h_bytes_per_step": 4 * eng.grads.flat.numel() * VIEWS_C1,
                   "note": "public API per view: render() (one host sync for the entry count, fresh SplatList) + "
                           "render_backward() with dL/dI from pinned host memory; every gradient field copied "
                           f"to pinned host memory; views round-robin over {n_streams} streams"},
           "traversed_pairs_per_view": ppv, "entries_per_view": float(np.mean(entries)),
           "kernel_ms": {"composite_fwd_train": fwd_ms, "composite_bwd": bwd_ms},
           "roofline": {"bound": "fp32", "kernel": "k_composite_bwd_ck", "achieved": achieved, "peak": peak,
                        "unit": "TFLOP/s", "frac": achieved / peak, "traffic": None, "flop_per_unit": FLOP_BWD_PAIR,
                        "units_per_launch": ppv, "kernel_ms_in_timed_region": bwd_ms, "peak_source": note,
                        "fwd_frac": FLOP_PER_PAIR * ppv / (fwd_ms * 1e-3) / 1e12 / peak},
           "step_roofline": {"roofline_ms_per_unit": roof_s * 1e3,
                             "measured_ms_per_unit": ms / (VIEWS_C1 * args.steps),
                             "frac": roof_s * 1e3 / (ms / (VIEWS_C1 * args.steps)),
                             "frac_single_view": roof_s * 1e3 / ms_unit,
                             "model": "SURVEY 8d: binning + 156 B/G projection + 248 B/G chain rule at the HBM "
                                      "peak, (17 + 51) FLOP per traversed pair at the FP32 peak (182 us in SURVEY)"},
           "clocks": clk.summary(),
           "config": {"workload": f"C1: {cloud.n_points:,} ACUI Gaussians (G={G_C1}), {d}x{d} detector, "
                                  f"{VIEWS_C1} views per GPU per step, each forward + backward",
                      "l2": "working set (~60 MB) fits L2; the C1 unit is one view"}}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        blk["cpu_baseline"] = safe(lambda: cpu_baseline("C1"))
    return blk


def probe_train(tr) -> tuple[float, float, float]:
    """(traversed pairs, entries, active splats) per training view, mean over
    the trainer's views, for its current cloud (untimed, own frame)."""
    from paper_2403_04116_b200.engine import Frame

    fr = Frame(tr.cloud.n_points, tr.h, tr.w, "cuda")
    p, e, a = [], [], []
    for cam in tr.cams.values():
        fr.preprocess(tr.cloud, cam)
        a_n, e_n, _ = fr.ensure_binned()
        fr.composite()
        p.append(traversed_pairs(fr))
        e.append(e_n)
        a.append(a_n)
    return float(np.mean(p)), float(np.mean(e)), float(np.mean(a))


def train_block(args, timed, clock_cls, local, world: int = 1, c5: bool = False) -> dict:
    """N=1 -> C2: ~100k Gaussians, 50 training views at 512x512, full
    training iterations (render fwd+bwd, L1, Adam, densify/prune every 100)
    through the public Trainer API.  N>1 (or ``c5``) -> C5: 493k Gaussians,
    one view per GPU per step, NCCL all-reduce of the flat gradient
    (bucketed, overlapped with the fused Adam), DataParallelTrainer - at
    N = 1 the single-GPU point of that scaling curve (no collective).  One
    step = ``--train-iters-per-step`` iterations."""
    import torch

    from paper_2403_04116_b200 import _native, acui, geometry
    from paper_2403_04116_b200.gaussians import GaussianCloud
    from paper_2403_04116_b200.parallel import DataParallelTrainer
    from paper_2403_04116_b200.trainer import TrainConfig, Trainer

    c5 = c5 or world > 1
    g = G_C3 if c5 else G_C2
    sc = geometry.ScannerConfig(L_SO, L_SD, DET, DET, 192.0 / DET, geometry.equal_interval_angles(100))
    ds, prep_s = phantom_dataset(g, sc)
    init = acui.init_alternative_arrays("cuboid", acui.benchmark_spec(g), 16, 0)
    cfg = TrainConfig(iterations=20_000, log_interval=10**9, eval_interval=10**9)
    per = args.train_iters_per_step
    out = {}
    # prime the process once (caching-allocator segments for the density-
    # control resizes, lazily loaded kernels): without it whichever mode runs
    # first measured ~15 % slow
    prime = Trainer(ds, GaussianCloud(**init, device="cuda"), cfg)
    for _ in range(7 * per):
        prime.step()
    del prime
    torch.cuda.synchronize()
    for mode in ("device", "e2e"):
        if not c5:
            tr = Trainer(ds, GaussianCloud(**init, device="cuda"), cfg, targets_on_host=(mode == "e2e"))
        else:
            tr = DataParallelTrainer(ds, GaussianCloud(**init, device="cuda"), cfg,
                                     targets_on_host=(mode == "e2e"), collective=args.collective)
        warm = max(args.warmup, 5)  # reach densify_from_iter = 500
        for _ in range(warm * per):
            tr.step()
        n0 = tr.cloud.n_points
        probe0 = probe_train(tr) if mode == "device" else None
        l0 = _native.kernel_launches()
        ev0 = tr.densify_events
        kev = {"fwd": [], "bwd": [], "pair": []}
        idx = [0]

        def step():
            if mode == "device" and idx[0] == args.steps - 1:  # kernel events during the last timed step
                tr.kernel_events = kev
            idx[0] += 1
            for _ in range(per):
                tr.step()

        with clock_cls(local) as clk:
            ms = timed(step, args.steps)
        tr.kernel_events = None
        out[mode] = {"ms": ms, "launches": _native.kernel_launches() - l0, "n0": n0, "n1": tr.cloud.n_points,
                     "densify_events": tr.densify_events - ev0, "clocks": clk.summary(),
                     "fwd_ms": ev_mean_ms(kev["fwd"]) if kev["fwd"] else None,
                     "bwd_ms": ev_mean_ms(kev["bwd"]) if kev["bwd"] else None,
                     "pair_ms": ev_mean_ms(kev["pair"]) if kev["pair"] else None,
                     "probe": (probe0, probe_train(tr)) if mode == "device" else None}
        torch.cuda.synchronize()
    iters = per * args.steps
    d, e = out["device"], out["e2e"]
    # work units of the timed window: traversed pairs / entries / active
    # splats per iteration over all training views, probed on the cloud at
    # the window's start and end (N grows at each density-control event)
    (p0, e0, a0), (p1, e1, a1) = d["probe"]
    ppi, epi, api = (p0 + p1) / 2, (e0 + e1) / 2, (a0 + a1) / 2
    n_mean = (d["n0"] + d["n1"]) / 2
    peak, note = fp32_peak()
    hpk, _ = hbm_peak()
    ms_iter = d["ms"] / iters
    roof_s = (sort_bytes(api, epi, (DET // 16) ** 2) + (156 + 248 + 756) * n_mean + 12 * DET * DET) / (hpk * 1e9) \
        + (FLOP_PER_PAIR + FLOP_BWD_PAIR) * ppi / (peak * 1e12)
    if d["pair_ms"] is not None:
        # the trainer's overlapped forward + reverse replay (xg_composite_train_pair):
        # one roofline over both kernels, (17 + 51) FLOP per traversed pair
        pair_ach = (FLOP_PER_PAIR + FLOP_BWD_PAIR) * ppi / (d["pair_ms"] * 1e-3) / 1e12
        tp = ROOT / "profiles" / "ncu_train_pair.json"
        pair_traffic = json.loads(tp.read_text())["dram_bytes_per_iteration"] if (tp.exists() and world == 1 and not c5) \
            else None
        train_roof = {"bound": "fp32", "kernel": "k_composite_fwd_np + k_composite_bwd_stream (one overlapped pair, "
                                                 "xg_composite_train_pair)",
                      "achieved": pair_ach, "peak": peak, "unit": "TFLOP/s", "frac": pair_ach / peak,
                      "traffic": pair_traffic,
                      "traffic_source": "profiles/ncu_train_pair.json (dram read + write of both kernels at C2, ncu)"
                      if pair_traffic else None, "flop_per_unit": FLOP_PER_PAIR + FLOP_BWD_PAIR, "units_per_launch": ppi,
                      "kernel_ms_in_timed_region": d["pair_ms"], "peak_source": note,
                      "units_note": "traversed pairs per iteration: mean over the 50 train views, probed on "
                                    "the cloud at the start and the end of the timed window; the pair's time runs "
                                    "from the forward's launch to the end of the replay (CUDA events around both)"}
    else:
        bwd_ach = FLOP_BWD_PAIR * ppi / (d["bwd_ms"] * 1e-3) / 1e12
        fwd_ach = FLOP_PER_PAIR * ppi / (d["fwd_ms"] * 1e-3) / 1e12
        train_roof = {"bound": "fp32", "kernel": "k_composite_bwd_ck", "achieved": bwd_ach, "peak": peak,
                      "unit": "TFLOP/s", "frac": bwd_ach / peak, "traffic": None, "flop_per_unit": FLOP_BWD_PAIR,
                      "units_per_launch": ppi, "kernel_ms_in_timed_region": d["bwd_ms"], "peak_source": note,
                      "fwd_kernel": "k_composite_fwd (tracking, xg_composite_fwd_train)",
                      "fwd_achieved": fwd_ach, "fwd_frac": fwd_ach / peak,
                      "units_note": "traversed pairs per iteration: mean over the 50 train views, probed on "
                                    "the cloud at the start and the end of the timed window"}
    name = (f"C2: {g}^3-lattice ACUI init ({(2 * (g // 4) + 3) ** 3:,} Gaussians), 50 train views of a "
            f"100-view 512x512 sweep, full iterations incl. densify/prune every 100 ({per // 100} events per step)"
            if not c5 else
            f"C5: {(2 * (g // 4) + 3) ** 3:,} Gaussians, 512x512, data-parallel x{world}: one view per GPU per "
            + ("step, NCCL all-reduce of the 27N gradient bucketed and overlapped with the fused Adam"
               if args.collective == "nccl" else
               "step, the 27N gradient reduce-scattered and all-gathered over peer memory with Adam fused "
               "into the all-gather (csrc/xg_dp.cu)")
            + (" (N = 1: no collective, the curve's single-GPU point)" if world == 1 else ""))
    blk = {"metric": "train iters/s", "value": iters / (d["ms"] / 1e3), "unit": "iters/s",
            "views_per_s": iters * world / (d["ms"] / 1e3),
            "ms_per_iter": d["ms"] / iters,
            "config": {"workload": name,
                       "iters_per_step": per, "warmup_iters": max(args.warmup, 5) * per,
                       "n_points_timed": [d["n0"], d["n1"]], "densify_events": d["densify_events"],
                       "targets": f"default voxel phantom ({g}^3, 100 mm) cone-beam projected on the GPU "
                                  f"(xg_project_volume), normalised, 3 % noise - {prep_s:.2f} s for "
                                  f"{len(sc.angles)} views"},
            "e2e": {"value": iters / (e["ms"] / 1e3), "unit": "iters/s", "h2d_bytes_per_step": 4 * DET * DET * per,
                    "d2h_bytes_per_step": 8 * per,
                    "note": "targets in pinned host memory, copied H2D every iteration; L1 loss copied D2H"},
            "gpu_launches": int(d["launches"]), "clocks": d["clocks"],
            "traversed_pairs_per_iter": ppi, "entries_per_iter": epi,
            "kernel_ms": {"composite_fwd_train": d["fwd_ms"], "composite_bwd": d["bwd_ms"],
                          "train_pair": d["pair_ms"]},
            "roofline": train_roof,
            "step_roofline": {"roofline_ms_per_iter": roof_s * 1e3, "measured_ms_per_iter": ms_iter,
                              "frac": roof_s * 1e3 / ms_iter,
                              "model": "SURVEY 8d: binning + 156 B/G projection + 248 B/G chain rule + 756 B/G "
                                       "Adam + 12 B/px L1 at the HBM peak, (17 + 51) FLOP per traversed pair at "
                                       "the FP32 peak (744 us per iteration on the initial cloud in SURVEY)"}}
    if world == 1 and not c5 and not args.no_cpu_baseline:
        del tr
        torch.cuda.empty_cache()
        v = int(ds.train_indices[0])
        blk["cpu_baseline"] = safe(lambda: cpu_baseline(
            "C2", units=min(cpu_workers("C2"), 16), target=np.asarray(ds.images[v], np.float64),
            angles=np.full(16, float(ds.angles[v]))))
        if blk["cpu_baseline"].get("value"):
            blk["cpu_baseline"]["sample"] += "; each worker runs the first iteration from the ACUI init"
    return blk


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
