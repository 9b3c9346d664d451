"""Benchmark of the DRR hot path (BASELINE.json metric).

Default workload (N=1): C3 of BASELINE.json - 493,039 ACUI Gaussians
(cuboid G=152, interval 2, 16 features, seed 0), 512x512 cone-beam
detector (L_SO 1000, L_SD 1500, pitch 192/512 mm), a 360-view novel-view
sweep over [0, pi).  One "step" = one 360-view sweep per GPU.  Multi-GPU
(torchrun) shards views: rank r renders the sweep offset by r/N of the
0.5 degree step - disjoint view sets, no collective on the data path
(weak scaling: 360 views per GPU per step).

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


def _cpu_init(kind: str):
    os.environ["OMP_NUM_THREADS"] = "1"
    arrs = c3_arrays()
    if kind == "reference":
        sys.path.insert(0, str(ROOT / "oracle" / "_ref"))
        from xsplat.gaussians import GaussianCloud
        from xsplat.geometry import ScannerConfig
        from xsplat.rasterizer import set_backend

        set_backend("compiled")
        f32 = {k: np.asarray(v, np.float32).astype(np.float64) for k, v in arrs.items()}
        _CPU_STATE["cloud"] = GaussianCloud(**f32)
        _CPU_STATE["scanner"] = ScannerConfig(L_SO, L_SD, DET, DET, 192.0 / DET)
    else:
        _CPU_STATE["fields"] = {k: np.asarray(v, np.float32) for k, v in arrs.items()}
    _CPU_STATE["kind"] = kind


def _cpu_render(phi: float) -> float:
    t0 = time.perf_counter()
    if _CPU_STATE["kind"] == "reference":
        from xsplat.rasterizer import render_view

        render_view(_CPU_STATE["cloud"], _CPU_STATE["scanner"], phi)
    else:
        from oracle import oracle as orc

        cam = orc.camera_from_view(L_SO, L_SD, DET, DET, 192.0 / DET, phi)
        orc.render(_CPU_STATE["fields"], np.ones(16, np.float32), cam)
    return time.perf_counter() - t0


def cpu_workers() -> int:
    n = os.cpu_count() or 1
    try:
        import psutil

        mem = psutil.virtual_memory().available
        n = min(n, max(1, int(mem // (3 * 2**30))))  # ~1.5-2.5 GB peak per reference process
    except Exception:
        pass
    return max(1, min(n, 64))


def cpu_sweep_pool(kind: str, workers: int):
    import multiprocessing as mp

    ctx = mp.get_context("fork")
    return ctx.Pool(workers, initializer=_cpu_init, initargs=(kind,))


def cpu_baseline(views_per_step: int | None = None) -> dict:
    """Bounded sample of the C3 workload on the host: one view per worker
    process (the reference is single-threaded, cli.py:4-7)."""
    kind = "reference" if _ref_available() else "port"
    workers = cpu_workers()
    nv = views_per_step or workers
    with cpu_sweep_pool(kind, workers) as pool:
        angles = sweep_angles(0, 1)[:: max(1, VIEWS // nv)][:nv]
        t0 = time.perf_counter()
        per = pool.map(_cpu_render, list(angles), chunksize=1)
        wall = time.perf_counter() - t0
    return {"value": nv / wall, "unit": "fps", "cores": workers, "kind": kind,
            "sample": f"{nv} of the 360 C3 views ({'xsplat compiled backend' if kind == 'reference' else 'oracle C port'}, "
                      f"1 view per process, {workers} processes, OMP_NUM_THREADS=1; "
                      f"single view {np.median(per):.1f} s median)"}


def run_reference(args) -> None:
    rank, world, _ = dist_env()
    if rank != 0:
        return
    kind = "reference" if _ref_available() else "port"
    workers = cpu_workers()
    with cpu_sweep_pool(kind, workers) as pool:
        angles = list(sweep_angles(0, 1)[:: max(1, VIEWS // workers)][:workers])
        for _ in range(args.warmup):
            pool.map(_cpu_render, angles, chunksize=1)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            pool.map(_cpu_render, angles, chunksize=1)
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
    p = ROOT / "profiles" / "fp32_peak.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["fp32_tflops"]), f"measured FFMA peak on this pool's B200 (profiles/fp32_peak.json)"
    return 74.45, "nominal 148 SM x 128 FMA x 2 x 1.965 GHz (no measured FP32 peak)"


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
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2403_04116_b200 import _native, geometry
    from paper_2403_04116_b200.gaussians import GaussianCloud
    from paper_2403_04116_b200.inference import SweepRenderer

    arrs = c3_arrays()
    cloud = GaussianCloud(**arrs, device="cuda")
    sc = geometry.ScannerConfig(L_SO, L_SD, DET, DET, 192.0 / DET)
    angles = sweep_angles(rank, world)
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

    def step():
        # composite-kernel events on their own stream during the last timed step
        ev = comp_events if step_idx[0] == args.steps - 1 else None
        step_idx[0] += 1
        rend.render(angles, out=out, check=False, composite_events=ev)

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

    total_views = VIEWS * args.steps * world
    value = total_views / (ms / 1e3)
    e2e_value = total_views / (ms_e2e / 1e3)
    peak, peak_note = fp32_peak()
    comp_iso_ms = float(np.mean(comp_iso))
    achieved = FLOP_PER_PAIR * pairs_per_view / (comp_ctx * 1e-3) / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": "fps", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: ACUI cuboid cloud (BASELINE C3 generator, seed 0), analytic cameras",
        "config": {"workload": "C3: 493,039 Gaussians (G=152), 512x512 detector, 360-view novel-view sweep "
                               "per GPU per step", "views_per_step_per_gpu": VIEWS, "streams": args.streams,
                   "l2": "inputs larger than L2 (6M-entry lists + 1 MB images per view, 360 views/step)",
                   "views_per_composite_launch": args.batch,
                   "parallelism": f"view-sharded x{world}"},
        "e2e": {"value": e2e_value, "unit": "fps",
                "h2d_bytes_per_step": 128 * VIEWS + 4 * cloud.flat.numel(),
                "d2h_bytes_per_step": 4 * DET * DET * VIEWS,
                "note": "same sweep through SweepRenderer.render: the cloud uploaded from pinned host "
                        "memory at the start of every step, each image copied to pinned host memory, "
                        "inside the timed region; the per-view camera (128 B xg_camera) travels as "
                        "kernel parameters"},
        "roofline": {"bound": "fp32", "kernel": "k_composite_fwd_batch" if args.batch > 1 else "k_composite_fwd",
                     "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s", "frac": achieved / peak,
                     "traffic": (dram_traffic_per_view(args.batch > 1) * launch_views
                                 if dram_traffic_per_view(args.batch > 1) else None),
                     "flop_per_unit": FLOP_PER_PAIR, "units_per_launch": pairs_per_view * launch_views,
                     "views_per_launch": launch_views,
                     "kernel_ms_in_timed_region": comp_ctx * launch_views, "kernel_ms_isolated": comp_iso_ms,
                     "peak_source": peak_note},
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
        "ms_per_view": ms / (VIEWS * args.steps),
    }
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
    if not args.no_c4:
        line["stress_c4"] = c4_block(args, timed, world, rank)
    if not args.no_train:
        line["train_c2" if world == 1 else "train_c5"] = train_block(args, timed, ClockSampler, local, world)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(args.cpu_sample_views or None)
        except Exception as exc:  # report, never fake
            line["cpu_baseline"] = {"value": None, "error": repr(exc)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


G_C4, DET_C4, VIEWS_C4 = 196, 1024, 8


def c4_block(args, timed, world: int, rank: int) -> dict:
    """C4 of BASELINE.json: 1,030,301 ACUI Gaussians at a 1024x1024 detector
    (binning/sort and compositing stress).  One step = 8 views (45 degree
    steps, offset per rank); per-stage times from CUDA events on single
    views, throughput from the multi-stream sweep with images left in HBM."""
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
    entries = []
    for phi in angles:
        cam = rend.camera(phi)
        fr.preprocess(cloud, cam)
        entries.append(fr.ensure_binned()[1])
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
    ms = timed(lambda: rend.render(angles, out=out, check=False), args.steps)
    rend.render(angles, out=out)  # status check
    return {"metric": "fps (1024x1024 cone-beam projections/s), 1M Gaussians",
            "value": VIEWS_C4 * args.steps * world / (ms / 1e3), "unit": "fps",
            "ms_per_view": ms / (VIEWS_C4 * args.steps),
            "stages_ms_isolated": {"preprocess": stages[0], "bin_sort": stages[1], "composite": stages[2]},
            "entries_per_view": float(np.mean(entries)),
            "config": {"workload": f"C4: {cloud.n_points:,} ACUI Gaussians (G={G_C4}), {DET_C4}x{DET_C4} detector, "
                                   f"{VIEWS_C4} views per GPU per step", "streams": args.streams}}


def train_block(args, timed, clock_cls, local, world: int = 1) -> dict:
    """N=1 -> C2: ~100k Gaussians, 50 training views at 512x512, full
    training iterations (render fwd+bwd, L1, Adam, densify/prune every 100)
    through the public Trainer API.  N>1 -> C5: 493k Gaussians, one view per
    GPU per step, NCCL all-reduce of the flat gradient (bucketed, overlapped
    with the fused Adam), DataParallelTrainer.  One step = 100 iterations."""
    import torch

    from paper_2403_04116_b200 import _native, acui, geometry
    from paper_2403_04116_b200.gaussians import GaussianCloud
    from paper_2403_04116_b200.parallel import DataParallelTrainer
    from paper_2403_04116_b200.trainer import TrainConfig, Trainer

    g = G_C2 if world == 1 else G_C3
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
        if world == 1:
            tr = Trainer(ds, GaussianCloud(**init, device="cuda"), cfg, targets_on_host=(mode == "e2e"))
        else:
            tr = DataParallelTrainer(ds, GaussianCloud(**init, device="cuda"), cfg,
                                     targets_on_host=(mode == "e2e"))
        warm = max(args.warmup, 5)  # reach densify_from_iter = 500
        for _ in range(warm * per):
            tr.step()
        n0 = tr.cloud.n_points
        l0 = _native.kernel_launches()
        ev0 = tr.densify_events
        with clock_cls(local) as clk:
            ms = timed(lambda: [tr.step() for _ in range(per)], args.steps)
        out[mode] = {"ms": ms, "launches": _native.kernel_launches() - l0, "n0": n0, "n1": tr.cloud.n_points,
                     "densify_events": tr.densify_events - ev0, "clocks": clk.summary()}
        torch.cuda.synchronize()
    iters = per * args.steps
    d, e = out["device"], out["e2e"]
    name = (f"C2: {g}^3-lattice ACUI init ({(2 * (g // 4) + 3) ** 3:,} Gaussians), 50 train views of a "
            f"100-view 512x512 sweep, full iterations incl. densify/prune every 100 ({per // 100} events per step)"
            if world == 1 else
            f"C5: {(2 * (g // 4) + 3) ** 3:,} Gaussians, 512x512, data-parallel x{world}: one view per GPU per "
            "step, NCCL all-reduce of the 27N gradient bucketed and overlapped with the fused Adam")
    return {"metric": "train iters/s", "value": iters / (d["ms"] / 1e3), "unit": "iters/s",
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
            "gpu_launches": int(d["launches"]), "clocks": d["clocks"]}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
