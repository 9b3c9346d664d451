import sys, numpy as np, torch
sys.path.insert(0, ".")
from oracle import oracle as orc
import paper_2403_04116_b200 as xg
from paper_2403_04116_b200 import acui
for g, d in ((68, 1024), (152, 1024), (196, 512), (152, 1008), (152, 992), (196, 1024)):
    arrs = {k: np.asarray(v, np.float32) for k, v in acui.init_alternative_arrays("cuboid", acui.benchmark_spec(g), 16, 0).items()}
    cloud = xg.GaussianCloud(**arrs, device="cuda")
    sc = xg.ScannerConfig(1000.0, 1500.0, d, d, 192.0 / d)
    proj, sp = xg.render(cloud, xg.extrinsic_from_angle(sc, 0.7), xg.intrinsic_from_config(sc), (d, d))
    cam = orc.camera_from_view(1000.0, 1500.0, d, d, 192.0 / d, 0.7)
    pre = orc.preprocess(arrs, np.ones(16, np.float32), cam)
    b = orc.bin_entries(pre, cam)
    mine = sp.entry_ids.cpu().numpy().astype(np.uint32)
    print(g, d, "N", cloud.n_points, "T", b["tile_ranges"].shape[0], "E", b["n_entries"], "mismatch", int((mine != b["entry_splat"]).sum()), flush=True)
