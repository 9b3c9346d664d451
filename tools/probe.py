"""Quick per-stage timing probe on one GPU (development aid)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2403_04116_b200 import acui, geometry
from paper_2403_04116_b200.engine import Frame

def main(g=152, d=512, views=20):
    arrs = acui.init_alternative_arrays("cuboid", acui.benchmark_spec(g), 16, 0)
    cloud = acui.GaussianCloud(**arrs, device="cuda")
    sc = geometry.ScannerConfig(1000.0, 1500.0, d, d, 192.0 / d, geometry.equal_interval_angles(360))
    intr = geometry.intrinsic_from_config(sc)
    fr = Frame(cloud.n_points, d, d, "cuda", entry_capacity=30 * cloud.n_points)
    cams = [geometry.camera_pod(geometry.extrinsic_from_angle(sc, float(p)), intr, (d, d)) for p in sc.angles[:views]]
    fr.preprocess(cloud, cams[0]); a, e, s = fr.ensure_binned(); fr.composite(); torch.cuda.synchronize()
    print(f"N={cloud.n_points} D={d} active={a} entries={e} status={s}")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t = np.zeros(4)
    for cam in cams:
        ev[0].record(); fr.preprocess(cloud, cam); ev[1].record(); fr.bin(); ev[2].record(); fr.composite(); ev[3].record()
        torch.cuda.synchronize()
        t[:3] += [ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3])]
        ev[0].record(); fr.composite(track=False); ev[1].record()
        torch.cuda.synchronize()
        t[3] += ev[0].elapsed_time(ev[1])
    t /= len(cams)
    print(f"per view ms: preprocess {t[0]:.3f} bin {t[1]:.3f} composite {t[2]:.3f} (inference {t[3]:.3f}) "
          f"total {t[:3].sum():.3f} -> {1000/t[:3].sum():.0f} fps")
    # backward timing
    acc = torch.zeros((cloud.n_points, 8), device="cuda")
    gflat = torch.empty_like(cloud.flat); sn = torch.empty(cloud.n_points, device="cuda"); vis = torch.empty(cloud.n_points, dtype=torch.uint8, device="cuda")
    dl = torch.randn(d, d, device="cuda") / (d * d)
    ev[0].record(); fr.backward(cloud, acc, gflat, sn, vis, dl_dimage=dl); ev[1].record(); torch.cuda.synchronize()
    ev[0].record(); fr.backward(cloud, acc, gflat, sn, vis, dl_dimage=dl); ev[1].record(); torch.cuda.synchronize()
    print(f"backward (composite_bwd + preprocess_bwd) ms: {ev[0].elapsed_time(ev[1]):.3f}")

if __name__ == "__main__":
    main(*(int(x) for x in sys.argv[1:]))
