"""Summarise an ncu report (development aid): key throughput metrics, stall
reasons and the per-address instruction / stall-sample distribution."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "sm__cycles_active.avg", "smsp__cycles_active.avg",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep, lo=None, hi=None):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, units, v = rows[0], rows[1], rows[2]
    d = dict(zip(h, v))
    u = dict(zip(h, units))
    for k in KEYS:
        if k in d:
            print(f"  {k:64s} {d[k]} {u[k]}")
    st = [(k, float(d[k] or 0)) for k in h if k.startswith("smsp__average_warps_issue_stalled")
          and k.endswith("_per_issue_active.ratio")]
    for k, x in sorted(st, key=lambda t: -t[1])[:8]:
        print(f"  {k.replace('smsp__average_warps_issue_stalled_', 'stall ').replace('_per_issue_active.ratio', ''):64s} {x:.3f}")
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    hh, data = src[1], src[2:]
    ai, si, ie, ss = (hh.index(x) for x in ("Address", "Source", "Instructions Executed",
                                            "Warp Stall Sampling (All Samples)"))
    base = int(data[0][ai], 16)
    tot = sum(int(r[ie]) for r in data)
    tots = sum(int(r[ss]) for r in data)
    blk = {}
    for r in data:
        k = (int(r[ai], 16) - base) // 0x200
        a = blk.setdefault(k, [0, 0])
        a[0] += int(r[ie])
        a[1] += int(r[ss])
    print(f"  warp instructions {tot}, stall samples {tots}")
    for k, (n, s) in sorted(blk.items()):
        if n > 0.005 * tot or s > 0.005 * tots:
            print(f"  {k * 0x200:#07x} inst {100 * n / tot:5.1f}%  samples {100 * s / tots:5.1f}%")
    if lo is not None:
        for r in data:
            off = int(r[ai], 16) - base
            if lo <= off < hi:
                print(f"{off:#07x} {int(r[ie]):>10d} {int(r[ss]):>5d}  {r[si].strip()[:90]}")


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0], *(int(x, 16) for x in a[1:3]))
