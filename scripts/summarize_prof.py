"""Summarise gpurun_out/ ncu artefacts into profiles/ (tracked).

    python scripts/summarize_prof.py TAG [launch_csv] [rep ...]

Writes profiles/launches_TAG.txt (per-kernel totals of an ncu launch list,
`--metrics gpu__time_duration.sum`) and profiles/ncu_TAG_<kernel>.txt (key
`--set full` metrics + per-launch DRAM bytes for each .ncu-rep).
"""
import collections
import csv
import io
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles")

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_issued.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "smsp__average_warp_latency_per_inst_issued.ratio",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum"]


def launches(tag, path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, n = collections.defaultdict(float), collections.Counter()
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0,
              "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("void ", "")
        tot[name] += v
        n[name] += 1
    T = sum(tot.values())
    lines = [f"# ncu launch list ({path}); gpu__time_duration.sum, --clock-control none",
             f"# cold-cache serialised per-launch times: compare SHARES, not absolutes",
             f"# total {T / 1e3:.1f} ms over {sum(n.values())} launches", "",
             f"{'kernel':70s} {'total_ms':>10s} {'share':>7s} {'launches':>8s} {'avg_us':>9s}"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"{k[:70]:70s} {v / 1e3:10.2f} {v / T:7.1%} {n[k]:8d} {v / n[k]:9.1f}")
    dst = os.path.join(OUT, f"launches_{tag}.txt")
    open(dst, "w").write("\n".join(lines) + "\n")
    print(dst)


def rep(tag, path):
    res = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True)
    rows = list(csv.reader(io.StringIO(res.stdout)))
    if len(rows) < 3:
        print("no data in", path)
        return
    h, units, vals = rows[0], rows[1], rows[2:]
    # several launches in one report: summarise the longest (the finest
    # level), list the others
    ti = h.index("gpu__time_duration.sum")
    num = lambda x: float(x.replace(",", "")) if x else 0.0
    best = max(range(len(vals)), key=lambda r: num(vals[r][ti]))
    row = vals[best]
    name = row[h.index("Kernel Name")].split("(")[0].replace("void ", "")
    lines = [f"# ncu --set full --clock-control none: {os.path.basename(path)}",
             f"# kernel: {name}" + (f" (longest of {len(vals)} launches)" if len(vals) > 1 else ""),
             ""]
    for k in KEYS:
        if k in h:
            i = h.index(k)
            lines.append(f"{k:60s} {row[i]:>18s} {units[i]}")
    stalls = sorted(((num(row[i]), k) for i, k in enumerate(h)
                     if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                     and not k.endswith("not_issued")), reverse=True)
    tot = sum(v for v, _ in stalls) or 1.0
    if stalls:
        lines += ["", "# warp-state samples (top 6)"]
        for v, k in stalls[:6]:
            lines.append(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', 'stall_'):60s} "
                         f"{v / tot:17.1%}")
    if len(vals) > 1:
        gi = h.index("launch__grid_size") if "launch__grid_size" in h else None
        lines += ["", "# all launches: grid, us"]
        for r in vals:
            lines.append(f"  {r[gi] if gi is not None else '':>8s} {num(r[ti]):10.2f}")
    short = name.split("::")[-1].split("<")[0]
    dst = os.path.join(OUT, f"ncu_{tag}_{short}.txt")
    open(dst, "w").write("\n".join(lines) + "\n")
    print(dst)


if __name__ == "__main__":
    tag = sys.argv[1]
    for a in sys.argv[2:]:
        if a.endswith(".csv"):
            launches(tag, a)
        elif a.endswith(".ncu-rep"):
            rep(tag, a)
