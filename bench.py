"""Benchmark: full spatial + tonal data optimization of a synthetic 4K RGB
image at 5% mask density (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one `run_pipeline` (cli.py:251-257: `dd` densification + `ras+vi`
tonal optimization, PipelineConfig defaults) over one synthetic image
(SURVEY.md section 8d `synth`).  `value` is the device-timed wall time of a
step with the input already resident in HBM (CUDA events on the launching
stream, barrier + synchronize on both sides, max over ranks); `e2e` is the
same step through the public API with the input in pinned host memory and
the result (mask + stored values) read back inside the timed region.  Under
torchrun each rank optimizes its own image (replicas: the path has no data
exchange across images), so `scaling` is "weak".

`strips` (BASELINE.json configs[4]) is the north_star's multi-GPU layout for
one large image: a 7680x4320 RGB inpainting solve cut into one row strip
per rank, halo exchange / norm all-reduce over NCCL (csrc/strips.cu),
strong scaling, Mpixel-iterations/s.

`strips_pipeline` (N > 1) is the same 4K pipeline on ONE image cut into
row strips over the ranks (every solve, the Delaunay step and the
accumulate partitioned; jump flooding replicated; RAS blocks sharded):
strong scaling of the metric's wall time.

`--impl reference` times the reference algorithm's CPU implementation (the
oracle port under oracle/: C kernel table + numpy orchestration, bit-exact
with the reference) on the host cores, on bounded samples of the 4K
workload's own work units (finest V-cycles on the initial and final masks,
RAS block V-cycles, JFA / Delaunay / accumulate passes), weighted by the
unit census of the reference's own measured 4K run (oracle/sampled.py,
tests/golden/large_cfg4.json).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

H, W, C = 2160, 3840, 3
METRIC = "4K RGB 5% mask: spatial+tonal opt wall time (s); solver HBM GB/s vs peak"
WORKLOAD = "3840x2160 RGB synthetic, 5% density, dd (20 iters) + ras+vi (PipelineConfig defaults)"


def _ncu_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum of one finest-level 4K
    launch of `kernel` from the newest committed ncu --set full summary
    (profiles/ncu_<tag>_<kernel>.txt, scripts/summarize_prof.py), or None."""
    import glob
    import re
    # the tag named in profiles/LATEST (the newest profile round), else the
    # lexicographically last tag
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"ncu_*_{kernel}.txt")))
    try:
        with open(os.path.join(ROOT, "profiles", "LATEST")) as fh:
            latest = os.path.join(ROOT, "profiles", f"ncu_{fh.read().strip()}_{kernel}.txt")
        if os.path.exists(latest):
            files.append(latest)
    except OSError:
        pass
    if not files:
        return None
    tot = 0.0
    issue = None
    for line in open(files[-1]):
        m = re.match(r"dram__bytes_(read|write)\.sum\s+([\d.]+)\s+(\w+)", line)
        if m:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(m.group(3), 1)
            tot += float(m.group(2)) * scale
        m = re.match(r"sm__inst_issued\.avg\.pct_of_peak_sustained_active\s+([\d.]+)", line)
        if m:
            issue = float(m.group(1)) / 100.0
    return ({"bytes": tot, "issue": issue, "source": os.path.relpath(files[-1], ROOT)}
            if tot else None)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    def __init__(self, gpu_index=0):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self._proc = None
        return self

    def _read(self):
        for line in self._proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self._proc is not None:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons}


def _dist():
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return world, rank, local


def _max_over_ranks(x, world, device="cuda"):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def _cpu_sampled(steps, warmup, threads_one=True):
    """The oracle port timed on a bounded sample of the 4K workload's own
    work units (oracle/sampled.py): returns (estimate dict, per-step s)."""
    from oracle import sampled
    smp = sampled.Sampler()
    nthr = os.cpu_count() or 1
    sampled.set_threads(nthr)
    step_s = []
    for i in range(warmup + steps):
        dt = smp.step("init" if i % 2 == 0 else "final")
        if i >= warmup:
            step_s.append(dt)
        if i == warmup - 1:
            smp.reset()
    est = smp.estimate()
    est["threads"] = sampled.get_threads()
    if threads_one:
        smp.reset()
        sampled.set_threads(1)
        for which in ("init", "final"):
            smp.step(which)
        est["estimate_1thread_s"] = smp.estimate()["estimate_s"]
        sampled.set_threads(nthr)
    est["cpu_model"] = sampled.cpu_model()
    est["cpu_count"] = os.cpu_count()
    est["reference_note"] = smp.reference_note()
    return est, step_s


def _cpu_line(est, step_s):
    return {"value": est["estimate_s"], "unit": "s", "cores": est["threads"], "kind": "port",
            "sample": (f"oracle port (C kernels, OpenMP x{est['threads']}) timed on the 4K "
                       f"workload's own work units -- finest V-cycles on the initial and final "
                       f"masks, 64x64 RAS block V-cycles, JFA / Delaunay / accumulate passes; "
                       f"{len(step_s)} step(s) of {statistics.mean(step_s):.1f} s -- weighted by "
                       f"the unit census of the reference's measured 4K run "
                       f"(units cover {est['covered']:.0%} of its time; "
                       f"oracle/sampled.py)"),
            "estimate_1thread_s": est.get("estimate_1thread_s"),
            "cpu_model": est["cpu_model"], "cpu_count": est["cpu_count"],
            "unit_means_s": est["unit_means_s"], "counts": est["counts"],
            "reference_measured": est["reference_note"]}


def run_reference(args):
    """CPU arm: the oracle port on the host cores, one bounded 4K work-unit
    sample per step (oracle/sampled.py); value = the full-run estimate."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    est, step_s = _cpu_sampled(args.steps, args.warmup)
    value = est["estimate_s"]
    cpu = _cpu_line(est, step_s)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.mean(step_s) * 1e3, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": _config(args, args.gpus, False),
        "sample": ("each step = one bounded sample of the 4K workload (ms_per_step is the "
                   "sample's time); value = the full-run estimate from the sampled unit "
                   "costs x the reference's unit census (cpu_baseline.sample)"),
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _config(args, world, strips_mode):
    return {"workload": WORKLOAD, "H": H, "W": W, "C": C, "density": 0.05,
            "parallelism": (f"row strips x{world} (one image; solves and the Delaunay / "
                            "accumulate steps on strips, JFA replicated, RAS blocks "
                            "sharded)"
                            if strips_mode else f"replicas x{world} (one image per GPU)"),
            "l2": "working set (>1 GB per step) exceeds the 126 MB L2"}


S5 = (4320, 7680, 3)  # BASELINE.json configs[4]: 8K RGB, row strips over the ranks


def run_strips(world, rank, steps=3):
    """configs[4]: a 7680x4320 RGB inpainting solve (cold FMG to the default
    1e-4, 5% random mask) cut into one row strip per rank (csrc/strips.cu:
    halo exchange + band-norm all-reduce + agglomeration broadcasts over
    NCCL; at N = 1 a single strip).  Strong scaling: the image is fixed.
    Time = CUDA events around each solve, max over ranks; Mpixel-iterations
    = pixels x finest-level V-cycles."""
    import numpy as np
    import torch

    import paper_2401_06747_b200 as sp
    from oracle.oracle import synth  # input generator only
    from paper_2401_06747_b200.strips import StripSolver

    H5, W5, C5 = S5
    f = torch.from_numpy(synth(H5, W5, C5, seed=0)).cuda()
    m = torch.from_numpy((np.random.default_rng(5).random((H5, W5)) < 0.05)
                         .astype(np.uint8)).cuda()
    cfg = sp.MultigridConfig()
    solver = (StripSolver.distributed(H5, W5, C5, cfg=cfg) if world > 1
              else StripSolver(H5, W5, C5, strips=1, cfg=cfg))
    fi, mi = sp.Image(f), sp.Mask(m)
    u, rep = solver.inpaint(fi, mi)  # warm-up (allocations, NCCL channels)
    torch.cuda.synchronize()
    times, cycles = [], rep.iterations
    stream = torch.cuda.current_stream()
    for _ in range(steps):
        _barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        u, rep = solver.inpaint(fi, mi)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(_max_over_ranks(e0.elapsed_time(e1), world))
    ms = sorted(times)[len(times) // 2]
    # the gathered solution is the same on every rank
    chk = float(u.tensor()[:, ::97, ::89].double().sum())
    return {"workload": f"{W5}x{H5} RGB inpaint (cold FMG to 1e-4, 5% random mask)",
            "n_strips": world, "partitioned_levels": solver.La, "halo_rows": 48,
            "ms_per_solve": ms, "vcycles": int(cycles),
            "mpix_iter_per_s": H5 * W5 * cycles / (ms * 1e-3) / 1e6,
            "converged": bool(rep.converged), "checksum": chk,
            "scaling": "strong (fixed image, one strip per GPU)"}


def run_strip_pipeline(world, steps):
    """N > 1 beside the replicas: the same 4K pipeline on ONE image cut
    into one row strip per rank (every solve on strips over NCCL, geometry
    replicated, RAS blocks sharded) -- strong scaling of the metric's wall
    time.  Device time with CUDA events, max over ranks."""
    import torch

    import paper_2401_06747_b200 as sp
    from oracle.oracle import synth  # input generator only
    from paper_2401_06747_b200.strips import StripSolver
    try:
        cfg = sp.PipelineConfig()
        f = torch.from_numpy(synth(H, W, C, seed=0)).cuda()
        solver = StripSolver.distributed(H, W, C, cfg=cfg.solver().cfg)
        sp.run_pipeline(sp.Image(f), cfg, solver=solver)
        torch.cuda.synchronize()
        stream = torch.cuda.current_stream()
        _barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            mask, st, hist, _ = sp.run_pipeline(sp.Image(f), cfg, solver=solver)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = _max_over_ranks(e0.elapsed_time(e1) / steps, world)
        return {"value_s": ms / 1e3, "ms_per_step": ms, "n_strips": world,
                "partitioned_levels": solver.La, "final_mse": st.mse,
                "mask_count": mask.count, "scaling": "strong (one 4K image on N GPUs)"}
    except Exception as e:  # reported, never fatal to the replica measurement
        return {"error": f"{type(e).__name__}: {e}"}


def run_ours(args):
    import numpy as np
    import torch

    world, rank, local = _dist()
    import paper_2401_06747_b200 as sp
    from paper_2401_06747_b200 import _lib
    from paper_2401_06747_b200.solver import GridHierarchy, MultigridConfig
    from oracle.oracle import synth  # input generator only

    lib = _lib.load()
    strips_mode = args.partition == "strips"
    # replicas: one image per rank; strips: one image cut over the ranks
    f_host = synth(H, W, C, seed=0 if strips_mode else rank)
    f_dev = torch.from_numpy(f_host).cuda()
    f_pinned = torch.from_numpy(f_host).pin_memory()
    cfg = sp.PipelineConfig()
    stream = torch.cuda.current_stream()
    solver = None
    if strips_mode:
        from paper_2401_06747_b200.strips import StripSolver
        solver = (StripSolver.distributed(H, W, C, cfg=cfg.solver().cfg) if world > 1
                  else StripSolver(H, W, C, strips=1, cfg=cfg.solver().cfg))

    def step_device():
        mask, st, hist, _ = sp.run_pipeline(sp.Image(f_dev), cfg, solver=solver)
        return mask, st, hist

    for _ in range(args.warmup):
        mask, st, hist = step_device()
    torch.cuda.synchronize()

    # ---- device-resident timed region -------------------------------------
    _barrier(world)
    torch.cuda.synchronize()
    lib.sp_launch_count(1)
    lib.sp_work_count(0, 1)
    lib.sp_work_count(1, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        e0.record(stream)
        for _ in range(args.steps):
            mask, st, hist = step_device()
        e1.record(stream)
        torch.cuda.synchronize()
    launches = lib.sp_launch_count(0) // max(1, args.steps)
    work_img = lib.sp_work_count(0, 0) / max(1, args.steps)
    work_blk = lib.sp_work_count(1, 0) / max(1, args.steps)
    _barrier(world)
    ms = e0.elapsed_time(e1) / args.steps
    ms = _max_over_ranks(ms, world)

    # ---- end-to-end through the public API with host buffers --------------
    h2d = f_pinned.numel() * f_pinned.element_size()
    d2h = 0

    def step_e2e():
        m_e, st_e, _, _ = sp.run_pipeline(sp.Image(f_pinned), cfg, solver=solver)
        mask_h = m_e.indicator          # D2H: mask (u8)
        g_h = st_e.g.data               # D2H: stored values (dense f32 image)
        return mask_h.nbytes + g_h.nbytes

    step_e2e()  # untimed warm-up of the host path (page-locked staging blocks)
    _barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        d2h = step_e2e()
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / args.steps
    e2e_s = _max_over_ranks(e2e_s, world)

    # ---- per-kernel roofline on the finest level (CUDA events) ------------
    peak, peak_kind = _peaks()
    kern = {}
    hier = GridHierarchy.build(sp.Mask(mask.tensor()), sp.Image(f_dev.float()),
                               MultigridConfig(), channels=C)
    bsym = torch.empty_like(f_dev, dtype=torch.float32)
    from paper_2401_06747_b200.solver import _masked_rhs
    bsym = _masked_rhs(f_dev.float().contiguous(), mask.tensor())
    hier.solve_sym(bsym, tol=1e-4, cascade=True)
    import ctypes
    names = {0: "k_ws_resid<0> (sym_residual sweep)", 1: "k_oras_warp (ORAS local CG)",
             2: "k_oras_blend", 3: "k_ws_resid<1> (residual + restriction)",
             4: "k_ws_prolong (prolongation + add + enforce)"}
    for which in (0, 1, 2, 3, 4):
        t_ms, nbytes = ctypes.c_double(), ctypes.c_double()
        _lib.call("sp_hier_bench", hier._h, which, 20, ctypes.byref(t_ms), ctypes.byref(nbytes),
                  _lib.stream())
        gbs = nbytes.value / (t_ms.value * 1e-3) / 1e9
        kern[names[which]] = {"us": t_ms.value * 1e3, "bytes": nbytes.value,
                              "gbs": gbs, "frac": gbs / peak}
    dom = names[1]
    tr = _ncu_traffic("k_oras_warp")
    roof = {"bound": "hbm", "kernel": dom, "achieved": kern[dom]["gbs"], "peak": peak,
            "unit": "GB/s", "frac": kern[dom]["frac"],
            "traffic": tr["bytes"] if tr else None,
            "traffic_source": tr["source"] if tr else None,
            "peak_kind": peak_kind,
            "issue_utilization": tr.get("issue") if tr else None,
            "note": "dominant kernel = ORAS local CG (on-chip, latency bound: HBM frac is low "
                    "by nature, issue_utilization = ncu sm__inst_issued of the same capture); "
                    "stencil sweep roofline in `stencil_roofline`"}
    sten = names[0]
    trs = _ncu_traffic("k_ws_resid")
    stencil_roofline = {"bound": "hbm", "kernel": sten, "achieved": kern[sten]["gbs"],
                        "peak": peak, "unit": "GB/s", "frac": kern[sten]["frac"],
                        "traffic": trs["bytes"] if trs else None,
                        "traffic_source": trs["source"] if trs else None}

    # solver level: a warm finest V-cycle of the same hierarchy against the
    # SURVEY.md 8(d) algorithmic V-cycle traffic (68 B per finest px.ch:
    # (4/3) x (two fused smoothing sweeps + residual + restriction +
    # prolongation))
    u_w, _ = hier.solve_sym(bsym, tol=1e-4, cascade=True)
    nvc = 20
    hier.solve_sym(bsym, init=u_w, tol=None, cycles=2)
    torch.cuda.synchronize()
    v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    v0.record(stream)
    hier.solve_sym(bsym, init=u_w, tol=None, cycles=nvc)
    v1.record(stream)
    torch.cuda.synchronize()
    vc_ms = v0.elapsed_time(v1) / nvc
    vc_bytes = 68.0 * H * W * C
    solver = {"vcycle_ms": vc_ms, "alg_bytes": vc_bytes,
              "gbs": vc_bytes / (vc_ms * 1e-3) / 1e9,
              "frac_measured_peak": vc_bytes / (vc_ms * 1e-3) / 1e9 / peak,
              "frac_8tbs": vc_bytes / (vc_ms * 1e-3) / 1e9 / 8000.0,
              "note": "warm 4K RGB V-cycle (solver.py:283-300) incl. the solve's copies; "
                      "bytes = SURVEY.md 8(d) 68 B per finest px.ch"}
    pipe_work = {"image_px_vcycles": work_img, "block_px_vcycles": work_blk,
                 "mpix_iter_per_s": work_img / (ms * 1e-3) / 1e6,
                 "mpix_iter_per_s_incl_blocks": (work_img + work_blk) / (ms * 1e-3) / 1e6,
                 "note": "finest-level pixels x V-cycles per step (image solves; RAS 64x64 "
                         "block solves separately) / device step time"}

    strips = None if args.no_strips else run_strips(world, rank)
    strip_pipe = None
    if world > 1 and not strips_mode and not args.no_strips:
        strip_pipe = run_strip_pipeline(world, args.steps)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        est, step_s = _cpu_sampled(steps=2, warmup=0, threads_one=False)
        cpu = _cpu_line(est, step_s)

    # Mpixel-iterations/s: pixels x finest V-cycles of the step (dd + tonal)
    if rank == 0:
        line = {
            "metric": METRIC, "value": ms / 1e3, "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": False, "scaling": "strong" if strips_mode else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": _config(args, world, strips_mode),
            "result": {"final_mse": st.mse, "dd_mse": hist[-1][2], "mask_count": mask.count,
                       "images_per_s": (1 if strips_mode else world) / (ms / 1e3)},
            "roofline": roof, "stencil_roofline": stencil_roofline, "kernels": kern,
            "solver": solver, "throughput": pipe_work,
            "strips": strips,
            "strips_pipeline": strip_pipe,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--partition", choices=("replicas", "strips"), default="replicas",
                    help="N > 1: one image per GPU (default) or one image in row strips")
    ap.add_argument("--no-strips", action="store_true",
                    help="skip the 8K row-strip solve (configs[4])")
    args = ap.parse_args(argv)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
