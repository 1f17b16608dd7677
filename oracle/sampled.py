"""CPU baseline of the BASELINE.json workload by work-unit sampling at full
size.  TEST / MEASUREMENT INFRASTRUCTURE: only bench.py's cpu_baseline leg
and its `--impl reference` arm call this; nothing in the product path does.

Why sampling: the reference's full 3840x2160 RGB run (`run_pipeline`,
dd + ras+vi, cli.py:251-257) takes ~19 minutes of CPU (measured in the build
container by tests/golden/make_golden_large.py cfg4, the numba reference
itself), far above the few minutes a bench arm may take.  So each bench step
times a bounded sample of the SAME 4K workload -- the work units that carry
>= 90% of the reference's time -- on the oracle port (C kernel table under
OpenMP + numpy orchestration, bit-exact with the reference), and the
full-run figure is assembled from them:

    units (all at 3840x2160x3, the workload's own masks):
      vcycle_full   one finest-level V-cycle (solver.py:283-300) of the
                    image hierarchy: on the initial dithered mask (19,749 px,
                    densification iteration 0) and on the reference's final
                    5% mask (414,720 px); spatial V-cycles are charged the
                    mean of the two, tonal V-cycles the final-mask cost
      vcycle_local  one V-cycle of a 64x64 RAS block hierarchy (tonal.py:
                    120-131, cold local B / B^T products), 16 sampled blocks
                    of the final mask per step
      jfa / delaunay / accumulate   one densification geometry pass each
                    (geometry.py:92-223), on the initial and the final mask

    counts n_u and the reference's own seconds T_u: the census of the
    reference's 4K run (tests/golden/large_cfg4.json census_*: calls and
    seconds per unit, spatial at all threads, tonal single-threaded as the
    reference's RGB RAS is fastest that way).

    estimate = T_ref_total * sum_u n_u t_u / sum_u T_u

i.e. the reference's measured total (units + glue) rescaled by how fast
this host runs the same units; `covered` says what share of the reference's
time the units account for.  No size exponent is involved.
"""

from __future__ import annotations

import json
import os
import time

import numpy as np

from oracle import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
FIXTURE = os.path.join(os.path.dirname(HERE), "tests", "golden", "large_cfg4")
H, W, C = 2160, 3840, 3


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def set_threads(n):
    O.lib().ora_set_threads(int(n))


def get_threads():
    return int(O.lib().ora_get_threads())


def load_census():
    with open(FIXTURE + ".json") as fh:
        S = json.load(fh)
    G = np.load(FIXTURE + ".npz")
    final = np.unpackbits(G["final_mask_bits"])[:H * W].reshape(H, W).astype(np.uint8)
    return S, final


class Sampler:
    """Holds the 4K inputs and the per-unit timings of the oracle port."""

    def __init__(self, seed_blocks=0):
        O.build()
        self.S, final = load_census()
        self.f = O.synth(H, W, C, 0)
        init = O.analytic_mask(self.f, self.S["init_count"] / (H * W), dither="random",
                               sigma=1.0, seed=0, count=self.S["init_count"])
        self.masks = {"init": init, "final": final}
        self.cfg = O.SolverCfg()
        self.state = {}
        for k, m in self.masks.items():
            f32 = self.f.astype(np.float32)
            hier = self.cfg.hierarchy(m, f32)
            b = np.where(m[None].astype(bool), f32, 0).astype(np.float32)
            bsym = O.sym_rhs(b, m, 1.0)
            u = hier.cascade(C, np.float32)
            hier.enforce(0, u, bsym)
            err = O.error_map(u, self.f)
            _, _, rad = O.jump_flood_voronoi(m, None)
            self.state[k] = dict(hier=hier, bsym=bsym, u=u, err=err,
                                 hint=None if k == "init" else rad)
        # RAS 64x64 blocks of the final mask (tonal.py:309-386)
        d = O.build_decomposition(H, W, 64, 6)
        nbx = d["xs"].size
        rng = np.random.default_rng(seed_blocks)
        order = rng.permutation(d["nb"])
        self.blocks = []
        for bi in order:
            y0, x0 = int(d["ys"][bi // nbx]), int(d["xs"][bi % nbx])
            sub = np.ascontiguousarray(final[y0:y0 + d["bh"], x0:x0 + d["bw"]])
            if sub.sum() == 0:
                continue
            fb = self.f[:, y0:y0 + d["bh"], x0:x0 + d["bw"]].astype(np.float32)
            b = np.where(sub[None].astype(bool), fb, 0).astype(np.float32)
            self.blocks.append((self.cfg.hierarchy(sub, None), O.sym_rhs(b, sub, 1.0)))
        self.times = {k: [] for k in ("vcycle_init", "vcycle_final", "vcycle_local",
                                      "jfa_init", "jfa_final", "delaunay_init",
                                      "delaunay_final", "accumulate_init",
                                      "accumulate_final")}
        self._blk = 0

    def reset(self):
        for v in self.times.values():
            v.clear()

    def step(self, which, nlocal=16):
        """Time one unit sample on mask `which` ('init' / 'final'); returns
        the seconds the step took."""
        t_step = time.perf_counter()
        st = self.state[which]
        m = self.masks[which]
        t0 = time.perf_counter()
        st["hier"].vcycle(0, st["u"], st["bsym"])
        self.times[f"vcycle_{which}"].append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        lab, seeds, _ = O.jump_flood_voronoi(m, st["hint"])
        t1 = time.perf_counter()
        tris, _ = O.delaunay_from_voronoi(lab, seeds.shape[0])
        t2 = time.perf_counter()
        O.accumulate_errors(tris, st["err"], lab, seeds)
        t3 = time.perf_counter()
        self.times[f"jfa_{which}"].append(t1 - t0)
        self.times[f"delaunay_{which}"].append(t2 - t1)
        self.times[f"accumulate_{which}"].append(t3 - t2)
        # the 4K run does its ~110k local V-cycles back to back; one untimed
        # local V-cycle first wakes the OpenMP pool that the 4K units above
        # left parked (timed cold, the pool wake-ups dominate a 64x64
        # V-cycle: 15.9 vs 2.8 ms here, against the reference's own 3.3 ms)
        hier, bsym = self.blocks[self._blk % len(self.blocks)]
        u = np.zeros_like(bsym)
        hier.enforce(0, u, bsym)
        hier.vcycle(0, u, bsym)
        loc = []
        for _ in range(nlocal):
            hier, bsym = self.blocks[self._blk % len(self.blocks)]
            self._blk += 1
            u = np.zeros_like(bsym)
            hier.enforce(0, u, bsym)
            t0 = time.perf_counter()
            hier.vcycle(0, u, bsym)
            loc.append(time.perf_counter() - t0)
        self.times["vcycle_local"].append(float(np.mean(loc)))
        return time.perf_counter() - t_step

    def unit_means(self):
        mean = {k: float(np.mean(v)) for k, v in self.times.items() if v}
        g = lambda k: mean.get(k, mean.get(k.replace("_init", "_final"),  # noqa: E731
                                            mean.get(k.replace("_final", "_init"))))
        return {
            "vcycle_spatial": 0.5 * (g("vcycle_init") + g("vcycle_final")),
            "vcycle_tonal": g("vcycle_final"),
            "vcycle_local": mean["vcycle_local"],
            "jfa": 0.5 * (g("jfa_init") + g("jfa_final")),
            "delaunay": 0.5 * (g("delaunay_init") + g("delaunay_final")),
            "accumulate": 0.5 * (g("accumulate_init") + g("accumulate_final")),
        }

    def estimate(self):
        """Full-run estimate (seconds) from the unit means and the census."""
        S = self.S
        cs, ct = S["census_spatial"], S["census_tonal"]
        u = self.unit_means()
        rows = [
            ("vcycle_spatial", cs["vcycle_full"]),
            ("vcycle_tonal", ct["vcycle_full"]),
            ("vcycle_local", ct["vcycle_local"]),
            ("jfa", cs["jfa"]), ("delaunay", cs["delaunay"]), ("accumulate", cs["accumulate"]),
        ]
        ours = sum(r[1]["calls"] * u[r[0]] for r in rows)
        ref_units = sum(r[1]["seconds"] for r in rows)
        ref_total = S["seconds_spatial_wall"] + S["seconds_tonal"]
        return {
            "estimate_s": ref_total * ours / ref_units,
            "units_s": ours,
            "covered": ref_units / ref_total,
            "unit_means_s": u,
            "counts": {r[0]: r[1]["calls"] for r in rows},
            "reference_total_s": ref_total,
            "reference_units_s": ref_units,
        }

    def reference_note(self):
        S = self.S
        m = S.get("machine", {})
        return (f"reference (numba) 4K run measured in the build container: "
                f"{S['seconds_spatial_wall']:.0f} s spatial ({m.get('numba_threads')} threads) "
                f"+ {S['seconds_tonal']:.0f} s tonal (1 thread) on {m.get('cpu_count')}x "
                f"{m.get('cpu_model')}")
