"""The optimize pipeline: spatial then tonal stage (cli.py:34-257 parity).

``PipelineConfig`` is the reference's flat bag of tunables (cli.py:34-119)
with the same field names, defaults and validation; ``run_pipeline`` is the
call BASELINE.json's metric times (cli.py:251-257).  Everything between the
input upload and the final read-back runs on the device.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

from .grid import Image, Mask
from .solver import InpaintSolver, MultigridConfig, OrasConfig
from .spatial import (DensificationConfig, NlpeConfig, PsConfig, analytic_mask,
                      delaunay_densify, nlpe, probabilistic_sparsify, uniform_random_mask)
from .tonal import (InitConfig, RasTonalConfig, cgnr_tonal, initial_state,
                    neighbor_balance_init, ras_tonal, voronoi_richardson_init)

SPATIAL_METHODS = ("dd", "aa", "ps", "ps+nlpe", "random")
TONAL_METHODS = ("none", "balance", "voronoi-init", "cgnr", "ras", "ras+vi")


@dataclass
class PipelineConfig:
    """cli.py:34-119."""

    density: float = 0.05
    spatial: str = "dd"
    tonal: str = "ras+vi"
    seed: int = 0
    block: int = 32
    overlap: int = 6
    alpha: float = 1.0
    rho: float = 0.25
    levels: int = 0
    pre: int = 1
    post: int = 1
    cycles: int = 1
    mode: str = "fmg"
    tol: float = 1e-4
    max_cycles: int = 100
    dtype: str = "float32"
    iterations: int = 20
    growth: float = 1.0
    initial_fraction: float = -1.0
    initial_scheme: str = "laplacian-dither"
    init_sigma: float = 1.0
    ps_p: float = 0.3
    ps_q: float = 0.005
    nlpe_cycles: int = 5
    nlpe_candidates: int = 5
    tonal_block: int = 64
    tonal_overlap: int = 6
    local_iters: int = 30
    local_tol: float = 0.1
    inner_cycles: int = 2
    rel_improvement: float = 1e-3
    max_outer: int = 50
    final_tol: float = 1e-6
    vi_tau: float = 1.0
    vi_weights: str = "inverse-log"
    vi_steps: int = 20
    deterministic_output: bool = False

    def validate(self):
        if self.spatial not in SPATIAL_METHODS:
            raise ValueError(f"spatial must be one of {SPATIAL_METHODS}")
        if self.tonal not in TONAL_METHODS:
            raise ValueError(f"tonal must be one of {TONAL_METHODS}")
        if not 0 < self.density <= 1:
            raise ValueError("density must be in (0, 1]")

    def solver(self) -> InpaintSolver:
        return InpaintSolver(MultigridConfig(
            levels=self.levels, pre=self.pre, post=self.post, cycles=self.cycles,
            mode=self.mode, tol=self.tol if self.tol > 0 else None,
            max_cycles=self.max_cycles, dtype=self.dtype,
            oras=OrasConfig(block=self.block, overlap=self.overlap, alpha=self.alpha,
                            rho=self.rho)))

    def densification(self) -> DensificationConfig:
        frac = None if self.initial_fraction < 0 else self.initial_fraction
        return DensificationConfig(density=self.density, iterations=self.iterations,
                                   growth=self.growth, initial_fraction=frac,
                                   initial_scheme=self.initial_scheme,
                                   init_sigma=self.init_sigma, seed=self.seed)

    def ras(self) -> RasTonalConfig:
        return RasTonalConfig(block=self.tonal_block, overlap=self.tonal_overlap,
                              local_iters=self.local_iters, local_tol=self.local_tol,
                              inner_cycles=self.inner_cycles,
                              rel_improvement=self.rel_improvement, max_outer=self.max_outer,
                              final_tol=self.final_tol)

    def vi(self) -> InitConfig:
        return InitConfig(tau=self.vi_tau, weight_scheme=self.vi_weights,
                          max_steps=self.vi_steps, inner_cycles=self.inner_cycles,
                          final_tol=self.final_tol)


def run_spatial(f: Image, cfg: PipelineConfig, solver: InpaintSolver):
    """cli.py:206-225: (mask, history or None)."""
    n = f.height * f.width
    target = int(cfg.density * n)
    if cfg.spatial == "dd":
        mask, _, hist = delaunay_densify(f, cfg.densification(), solver)
        return mask, hist
    if cfg.spatial == "aa":
        return analytic_mask(f, cfg.density, dither="floyd-steinberg", sigma=cfg.init_sigma,
                             seed=cfg.seed), None
    if cfg.spatial == "random":
        return uniform_random_mask(f.height, f.width, target, cfg.seed), None
    ps_cfg = PsConfig(candidate_fraction=cfg.ps_p, return_fraction=cfg.ps_q, seed=cfg.seed)
    mask = probabilistic_sparsify(f, cfg.density, ps_cfg, solver)
    if cfg.spatial == "ps+nlpe":
        mask = nlpe(f, mask, NlpeConfig(cycles=cfg.nlpe_cycles, candidates=cfg.nlpe_candidates,
                                        seed=cfg.seed), solver)
    return mask, None


def run_tonal(f: Image, mask: Mask, cfg: PipelineConfig, solver: InpaintSolver):
    """cli.py:228-248: the final TonalState."""
    if cfg.tonal == "none":
        return initial_state(f, mask, solver, final_tol=cfg.final_tol)
    if cfg.tonal == "balance":
        u, _ = solver.inpaint(f, mask, tol=cfg.final_tol)
        return neighbor_balance_init(f, u, mask, solver, final_tol=cfg.final_tol)
    if cfg.tonal == "voronoi-init":
        return voronoi_richardson_init(f, mask, cfg.vi(), solver)
    if cfg.tonal == "cgnr":
        return cgnr_tonal(f, mask, solver=solver, rel_improvement=cfg.rel_improvement,
                          max_iters=cfg.max_outer, inner_cycles=cfg.inner_cycles,
                          final_tol=cfg.final_tol)
    if cfg.tonal == "ras":
        return ras_tonal(f, mask, cfg=cfg.ras(), solver=solver)
    vi = voronoi_richardson_init(f, mask, cfg.vi(), solver)
    return ras_tonal(f, mask, init=vi, cfg=cfg.ras(), solver=solver)


def run_pipeline(f: Image, cfg: PipelineConfig, solver=None):
    """cli.py:251-257: (mask, state, spatial history, seconds).  `solver`
    (optional, not in the reference) replaces ``cfg.solver()`` -- e.g. a
    `strips.StripSolver` that runs every inpainting solve on row strips."""
    cfg.validate()
    solver = cfg.solver() if solver is None else solver
    t0 = time.perf_counter()
    # one upload of a host image for the whole run (every stage reads f)
    f = Image(f.tensor())
    mask, spatial_hist = run_spatial(f, cfg, solver)
    state = run_tonal(f, mask, cfg, solver)
    return mask, state, spatial_hist, time.perf_counter() - t0
