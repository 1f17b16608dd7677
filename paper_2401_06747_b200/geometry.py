"""Discrete geometry over the stored-pixel set (geometry.py parity).

Mirrors /root/reference/pkg/src/sparsepaint/geometry.py:21-272.  The
densification loop drives the native workspace ``GeoWorkspace``
(csrc/geometry.cu): jump flooding, the Delaunay corner scan with radix
sort + unique, atomicMin rasterization and per-triangle sequential sums all
stay in HBM.  The public functions below return the reference's dataclasses
(numpy arrays) for drop-in use.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream
from .grid import Mask


@dataclass
class VoronoiLabels:
    """geometry.py:21-39."""

    labels: np.ndarray
    seeds: np.ndarray
    max_radius: float = 0.0

    @property
    def height(self) -> int:
        return self.labels.shape[0]

    @property
    def width(self) -> int:
        return self.labels.shape[1]

    @property
    def nseeds(self) -> int:
        return self.seeds.shape[0]


@dataclass
class DelaunayMesh:
    """geometry.py:42-59."""

    vertices: np.ndarray
    triangles: np.ndarray
    edges: np.ndarray
    degenerate: bool = False

    @property
    def ntriangles(self) -> int:
        return self.triangles.shape[0]


@dataclass
class CellErrors:
    """geometry.py:62-73."""

    sums: np.ndarray
    argmax_flat: np.ndarray
    argmax_val: np.ndarray
    unassigned: float = 0.0

    @property
    def total(self) -> float:
        return float(self.sums.sum()) + self.unassigned


def steps_for(max_dim: int, start_hint) -> np.ndarray:
    """geometry.py:76-89 (host mirror of the schedule the native
    workspace builds): [1] followed by the halving sequence."""
    if start_hint is not None and start_hint >= 1:
        start = 1 << max(0, math.ceil(math.log2(max(1.0, start_hint))))
        start = min(start, max(1, max_dim // 2))
    elif max_dim >= 2:
        start = 1 << (math.ceil(math.log2(max_dim)) - 1)
    else:
        start = 1
    steps = [1]
    s = start
    while s >= 1:
        steps.append(s)
        s //= 2
    return np.array(steps, dtype=np.int64)


class GeoWorkspace:
    """Native per-(H, W) geometry workspace (sp_geo_*)."""

    def __init__(self, height: int, width: int):
        self.height, self.width = height, width
        self._g = ctypes.c_void_p()
        call("sp_geo_create", ctypes.byref(self._g), height, width)
        self.m = 0
        self.ntris = 0
        self.max_radius = 0.0
        self.nsteps = 0

    def __del__(self):
        g = getattr(self, "_g", None)
        if g is not None and g.value:
            try:
                _lib.load().sp_geo_destroy(g)
            except Exception:
                pass
            self._g = None

    def voronoi(self, mask_t: torch.Tensor, start_hint=None):
        m = ctypes.c_long()
        rad = ctypes.c_double()
        ns = ctypes.c_int()
        hint = -1.0 if start_hint is None else float(start_hint)
        call("sp_geo_voronoi", self._g, ptr(mask_t), hint, ctypes.byref(m),
             ctypes.byref(rad), ctypes.byref(ns), stream())
        self.m, self.max_radius, self.nsteps = m.value, rad.value, ns.value
        self.ntris = 0
        return self.m, self.max_radius

    def delaunay(self):
        t = ctypes.c_long()
        call("sp_geo_delaunay", self._g, ctypes.byref(t), stream())
        self.ntris = t.value
        return self.ntris

    def accumulate(self, err_t: torch.Tensor, voronoi=False):
        call("sp_geo_accumulate", self._g, ptr(err_t), int(bool(voronoi)), stream())

    def select(self, mask_t: torch.Tensor, nbuckets: int, want: int) -> int:
        p = ctypes.c_long()
        call("sp_geo_select", self._g, ptr(mask_t), int(nbuckets), int(want), ctypes.byref(p),
             stream())
        return p.value

    def fill_highest_error(self, err_t, mask_t, want: int):
        call("sp_geo_fill_highest_error", self._g, ptr(err_t), ptr(mask_t), int(want), stream())

    def load(self, lab_t: torch.Tensor, seeds):
        """Install caller labels / seed rows (e.g. a user VoronoiLabels)."""
        seeds = np.asarray(seeds).reshape(-1, 2)
        sy = _lib.to_dev(seeds[:, 0].astype(np.int32))
        sx = _lib.to_dev(seeds[:, 1].astype(np.int32))
        lab_c = lab_t.to(torch.int32).contiguous()   # alive until the launch is queued
        call("sp_geo_load", self._g, ptr(lab_c), ptr(sy), ptr(sx), int(seeds.shape[0]),
             stream())
        self.m = int(seeds.shape[0])
        self.ntris = 0

    # -- row-strip partition (StripGeometry) ------------------------------
    def corner_keys(self, r0: int, r1: int) -> torch.Tensor:
        """Sorted unique triangle keys of the corners in rows [r0, r1)
        (int64 view of the packed u64 keys)."""
        n = ctypes.c_long()
        call("sp_geo_corner_keys", self._g, int(r0), int(r1), ctypes.byref(n), stream())
        keys = torch.empty(n.value, dtype=torch.int64, device=_lib.device())
        if n.value:
            call("sp_geo_keys_copy", self._g, ptr(keys), n.value, stream())
        return keys

    def delaunay_from_keys(self, keys: torch.Tensor) -> int:
        t = ctypes.c_long()
        keys = keys.contiguous()
        call("sp_geo_delaunay_from_keys", self._g, ptr(keys), int(keys.numel()),
             ctypes.byref(t), stream())
        self.ntris = t.value
        return self.ntris

    def raster_rows(self, r0: int, r1: int):
        call("sp_geo_raster_rows", self._g, int(r0), int(r1), stream())

    def assign_rows(self, r0: int, r1: int) -> torch.Tensor:
        out = torch.empty((r1 - r0, self.width), dtype=torch.int32, device=_lib.device())
        call("sp_geo_assign_rows", self._g, ptr(out), int(r0), int(r1), 0, stream())
        return out

    def set_assign_rows(self, rows: torch.Tensor, r0: int, r1: int):
        rows = rows.to(torch.int32).contiguous()
        call("sp_geo_assign_rows", self._g, ptr(rows), int(r0), int(r1), 1, stream())

    def reduce_range(self, err_t: torch.Tensor, t0: int, t1: int):
        call("sp_geo_reduce_range", self._g, ptr(err_t), int(t0), int(t1), stream())

    def set_buckets(self, sums, amax, aval, t0: int):
        sums, amax, aval = sums.contiguous(), amax.contiguous(), aval.contiguous()
        call("sp_geo_set_buckets", self._g, ptr(sums), ptr(amax), ptr(aval), int(t0),
             int(t0 + sums.numel()), stream())

    # -- exports -----------------------------------------------------------
    def labels_tensor(self):
        lab = torch.empty((self.height, self.width), dtype=torch.int32, device=_lib.device())
        call("sp_geo_export", self._g, ptr(lab), None, None, None, None, None, None, 0, stream())
        return lab

    def seeds_tensor(self):
        sy = torch.empty(self.m, dtype=torch.int32, device=_lib.device())
        sx = torch.empty(self.m, dtype=torch.int32, device=_lib.device())
        call("sp_geo_export", self._g, None, ptr(sy), ptr(sx), None, None, None, None, 0,
             stream())
        return torch.stack([sy, sx], dim=1)

    def triangles_tensor(self):
        tris = torch.empty((self.ntris, 3), dtype=torch.int32, device=_lib.device())
        if self.ntris:
            call("sp_geo_export", self._g, None, None, None, ptr(tris), None, None, None, 0,
                 stream())
        return tris

    def buckets(self, n):
        sums = torch.empty(n, dtype=torch.float64, device=_lib.device())
        amax = torch.empty(n, dtype=torch.int64, device=_lib.device())
        aval = torch.empty(n, dtype=torch.float64, device=_lib.device())
        if n:
            call("sp_geo_export", self._g, None, None, None, None, ptr(sums), ptr(amax),
                 ptr(aval), int(n), stream())
        return sums, amax, aval


class DistGather:
    """All-gather of variable-length 1-D tensors over the current
    ``torch.distributed`` group: device tensors under NCCL, host copies
    under other backends (gloo: the CPU harness, ranks sharing one GPU)."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.dev = None if dist.get_backend() == "nccl" else torch.device("cpu")

    def allgather_var(self, t: torch.Tensor):
        home = t.device
        dev = self.dev or home
        t = t.reshape(-1).to(dev)
        n = torch.tensor([t.numel()], dtype=torch.int64, device=dev)
        ns = [torch.empty_like(n) for _ in range(self.world)]
        self.dist.all_gather(ns, n)
        ns = [int(x.item()) for x in ns]
        pad = torch.zeros(max(ns), dtype=t.dtype, device=dev)
        pad[:t.numel()] = t
        out = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(out, pad)
        return [o[:k].to(home) for o, k in zip(out, ns)]


class StripGeometry:
    """The Delaunay step and the accumulate of `delaunay_densify` on row
    strips (csrc/geometry.cu geo_corner_keys ...):
    rank `rank` of `comm` scans the corners of its rows, the sorted key lists
    are all-gathered and merged; it rasterises its rows, the assignment rows
    are all-gathered; it reduces its contiguous range of triangles over the
    full map, and the bucket ranges are all-gathered.  Jump flooding and the
    selection stay replicated.  Triangles, buckets and picks are bit-identical
    to the unpartitioned workspace for every strip count (every triangle's
    sequential f64 sum stays on one rank)."""

    def __init__(self, ws: GeoWorkspace, rows, rank: int, comm):
        self.ws, self.rows, self.rank, self.comm = ws, list(rows), rank, comm
        self.P = len(self.rows)
        self.calls = 0

    def delaunay(self) -> int:
        r0, r1 = self.rows[self.rank]
        parts = self.comm.allgather_var(self.ws.corner_keys(r0, r1))
        self.calls += 1
        return self.ws.delaunay_from_keys(torch.cat(parts))

    def accumulate(self, err_t: torch.Tensor):
        ws, P, rank = self.ws, self.P, self.rank
        r0, r1 = self.rows[rank]
        ws.raster_rows(r0, r1)
        parts = self.comm.allgather_var(ws.assign_rows(r0, r1))
        for p, part in enumerate(parts):
            if p != rank:
                a, b = self.rows[p]
                ws.set_assign_rows(part.view(b - a, ws.width), a, b)
        T = ws.ntris
        bounds = [T * p // P for p in range(P + 1)]
        t0, t1 = bounds[rank], bounds[rank + 1]
        ws.reduce_range(err_t, t0, t1)
        sums, amax, aval = ws.buckets(T)
        # one gather: sums, argmax (int64 bits) and argmax value of the range
        mine = torch.stack([sums[t0:t1], amax[t0:t1].view(torch.float64), aval[t0:t1]])
        got = self.comm.allgather_var(mine)
        for p, g in enumerate(got):
            if p != rank and g.numel():
                g = g.view(3, -1)
                ws.set_buckets(g[0], g[1].contiguous().view(torch.int64), g[2], bounds[p])
        self.calls += 1


_WS: dict = {}


def workspace(height, width) -> GeoWorkspace:
    """Per-thread-free cache of workspaces by geometry."""
    ws = _WS.get((height, width))
    if ws is None:
        if len(_WS) > 4:
            _WS.clear()
        ws = GeoWorkspace(height, width)
        _WS[(height, width)] = ws
    return ws


def jump_flood_voronoi(mask: Mask, start_hint: float | None = None) -> VoronoiLabels:
    """geometry.py:92-110."""
    m_t = mask.tensor()
    ws = workspace(*m_t.shape)
    ws.voronoi(m_t, start_hint)
    return VoronoiLabels(labels=ws.labels_tensor().cpu().numpy(),
                         seeds=ws.seeds_tensor().cpu().numpy(),
                         max_radius=ws.max_radius)


def _edges_device(lab: torch.Tensor) -> torch.Tensor:
    """Unique label-adjacency pairs (geometry.py:125-138), on the device."""
    pairs = []
    for a, b in ((lab[:, :-1], lab[:, 1:]), (lab[:-1, :], lab[1:, :])):
        a, b = a.reshape(-1).long(), b.reshape(-1).long()
        keep = a != b
        lo, hi = torch.minimum(a[keep], b[keep]), torch.maximum(a[keep], b[keep])
        pairs.append(lo * (1 << 32) + hi)
    keys = torch.unique(torch.cat(pairs)) if pairs else torch.empty(0, dtype=torch.int64)
    return torch.stack([keys >> 32, keys & 0xFFFFFFFF], dim=1).to(torch.int32)


def delaunay_from_voronoi(labels: VoronoiLabels) -> DelaunayMesh:
    """geometry.py:113-185.  Re-floods only if the workspace does not hold
    these labels already."""
    lab = _lib.to_dev(np.asarray(labels.labels, np.int32))
    h, w = lab.shape
    ws = workspace(h, w)
    ws.load(lab, np.asarray(labels.seeds))
    ws.delaunay()
    tris = ws.triangles_tensor().cpu().numpy()
    edges = _edges_device(lab).cpu().numpy()
    return DelaunayMesh(vertices=np.asarray(labels.seeds).copy(), triangles=tris,
                        edges=edges, degenerate=tris.shape[0] == 0)


def accumulate_errors(mesh: DelaunayMesh, error_map, labels: VoronoiLabels) -> CellErrors:
    """geometry.py:197-223: pixel -> lowest containing triangle (hull
    exterior -> lowest triangle of its cell seed); sequential row-major sums
    and first argmax per triangle."""
    from .kernels import cuda_impl as K
    err = np.asarray(error_map, dtype=np.float64)
    if err.ndim != 2:
        raise ValueError("error map must be a single (H, W) plane")
    if np.any(err < 0):
        raise ValueError("error map must be nonnegative")
    if mesh.ntriangles == 0:
        return CellErrors(sums=np.zeros(0), argmax_flat=np.zeros(0, np.int64),
                          argmax_val=np.zeros(0), unassigned=float(err.sum()))
    h, w = err.shape
    tris = np.ascontiguousarray(mesh.triangles.astype(np.int64))
    vy = np.ascontiguousarray(mesh.vertices[:, 0].astype(np.int64))
    vx = np.ascontiguousarray(mesh.vertices[:, 1].astype(np.int64))
    assign = K.assign_triangles(tris, vy, vx, h, w)
    smt = _seed_min_triangle(mesh, labels.nseeds)
    assign = K.fallback_assign(assign, labels.labels, smt)
    sums, amax, aval = K.reduce_cells(assign, err, mesh.ntriangles)
    return CellErrors(sums=sums, argmax_flat=amax, argmax_val=aval)


def _seed_min_triangle(mesh: DelaunayMesh, nseeds: int) -> np.ndarray:
    """geometry.py:188-194 (min triangle index per vertex)."""
    out = np.full(nseeds, -1, np.int32)
    if mesh.ntriangles:
        t = np.repeat(np.arange(mesh.ntriangles, dtype=np.int32), 3)
        v = mesh.triangles.ravel().astype(np.int64)
        np.minimum.at(out.view(np.uint32), v, t.view(np.uint32))
    return out


def voronoi_cell_errors(labels: VoronoiLabels, error_map):
    """geometry.py:226-244: bincount sums are sequential per cell in pixel
    order and lexsort picks the first maximum -- exactly reduce_cells with
    the labels as the assignment."""
    from .kernels import cuda_impl as K
    err = np.asarray(error_map, dtype=np.float64)
    return K.reduce_cells(np.asarray(labels.labels, np.int32), err, labels.nseeds)


def voronoi_weights(labels: VoronoiLabels, scheme: str = "inverse-log") -> np.ndarray:
    """geometry.py:247-264."""
    from .tonal import _cell_index, _voronoi_weights_t
    lab = _lib.to_dev(np.asarray(labels.labels, np.int32))
    seeds = _lib.to_dev(np.asarray(labels.seeds, np.int32))
    idx = _cell_index(lab, labels.nseeds)
    return _voronoi_weights_t(lab, seeds, idx, scheme).cpu().numpy()


def cell_weighted_average(labels: VoronoiLabels, weights, plane) -> np.ndarray:
    """geometry.py:267-272."""
    from .tonal import _cell_index, _cell_sum
    lab = _lib.to_dev(np.asarray(labels.labels, np.int32))
    idx = _cell_index(lab, labels.nseeds)
    vals = _lib.to_dev(np.asarray(weights, np.float64) * np.asarray(plane, np.float64))
    return _cell_sum(idx, vals).cpu().numpy()


def export_labels_ppm(labels: VoronoiLabels, path):
    """geometry.py:275-283 (debug dump)."""
    from .grid import Image
    from .pnm import write_image
    lab = labels.labels.astype(np.int64)
    r, g, b = (lab * 131 + 89) % 256, (lab * 197 + 53) % 256, (lab * 233 + 17) % 256
    write_image(path, Image(np.stack([r, g, b]).astype(np.float64)))


def export_mesh_text(mesh: DelaunayMesh, path):
    """geometry.py:286-294 (debug dump)."""
    with open(path, "w") as fh:
        for y, x in mesh.vertices:
            fh.write(f"v {x} {y}\n")
        for a, b in mesh.edges:
            fh.write(f"e {a} {b}\n")
        for a, b, c in mesh.triangles:
            fh.write(f"t {a} {b} {c}\n")
