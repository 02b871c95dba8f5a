"""Incremental Marching Cubes phases (mirror of reference pkg/src/voxmesh/mesher.py).

``extract_frame`` runs the device pipeline k_retype_place (typing, +refine,
implicit retriangulation, claim-based vertex placement) -> k_gc_normals (GC,
gradient normals, face-normal fallback) (csrc/vm_kernels.cuh) over an explicit
scope.  Strategies ``claim``, ``partition`` and ``serial`` are accepted; all run
the claim kernel (atomicCAS on the edge slot), since the result is independent
of the strategy, as the reference guarantees.

``meshing_scope`` / ``fused_halo`` are the reference's scope rules evaluated
on the host with device existence lookups; ``Engine.fuse_frame`` computes the
same sets on the device (k_scope_halo).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _lib
from .refine import RefineParams
from .store import BLOCK_SIZE, SpatialStore

STRATEGIES = ("serial", "claim", "partition")

_MINUS_OFFSETS = tuple((i, j, k) for i in (0, 1) for j in (0, 1) for k in (0, 1)
                       if (i, j, k) != (0, 0, 0))
_BOX_OFFSETS = tuple((i, j, k) for i in (-1, 0, 1) for j in (-1, 0, 1) for k in (-1, 0, 1))


def interpolate_vertex(d0: float, d1: float, p0, p1):
    """Zero crossing of the linear model through (p0, d0), (p1, d1)."""
    p0 = np.asarray(p0, dtype=np.float64)
    p1 = np.asarray(p1, dtype=np.float64)
    if d0 == d1:
        return 0.5 * (p0 + p1)
    return p0 + (d0 / (d0 - d1)) * (p1 - p0)


def meshing_scope(store: SpatialStore, collected):
    """mesher.py:499-527: (coord, cube mask or None) sorted by coordinate."""
    coll = [tuple(int(v) for v in c) for c in collected]
    if not coll:
        return []
    exists = store.contains(coll)
    full = {c for c, e in zip(coll, exists) if e}
    cand = [(c[0] - o[0], c[1] - o[1], c[2] - o[2]) for c in coll for o in _MINUS_OFFSETS]
    cex = store.contains(cand) if cand else []
    slabs: dict = {}
    for n, ok, o in zip(cand, cex, [o for _ in coll for o in _MINUS_OFFSETS]):
        if not ok or n in full:
            continue
        mask = slabs.get(n)
        if mask is None:
            mask = np.zeros((BLOCK_SIZE,) * 3, dtype=bool)
            slabs[n] = mask
        sl = tuple(slice(BLOCK_SIZE - 1, BLOCK_SIZE) if v else slice(None) for v in o)
        mask[sl] = True
    out = [(c, None) for c in full]
    out.extend(slabs.items())
    out.sort(key=lambda item: item[0])
    return out


def fused_halo(store: SpatialStore, collected):
    """mesher.py:530-543: allocated blocks within one step of a fused block."""
    coll = [tuple(int(v) for v in c) for c in collected]
    cand = sorted({(c[0] + o[0], c[1] + o[1], c[2] + o[2]) for c in coll for o in _BOX_OFFSETS})
    if not cand:
        return []
    ok = store.contains(cand)
    return [c for c, e in zip(cand, ok) if e]


def _masks_bytes(scope) -> Optional[np.ndarray]:
    if all(m is None for _, m in scope):
        return None
    out = np.zeros((len(scope), 64), np.uint8)
    for i, (_, m) in enumerate(scope):
        bits = np.ones(512, bool) if m is None else np.asarray(m, bool).reshape(512)
        out[i] = np.packbits(bits, bitorder="little")
    return out


def extract_frame(store: SpatialStore, scope, frame_index: int, strategy: str = "claim",
                  workers: int = 1, refine_params: Optional[RefineParams] = None,
                  halo=None) -> dict:
    """mesher.py:546-636 on the device.  Returns {"refined", "freed"}."""
    if strategy not in STRATEGIES:
        raise ValueError(f"unknown strategy {strategy!r}")
    scope = [(tuple(int(v) for v in c), m) for c, m in scope]
    if not scope:
        return {"refined": 0, "freed": 0}
    coords = _lib.coords_array([c for c, _ in scope])
    masks = _masks_bytes(scope)
    hc = None if halo is None else _lib.coords_array(halo)
    rp = refine_params or RefineParams(enabled=False)
    out = np.zeros(2, np.int64)
    store._touch()
    _lib.check(_lib.load().vm_extract(store._h, _lib.ptr(coords), _lib.ptr(masks), len(coords),
                                      _lib.ptr(hc), -1 if hc is None else len(hc),
                                      int(frame_index), _lib.STRATEGY_CODES[strategy],
                                      int(bool(rp.enabled)), float(rp.epsilon), _lib.ptr(out)))
    return {"refined": int(out[0]), "freed": int(out[1])}


def garbage_collect(store: SpatialStore, blocks) -> int:
    """mesher.py:333-356 on the device; returns the number of vertices freed."""
    c = _lib.coords_array(blocks)
    freed = C.c_int64()
    store._touch()
    _lib.check(_lib.load().vm_garbage_collect(store._h, _lib.ptr(c), len(c), C.byref(freed)))
    return int(freed.value)


def compute_normals(store: SpatialStore, blocks) -> None:
    """mesher.py:442-486 on the device (gradient + face-normal fallback)."""
    c = _lib.coords_array(blocks)
    store._touch()
    _lib.check(_lib.load().vm_compute_normals(store._h, _lib.ptr(c), len(c)))


__all__ = ["STRATEGIES", "interpolate_vertex", "meshing_scope", "fused_halo", "extract_frame",
           "garbage_collect", "compute_normals"]
