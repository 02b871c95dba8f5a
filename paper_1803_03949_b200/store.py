"""Device-resident spatial store (mirror of reference pkg/src/voxmesh/store.py).

``SpatialStore`` owns one B200 engine (``vm_create``): the bucketed block hash
table, the SoA block heap, and the vertex / triangle arenas all live in HBM
(layout: DESIGN.md section 2).  The reference's host-side views -- ``Block``
arrays, ``VertexPool`` / ``TrianglePool`` attributes, ``blocks()`` in sorted
order -- are served from a read-only host snapshot that is refreshed lazily
after any mutating call.  Mutating a snapshot array does not write back; use
``set_block_samples`` to upload corner samples.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass
from typing import Iterator, NamedTuple, Optional

import numpy as np

from . import _lib
from .errors import ConsistencyError

BLOCK_SIZE = 8
CUBES_PER_BLOCK = BLOCK_SIZE ** 3
HASH_P1, HASH_P2, HASH_P3 = 73856093, 19349669, 83492791
DEFAULT_TABLE_SIZE = 1 << 20
_KEY_OFFSET = 1 << 20
_KEY_SPAN = 1 << 21


class Axis(enum.IntEnum):
    X = 0
    Y = 1
    Z = 2


class EdgeKey(NamedTuple):
    """A cube edge named by its owning cube (global coordinate) and axis."""

    cube: tuple
    axis: int


def hash_block(coord, table_size: int = DEFAULT_TABLE_SIZE) -> int:
    """store.py:84-87 -- the device uses the same function (csrc/vm_device.cuh)."""
    x, y, z = (int(v) for v in coord)
    return ((x * HASH_P1) ^ (y * HASH_P2) ^ (z * HASH_P3)) % table_size


def pack_coord(x: int, y: int, z: int) -> int:
    return (((x + _KEY_OFFSET) * _KEY_SPAN) + (y + _KEY_OFFSET)) * _KEY_SPAN + (z + _KEY_OFFSET)


@dataclass
class Block:
    """Host snapshot of one 8x8x8 brick (arrays indexed [x, y, z])."""

    coord: tuple
    tsdf: np.ndarray
    weight: np.ndarray
    type_prev: np.ndarray
    type_curr: np.ndarray
    edge_vertex: np.ndarray
    triangles: np.ndarray


@dataclass
class CompactMesh:
    positions: np.ndarray   # float64 (V, 3)
    normals: np.ndarray     # float64 (V, 3)
    ages: np.ndarray        # int64 (V,)
    indices: np.ndarray     # int32 (T, 3)


class VertexPoolView:
    """Snapshot of the device vertex arena with VertexPool's attribute names."""

    def __init__(self, store: "SpatialStore"):
        L = _lib.load()
        c = store._counters()
        n = c["vertex_count"]
        self.count = n
        self.recycled_total = c["vertex_recycled_total"]
        self.allocation_events = c["vertex_allocation_events"]
        self.max_vertices = store.max_vertices
        self.position = np.zeros((n, 3))
        self.normal = np.zeros((n, 3))
        self.color = np.zeros((n, 3))
        ref = np.zeros(n, np.int32)
        birth = np.zeros(n, np.int32)
        alive = np.zeros(n, np.uint8)
        free = np.zeros(c["vertex_free"], np.int32)
        _lib.check(L.vm_snapshot_vertices(store._h, n, _lib.ptr(self.position), _lib.ptr(self.normal),
                                          _lib.ptr(ref), _lib.ptr(birth), _lib.ptr(alive),
                                          _lib.ptr(free)))
        self.refcount = ref.astype(np.int64)
        self.birth_frame = birth.astype(np.int64)
        self.alive = alive.astype(bool)
        self.free = [int(h) for h in free]

    @property
    def live_count(self) -> int:
        return self.count - len(self.free)


class TrianglePoolView:
    def __init__(self, store: "SpatialStore"):
        L = _lib.load()
        c = store._counters()
        n = c["triangle_count"]
        self.count = n
        self.recycled_total = c["triangle_recycled_total"]
        verts = np.zeros((n, 3), np.int32)
        alive = np.zeros(n, np.uint8)
        free = np.zeros(c["triangle_free"], np.int32)
        _lib.check(L.vm_snapshot_triangles(store._h, n, _lib.ptr(verts), _lib.ptr(alive),
                                           _lib.ptr(free)))
        self.vertices = verts.astype(np.int64)
        self.alive = alive.astype(bool)
        self.free = [int(h) for h in free]

    @property
    def live_count(self) -> int:
        return self.count - len(self.free)


class SpatialStore:
    """Block hash table plus vertex/triangle arenas on the GPU."""

    def __init__(self, cube_size: float, table_size: int = DEFAULT_TABLE_SIZE,
                 max_vertices: Optional[int] = None, initial_blocks: int = 0,
                 initial_vertices: int = 0, initial_triangles: int = 0, rank: int = 0,
                 nranks: int = 1, tile_blocks: int = 8, halo_exchange: bool = False):
        if cube_size <= 0:
            raise ValueError("cube_size must be positive")
        self.cube_size = float(cube_size)
        self.block_extent = self.cube_size * BLOCK_SIZE
        self.table_size = int(table_size)
        self.max_vertices = max_vertices
        L = _lib.load()
        self.rank, self.nranks = int(rank), int(nranks)
        cfg = _lib.StoreConfig(self.cube_size, self.table_size, int(max_vertices or 0),
                               int(initial_blocks), int(initial_vertices), int(initial_triangles),
                               self.rank, self.nranks, int(tile_blocks), int(bool(halo_exchange)))
        h = C.c_void_p()
        _lib.check(L.vm_create(C.byref(cfg), C.byref(h)))
        self._h = h
        self._version = 0
        self._snap = None
        self._snap_version = -1
        self.degenerate_interpolations = 0

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            _lib._lib.vm_destroy(h)
            self._h = None

    # -- bookkeeping -------------------------------------------------------
    def _touch(self):
        self._version += 1

    def _counters(self) -> dict:
        c = _lib.CountersC()
        _lib.check(_lib.load().vm_counters(self._h, C.byref(c)))
        return {k: int(getattr(c, k)) for k in _lib.COUNTER_FIELDS}

    def snapshot_arrays(self) -> dict:
        """Dense host copies of every block, sorted by coordinate (the order of
        ``blocks()``): coords (n, 3), tsdf / weight / type_prev / type_curr
        (n, 8, 8, 8) -- the bulk form of the per-block views."""
        n = self._counters()["block_count"]
        out = dict(coords=np.zeros((n, 3), np.int32), tsdf=np.zeros((n, 8, 8, 8)),
                   weight=np.zeros((n, 8, 8, 8), np.int32), type_prev=np.zeros((n, 8, 8, 8), np.uint8),
                   type_curr=np.zeros((n, 8, 8, 8), np.uint8))
        _lib.check(_lib.load().vm_snapshot_blocks(self._h, n, *[_lib.ptr(out[k]) for k in
                                                               ("coords", "tsdf", "weight", "type_prev",
                                                                "type_curr")], None, None))
        c = out["coords"]
        order = np.lexsort((c[:, 2], c[:, 1], c[:, 0])) if n else np.zeros(0, int)
        return {k: v[order] for k, v in out.items()}

    def _snapshot(self):
        if self._snap_version == self._version and self._snap is not None:
            return self._snap
        n = self._counters()["block_count"]
        coords = np.zeros((n, 3), np.int32)
        tsdf = np.zeros((n, 8, 8, 8))
        weight = np.zeros((n, 8, 8, 8), np.int32)
        tp = np.zeros((n, 8, 8, 8), np.uint8)
        tc = np.zeros((n, 8, 8, 8), np.uint8)
        ev = np.zeros((n, 8, 8, 8, 3), np.int32)
        tri = np.zeros((n, 8, 8, 8, 5), np.int32)
        _lib.check(_lib.load().vm_snapshot_blocks(self._h, n, *[_lib.ptr(a) for a in
                                                               (coords, tsdf, weight, tp, tc, ev, tri)]))
        order = np.lexsort((coords[:, 2], coords[:, 1], coords[:, 0])) if n else np.zeros(0, int)
        blocks = {}
        for i in order:
            key = (int(coords[i, 0]), int(coords[i, 1]), int(coords[i, 2]))
            blocks[key] = Block(key, tsdf[i], weight[i], tp[i], tc[i], ev[i], tri[i])
        self._snap = blocks
        self._snap_version = self._version
        return blocks

    # -- block table -----------------------------------------------------------
    def block_of_point(self, p):
        q = np.floor(np.asarray(p, dtype=np.float64) / self.block_extent).astype(np.int64)
        return (int(q[0]), int(q[1]), int(q[2]))

    def contains(self, coords) -> np.ndarray:
        """Vectorised SpatialStore.get_block existence test (device lookup)."""
        c = _lib.coords_array(coords)
        out = np.zeros(len(c), np.uint8)
        _lib.check(_lib.load().vm_lookup(self._h, _lib.ptr(c), len(c), _lib.ptr(out)))
        return out.astype(bool)

    def get_block(self, coord) -> Optional[Block]:
        return self._snapshot().get(tuple(int(v) for v in coord))

    def get_or_allocate_block(self, coord) -> Block:
        self.set_block_samples([coord])
        return self.get_block(coord)

    def set_block_samples(self, coords, tsdf=None, weight=None) -> None:
        """Allocate blocks (if absent) and upload their corner samples.

        tsdf: (n, 8, 8, 8) float64 or None; weight: (n, 8, 8, 8) int32 or None.
        """
        c = _lib.coords_array(coords)
        t = None if tsdf is None else np.ascontiguousarray(np.asarray(tsdf, np.float64).reshape(len(c), 512))
        w = None if weight is None else np.ascontiguousarray(np.asarray(weight, np.int32).reshape(len(c), 512))
        self._touch()
        _lib.check(_lib.load().vm_set_blocks(self._h, _lib.ptr(c), len(c), _lib.ptr(t), _lib.ptr(w)))

    @property
    def block_count(self) -> int:
        return self._counters()["block_count"]

    @property
    def block_allocations(self) -> int:
        return self._counters()["block_allocations"]

    def blocks(self) -> Iterator[Block]:
        """All allocated blocks in sorted-coordinate order (deterministic)."""
        return iter(list(self._snapshot().values()))

    def block_coords(self) -> list:
        return list(self._snapshot().keys())

    # -- cube addressing ------------------------------------------------------
    @staticmethod
    def split_cube(cube):
        x, y, z = cube
        return ((x // BLOCK_SIZE, y // BLOCK_SIZE, z // BLOCK_SIZE),
                (x % BLOCK_SIZE, y % BLOCK_SIZE, z % BLOCK_SIZE))

    def corner_sample(self, cube):
        bc, lc = self.split_cube(cube)
        blk = self.get_block(bc)
        if blk is None:
            return 0.0, 0
        return float(blk.tsdf[lc]), int(blk.weight[lc])

    def owner_of_edge(self, cube, edge_index: int) -> EdgeKey:
        from .mc_tables import EDGE_AXIS, EDGE_OWNER_OFFSET
        off = EDGE_OWNER_OFFSET[edge_index]
        return EdgeKey((cube[0] + off[0], cube[1] + off[1], cube[2] + off[2]), EDGE_AXIS[edge_index])

    def resolve_edge(self, key: EdgeKey):
        bc, lc = self.split_cube(key.cube)
        blk = self.get_block(bc)
        if blk is None:
            return None
        return blk, lc, int(key.axis)

    def edge_vertex_handle(self, key: EdgeKey) -> int:
        slot = self.resolve_edge(key)
        if slot is None:
            return -1
        blk, lc, axis = slot
        return int(blk.edge_vertex[lc][axis])

    # -- pools ------------------------------------------------------------------
    @property
    def vertices(self) -> VertexPoolView:
        return VertexPoolView(self)

    @property
    def triangles(self) -> TrianglePoolView:
        return TrianglePoolView(self)

    def reserve(self, blocks: int = 0, vertices: int = 0, triangles: int = 0) -> None:
        _lib.check(_lib.load().vm_reserve(self._h, int(blocks), int(vertices), int(triangles)))

    # -- compaction ---------------------------------------------------------------
    def compact_mesh(self, current_frame: int = 0) -> CompactMesh:
        """store.py:388-425 on the device: radix-sorted block order, scans, remap."""
        L = _lib.load()
        nv = C.c_int64()
        nt = C.c_int64()
        _lib.check(L.vm_compact(self._h, int(current_frame), C.byref(nv), C.byref(nt)))
        pos = np.zeros((nv.value, 3))
        nrm = np.zeros((nv.value, 3))
        ages = np.zeros(nv.value, np.int64)
        idx = np.zeros((nt.value, 3), np.int32)
        _lib.check(L.vm_compact_fetch(self._h, _lib.ptr(pos), _lib.ptr(nrm), _lib.ptr(ages),
                                      _lib.ptr(idx)))
        return CompactMesh(pos, nrm, ages, idx)

    def irregular_cube_count(self) -> int:
        out = C.c_int64()
        _lib.check(_lib.load().vm_irregular_count(self._h, C.byref(out)))
        return int(out.value)


__all__ = ["BLOCK_SIZE", "CUBES_PER_BLOCK", "Axis", "EdgeKey", "Block", "CompactMesh",
           "SpatialStore", "VertexPoolView", "TrianglePoolView", "hash_block", "pack_coord",
           "ConsistencyError"]
