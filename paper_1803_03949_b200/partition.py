"""Spatial partition of one reconstruction across ranks.

Blocks belong to hashed tiles of ``tile_blocks``^3 blocks; rank r owns the
tiles whose hash is r and additionally collects, integrates and retypes a
1-block margin around them.  Integration depends only on the (broadcast)
depth frame and pose, so every margin block is bit-identical to its owner's
copy and all of rank r's owned results -- types, vertices, GC decisions,
normals -- are exact without any halo exchange during the frame.  What
crosses ranks:

* per frame, the additive StatsRow counters (``allreduce_frame_stats``), from
  which every rank rebuilds the reference's global StatsRow, including the
  arena high-water mark (``StatsCombiner``);
* at extraction, the owned blocks (``export_owned`` / ``merge_compact``),
  merged into one store and compacted on the device.

Redundant margin work replaces communication; DESIGN.md section 6 has the
cost model.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .store import CompactMesh, SpatialStore

# Counters the device keeps over owned blocks only (margin work is not counted),
# so they sum exactly over ranks.
ADDITIVE = ("blocks_active", "vertices_live", "triangles_live", "vertices_recycled_total",
            "irregular_cube_count", "new_vertices", "vertices_freed", "changed_cubes",
            "normals_computed", "fallback_normals")


class StatsCombiner:
    """Global StatsRow columns from per-rank (owned-block) counters.

    All additive columns sum over ranks.  ``vertices_allocated_total`` is the
    reference arena's high-water mark; since every allocation of a frame
    precedes every free (mesher.py:591-634), it is
    max over frames of (global live at frame start + global allocations).
    """

    def __init__(self):
        self.live = 0
        self.count = 0

    def combine(self, summed: dict) -> dict:
        peak = self.live + int(summed["new_vertices"])
        self.count = max(self.count, peak)
        self.live = int(summed["vertices_live"])
        out = {k: int(summed[k]) for k in ADDITIVE}
        out["vertices_allocated_total"] = self.count
        return out


def sum_stats(per_rank: list) -> dict:
    return {k: sum(int(d[k]) for d in per_rank) for k in ADDITIVE}


def allreduce_frame_stats(stats: dict, group=None, device=None) -> dict:
    """Sum this rank's per-frame counters over the process group."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([int(stats[k]) for k in ADDITIVE], dtype=torch.int64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return dict(zip(ADDITIVE, (int(v) for v in t.tolist())))


def export_blocks(store: SpatialStore, owned_only: bool = True) -> dict:
    """Dense host arrays of this store's (owned) blocks."""
    L = _lib.load()
    n = C.c_int64()
    _lib.check(L.vm_export_blocks(store._h, int(owned_only), C.byref(n), *([None] * 8)))
    k = n.value
    out = dict(coords=np.zeros((k, 3), np.int32), tsdf=np.zeros((k, 512)),
               weight=np.zeros((k, 512), np.int32), type_prev=np.zeros((k, 512), np.uint8),
               type_curr=np.zeros((k, 512), np.uint8), birth=np.zeros((k, 1536), np.int32),
               param=np.zeros((k, 1536)), normal=np.zeros((k, 1536, 3)))
    if k:
        _lib.check(L.vm_export_blocks(store._h, int(owned_only), C.byref(n),
                                      *[_lib.ptr(out[a]) for a in ("coords", "tsdf", "weight",
                                                                     "type_prev", "type_curr",
                                                                     "birth", "param", "normal")]))
    return out


def merge_stores(exports: list, cube_size: float, table_size: int = 1 << 21) -> SpatialStore:
    """One device store holding the union of the ranks' owned blocks."""
    st = SpatialStore(cube_size, table_size=table_size)
    for ex in exports:
        n = len(ex["coords"])
        if n:
            _lib.check(_lib.load().vm_import_blocks(
                st._h, n, *[_lib.ptr(np.ascontiguousarray(ex[a])) for a in
                            ("coords", "tsdf", "weight", "type_prev", "type_curr", "birth", "param",
                             "normal")]))
    st._touch()
    return st


def merge_compact(exports: list, cube_size: float, current_frame: int,
                  table_size: int = 1 << 21) -> CompactMesh:
    """store.py:388-425 over the union of the ranks' owned blocks."""
    return merge_stores(exports, cube_size, table_size).compact_mesh(current_frame)


class PartitionedEngine:
    """``Engine`` for one rank of a spatially partitioned reconstruction.

    Every rank feeds the same (broadcast) depth frames; ``fuse_frame`` returns
    the reference's *global* StatsRow (one int64 all-reduce per frame).
    ``compact`` gathers the owned blocks and returns the merged mesh on every
    rank.  ``group`` is a torch.distributed process group (NCCL or gloo).
    """

    def __init__(self, config, intrinsics, group=None, tile_blocks: int = 8, device=None):
        import dataclasses
        import torch.distributed as dist
        from .engine import Engine
        self.group = group
        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)
        self.device = device
        self.engine = Engine(dataclasses.replace(config, rank=self.rank, nranks=self.nranks,
                                                 tile_blocks=tile_blocks), intrinsics)
        self.combiner = StatsCombiner()
        self.stats = []

    def fuse_frame(self, depth, pose):
        from .engine import StatsRow
        row = self.engine.fuse_frame(depth, pose)
        g = self.combiner.combine(allreduce_frame_stats(self.engine.device_stats[-1], self.group,
                                                        self.device))
        out = StatsRow(frame=row.frame, blocks_active=g["blocks_active"],
                       vertices_live=g["vertices_live"], triangles_live=g["triangles_live"],
                       vertices_allocated_total=g["vertices_allocated_total"],
                       vertices_recycled_total=g["vertices_recycled_total"],
                       irregular_cube_count=g["irregular_cube_count"], fusion_ms=row.fusion_ms,
                       meshing_ms=row.meshing_ms, compact_ms=0.0)
        self.stats.append(out)
        return out

    def compact(self) -> CompactMesh:
        import torch.distributed as dist
        mine = export_blocks(self.engine.store, owned_only=True)
        parts = [None] * self.nranks
        dist.all_gather_object(parts, mine, group=self.group)
        return merge_compact(parts, self.engine.store.cube_size, self.engine.frame_index,
                             self.engine.store.table_size)


__all__ = ["PartitionedEngine", "StatsCombiner", "sum_stats", "allreduce_frame_stats", "export_blocks", "merge_stores",
           "merge_compact", "ADDITIVE"]
