"""Spatial partition of one reconstruction across ranks.

Blocks belong to hashed tiles of ``tile_blocks``^3 blocks; rank r owns the
tiles whose hash is r and meshes its owned blocks plus a 1-block margin around
them, so all of its owned results -- types, vertex slots, GC decisions,
normals -- are exact.  Where the margin blocks' samples come from is the
``halo`` mode:

* ``"margin"``: the rank integrates its margin blocks itself from the
  broadcast depth frame (integration depends only on the frame, the pose and
  the block's previous state, so they are bit-identical to the owner's) --
  no data-path collective, redundant integration;
* ``"exchange"`` (the north star's "boundary-block halos exchanged over
  NVLink with NCCL before meshing"): the rank collects and integrates its
  OWNED blocks only; each owner packs its collected boundary blocks (those in
  another rank's margin: coordinate + 512 tsdf + 512 weights), the ranks
  all-gather the records, and every rank adopts the ones in its margin
  before meshing (vm_partition_frame_begin / _finish).

What else crosses ranks:

* per frame, the additive StatsRow counters (``allreduce_frame_stats``), from
  which every rank rebuilds the reference's global StatsRow, including the
  arena high-water mark (``StatsCombiner``);
* at extraction (``compact``), each rank's owned-block metadata (packed
  keys, vertex / triangle counts, 48-word slot occupancy, ~200 B per block):
  all-gathered, k-way merged by block key into the global block order
  (store.py:396-406), after which every rank writes its owned vertices and
  triangles at their global positions on the device and the ranks' disjoint
  ranges are summed (one all-reduce per output array).

The collectives run over ``torch.distributed``: NCCL on device tensors, gloo on
host copies (the CPU / single-GPU multi-process tests).
has the cost model.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .store import CompactMesh, SpatialStore

# Counters the device keeps over owned blocks only (margin work is not counted),
# so they sum exactly over ranks.
ADDITIVE = ("blocks_active", "vertices_live", "triangles_live", "vertices_recycled_total",
            "irregular_cube_count", "new_vertices", "vertices_freed", "changed_cubes",
            "normals_computed", "fallback_normals")
HALO_MODES = ("margin", "exchange")


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


def _is_nccl(group) -> bool:
    import torch.distributed as dist
    return str(dist.get_backend(group)).lower() == "nccl"


def allreduce_frame_stats(stats: dict, group=None, device=None) -> dict:
    """Sum this rank's per-frame counters over the process group."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([int(stats[k]) for k in ADDITIVE], dtype=torch.int64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return dict(zip(ADDITIVE, (int(v) for v in t.tolist())))


# ---------------------------------------------------------------- compaction
@dataclass
class OwnedMeta:
    """One rank's owned blocks for the distributed compaction (sorted by key)."""
    keys: np.ndarray     # uint64 packed block coordinates (pack_coord order = (x, y, z) lexicographic)
    vcnt: np.ndarray     # int32 occupied edge slots per block
    tcnt: np.ndarray     # int32 triangles per block
    occ: np.ndarray      # uint32 (n, 48) slot occupancy


def owned_meta(store: SpatialStore) -> OwnedMeta:
    L = _lib.load()
    n = C.c_int64()
    _lib.check(L.vm_partition_compact_begin(store._h, C.byref(n)))
    k = n.value
    m = OwnedMeta(np.zeros(k, np.uint64), np.zeros(k, np.int32), np.zeros(k, np.int32),
                  np.zeros((k, 48), np.uint32))
    if k:
        _lib.check(L.vm_partition_compact_meta(store._h, _lib.ptr(m.keys), _lib.ptr(m.vcnt),
                                               _lib.ptr(m.tcnt), _lib.ptr(m.occ)))
    return m


@dataclass
class GlobalLayout:
    keys: np.ndarray      # uint64 (n,) all ranks' owned blocks, merged by key
    vbase: np.ndarray     # int64 exclusive vertex base per block
    tbase: np.ndarray     # int64 exclusive triangle base per block
    occ: np.ndarray       # uint32 (n, 48)
    occ_pre: np.ndarray   # int32 (n, 48) exclusive popcount prefix per word
    nv: int
    nt: int
    my_global: list       # per rank: int32 global positions of its blocks


def merge_meta(metas: list) -> GlobalLayout:
    """k-way merge of the ranks' sorted owned-block lists by packed key: the
    reference's sorted-block compaction order (store.py:396-406) over the
    union, with the vertex / triangle bases and slot prefixes of every block."""
    sizes = [len(m.keys) for m in metas]
    keys = np.concatenate([m.keys for m in metas]) if metas else np.zeros(0, np.uint64)
    order = np.argsort(keys, kind="stable")
    if len(keys) > 1 and not (np.diff(keys[order].astype(np.uint64)) > 0).all():
        raise RuntimeError("a block is owned by more than one rank")
    rank_of = np.empty(len(keys), np.int64)
    rank_of[order] = np.arange(len(keys))
    vcnt = np.concatenate([m.vcnt for m in metas]).astype(np.int64)[order]
    tcnt = np.concatenate([m.tcnt for m in metas]).astype(np.int64)[order]
    occ = np.ascontiguousarray(np.concatenate([m.occ for m in metas])[order]) if len(keys) else \
        np.zeros((0, 48), np.uint32)
    vbase = np.concatenate([[0], np.cumsum(vcnt)]).astype(np.int64)
    tbase = np.concatenate([[0], np.cumsum(tcnt)]).astype(np.int64)
    pc = np.bitwise_count(occ).astype(np.int32)
    occ_pre = np.ascontiguousarray((np.cumsum(pc, axis=1) - pc).astype(np.int32))
    offs = np.concatenate([[0], np.cumsum(sizes)])
    my = [np.ascontiguousarray(rank_of[offs[r]:offs[r + 1]].astype(np.int32)) for r in range(len(metas))]
    return GlobalLayout(np.ascontiguousarray(keys[order]), np.ascontiguousarray(vbase[:-1]),
                        np.ascontiguousarray(tbase[:-1]), occ, occ_pre, int(vbase[-1]), int(tbase[-1]), my)


def fill_owned(store: SpatialStore, lay: GlobalLayout, rank_index: int, current_frame: int, device):
    """This rank's vertices / triangles at their global positions (device
    tensors of the whole mesh, zero elsewhere)."""
    import torch
    pos = torch.zeros((lay.nv, 3), dtype=torch.float64, device=device)
    nrm = torch.zeros((lay.nv, 3), dtype=torch.float64, device=device)
    ages = torch.zeros(lay.nv, dtype=torch.int64, device=device)
    idx = torch.zeros((lay.nt, 3), dtype=torch.int32, device=device)
    torch.cuda.synchronize(device)
    _lib.check(_lib.load().vm_partition_compact_fill(
        store._h, _lib.ptr(lay.keys), _lib.ptr(lay.vbase), _lib.ptr(lay.tbase), _lib.ptr(lay.occ),
        _lib.ptr(lay.occ_pre), len(lay.keys), _lib.ptr(lay.my_global[rank_index]), int(current_frame),
        C.c_void_p(pos.data_ptr()), C.c_void_p(nrm.data_ptr()), C.c_void_p(ages.data_ptr()),
        C.c_void_p(idx.data_ptr())))
    return pos, nrm, ages, idx


META_WIDTH = 1 + 1 + 24   # int64 words per block: key, (vcnt << 32 | tcnt), 48 x u32 occupancy


def pack_meta(meta: OwnedMeta, rows: int) -> np.ndarray:
    buf = np.zeros((rows, META_WIDTH), np.int64)
    k = len(meta.keys)
    if k:
        buf[:k, 0] = meta.keys.view(np.int64)
        buf[:k, 1] = (meta.vcnt.astype(np.int64) << 32) | meta.tcnt.astype(np.int64)
        buf[:k, 2:] = np.ascontiguousarray(meta.occ).view(np.int64).reshape(k, 24)
    return buf


def unpack_meta(a: np.ndarray) -> OwnedMeta:
    return OwnedMeta(np.ascontiguousarray(a[:, 0]).view(np.uint64), (a[:, 1] >> 32).astype(np.int32),
                     (a[:, 1] & 0xFFFFFFFF).astype(np.int32),
                     np.ascontiguousarray(a[:, 2:]).view(np.uint32).reshape(-1, 48))


def gather_metas(meta: OwnedMeta, group=None, device="cpu") -> list:
    """Every rank's owned-block metadata on every rank: an all-gather of the
    counts, then one padded all-gather of META_WIDTH int64 words per block."""
    import torch
    import torch.distributed as dist
    n = torch.tensor([len(meta.keys)], dtype=torch.int64, device=device)
    ns = [torch.empty_like(n) for _ in range(dist.get_world_size(group))]
    dist.all_gather(ns, n, group=group)
    n_all = [int(x.item()) for x in ns]
    mx = max(n_all)
    if mx == 0:
        return [unpack_meta(np.zeros((0, META_WIDTH), np.int64)) for _ in n_all]
    src = torch.from_numpy(pack_meta(meta, mx)).to(device)
    parts = [torch.empty_like(src) for _ in n_all]
    dist.all_gather(parts, src, group=group)
    return [unpack_meta(p.cpu().numpy()[:k]) for p, k in zip(parts, n_all)]


def _to_mesh(pos, nrm, ages, idx) -> CompactMesh:
    return CompactMesh(pos.cpu().numpy(), nrm.cpu().numpy(), ages.cpu().numpy(), idx.cpu().numpy())


def compact_local(stores: list, current_frame: int, device="cuda") -> CompactMesh:
    """The distributed compaction of N ranks' stores held by ONE process (the
    same merge and fill as PartitionedEngine.compact, the sum done here)."""
    import torch
    metas = [owned_meta(s) for s in stores]
    lay = merge_meta(metas)
    acc = None
    for r, s in enumerate(stores):
        part = fill_owned(s, lay, r, current_frame, device)
        if acc is None:
            acc = [p.view(torch_int_view(p)) for p in part]
        else:
            for a, p in zip(acc, part):
                a += p.view(torch_int_view(p))
    pos, nrm, ages, idx = acc
    return _to_mesh(pos.view(torch.float64), nrm.view(torch.float64), ages, idx)


def torch_int_view(t):
    """Integer dtype of the same width: bit patterns add exactly when every
    element but one rank's is zero."""
    import torch
    return {torch.float64: torch.int64, torch.int64: torch.int64, torch.int32: torch.int32}[t.dtype]


# ---------------------------------------------------------------- legacy merge
def export_blocks(store: SpatialStore, owned_only: bool = True) -> dict:
    """Dense host arrays of this store's (owned) blocks (diagnostics, tests)."""
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
    """store.py:388-425 over the union of the ranks' owned blocks (one store)."""
    return merge_stores(exports, cube_size, table_size).compact_mesh(current_frame)


# ---------------------------------------------------------------- engine
class PartitionedEngine:
    """``Engine`` for one rank of a spatially partitioned reconstruction.

    Every rank feeds the same (broadcast) depth frames; ``fuse_frame`` returns
    the reference's *global* StatsRow (one int64 all-reduce per frame).
    ``compact`` returns the merged mesh on every rank.  ``group`` is a
    torch.distributed process group (NCCL: device tensors; gloo: host copies).
    """

    def __init__(self, config, intrinsics, group=None, tile_blocks: int = 8, device=None,
                 halo: str = "margin", shard_band: bool = True):
        import dataclasses

        import torch
        import torch.distributed as dist
        from .engine import Engine
        if halo not in HALO_MODES:
            raise ValueError(f"unknown halo mode {halo!r}")
        self.group = group
        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)
        self.halo = halo
        # halo exchange: each rank walks 1/N of the pixel rows and the ranks
        # all-gather the block keys they met (vm_partition_collect_keys)
        self.shard_band = bool(shard_band) and halo == "exchange" and self.nranks > 1
        self._keys = None
        self.nccl = _is_nccl(group)
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self.engine = Engine(dataclasses.replace(config, rank=self.rank, nranks=self.nranks,
                                                 tile_blocks=tile_blocks,
                                                 halo_exchange=halo == "exchange"), intrinsics)
        self.combiner = StatsCombiner()
        self.stats = []
        self._send = None
        self.exchange_log = []   # per frame: records sent by each rank (halo exchange)
        self.key_log = []        # per frame: block keys listed by each rank (sharded band walk)

    # -- collectives ---------------------------------------------------------
    def _stream_ctx(self):
        """NCCL work on the engine's stream (ordered with its kernels)."""
        import contextlib

        import torch
        if not self.nccl:
            return contextlib.nullcontext()
        h = C.c_void_p()
        _lib.check(_lib.load().vm_get_stream(self.engine.store._h, C.byref(h)))
        return torch.cuda.stream(torch.cuda.ExternalStream(h.value, device=self.device))

    def _all_gather_ints(self, values) -> np.ndarray:
        import torch
        import torch.distributed as dist
        dev = self.device if self.nccl else "cpu"
        t = torch.tensor(np.asarray(values, np.int64), dtype=torch.int64, device=dev)
        out = [torch.empty_like(t) for _ in range(self.nranks)]
        dist.all_gather(out, t, group=self.group)
        return np.stack([o.cpu().numpy() for o in out])

    def _all_gather_bytes(self, t, nbytes: int):
        """All-gather the first `nbytes` of a device uint8 tensor from every
        rank (equal sizes); returns the device tensor of nranks * nbytes."""
        import torch
        import torch.distributed as dist
        if self.nccl:
            out = torch.empty(self.nranks * nbytes, dtype=torch.uint8, device=self.device)
            with self._stream_ctx():
                dist.all_gather_into_tensor(out, t[:nbytes].contiguous(), group=self.group)
            return out
        src = t[:nbytes].cpu()
        parts = [torch.empty_like(src) for _ in range(self.nranks)]
        dist.all_gather(parts, src, group=self.group)
        out = torch.cat(parts).to(self.device)
        torch.cuda.synchronize(self.device)   # (the engine's stream reads it next)
        return out

    def _sum_(self, t):
        """In-place SUM over ranks of an integer (bit-pattern view) tensor."""
        import torch.distributed as dist
        if self.nccl:
            with self._stream_ctx():
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
            return t
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
        return h

    # -- frames ----------------------------------------------------------------
    def _exchange_frame(self, depth, pose):
        """Halo-exchange frame: begin (collect + integrate owned, pack the
        boundary blocks) -> all-gather of the records -> finish (adopt the
        margin records, mesh)."""
        import torch
        e = self.engine
        L = _lib.load()
        rec = _lib.GHOST_RECORD
        ptr, h, w, on_dev, keep = e._depth_args(depth)
        if self._send is None:
            self._send = torch.empty(4096 * rec, dtype=torch.uint8, device=self.device)
        torch.cuda.synchronize(self.device)
        n_send, n_own = C.c_int64(), C.c_int64()
        e.store._touch()
        if self.shard_band:
            # this rank's pixel-row slice (multiples of 8 rows), its block keys,
            # all-gathered: every rank then collects its relevant blocks from the union
            rows = [(h * r // self.nranks) // 8 * 8 for r in range(self.nranks)] + [h]
            r0, r1 = rows[self.rank], rows[self.rank + 1]
            if self._keys is None:
                self._keys = torch.empty(1 << 20, dtype=torch.int64, device=self.device)
            nk = C.c_int64(0)
            _lib.check(L.vm_partition_collect_keys(e.store._h, ptr, h, w, on_dev, C.byref(e._intr_c),
                                                   C.byref(_lib.pose_c(pose)), C.byref(e._fcfg), e.frame_index,
                                                   r0, r1, C.c_void_p(self._keys.data_ptr()),
                                                   self._keys.numel(), C.byref(nk)))
            kc = self._all_gather_ints([nk.value]).reshape(-1)
            kmax = int(kc.max())
            allk = None
            if kmax:
                g = self._all_gather_bytes(self._keys.view(torch.uint8), kmax * 8).view(torch.int64)
                allk = torch.cat([g[q * kmax:q * kmax + int(kc[q])] for q in range(self.nranks)])
                torch.cuda.synchronize(self.device)   # (the engine's stream reads the union next)
            self.key_log.append(kc.tolist())
            _lib.check(L.vm_partition_frame_begin_keys(
                e.store._h, C.c_void_p(allk.data_ptr()) if allk is not None else None,
                int(allk.numel()) if allk is not None else 0, C.c_void_p(self._send.data_ptr()),
                self._send.numel() // rec, C.byref(n_send), C.byref(n_own)))
            del allk
        else:
            _lib.check(L.vm_partition_frame_begin(e.store._h, ptr, h, w, on_dev, C.byref(e._intr_c),
                                                  C.byref(_lib.pose_c(pose)), C.byref(e._fcfg),
                                                  e.frame_index, C.c_void_p(self._send.data_ptr()),
                                                  self._send.numel() // rec, C.byref(n_send),
                                                  C.byref(n_own)))
        if n_send.value > self._send.numel() // rec:
            self._send = torch.empty(int(n_send.value * 1.25 + 64) * rec, dtype=torch.uint8,
                                     device=self.device)
            _lib.check(L.vm_partition_repack(e.store._h, C.c_void_p(self._send.data_ptr()),
                                             self._send.numel() // rec, C.byref(n_send)))
        counts = self._all_gather_ints([n_send.value]).reshape(-1).astype(np.int32)
        maxc = int(counts.max()) if len(counts) else 0
        self.exchange_log.append(counts.tolist())
        recv = self._all_gather_bytes(self._send, maxc * rec) if maxc else None
        st = _lib.Stats()
        _lib.check(L.vm_partition_frame_finish(e.store._h,
                                               C.c_void_p(recv.data_ptr()) if recv is not None else None,
                                               _lib.ptr(np.ascontiguousarray(counts)), self.nranks, maxc,
                                               C.byref(st)))
        del keep
        return e._record(st)

    def fuse_frame(self, depth, pose):
        from .engine import StatsRow
        row = (self._exchange_frame(depth, pose) if self.halo == "exchange"
               else self.engine.fuse_frame(depth, pose))
        g = self.combiner.combine(allreduce_frame_stats(self.engine.device_stats[-1], self.group,
                                                        self.device if self.nccl else None))
        out = StatsRow(frame=row.frame, blocks_active=g["blocks_active"],
                       vertices_live=g["vertices_live"], triangles_live=g["triangles_live"],
                       vertices_allocated_total=g["vertices_allocated_total"],
                       vertices_recycled_total=g["vertices_recycled_total"],
                       irregular_cube_count=g["irregular_cube_count"], fusion_ms=row.fusion_ms,
                       meshing_ms=row.meshing_ms, compact_ms=0.0)
        self.stats.append(out)
        return out

    def compact(self) -> CompactMesh:
        """Distributed store.py:388-425: gather the owned-block metadata, merge
        by key, fill the owned ranges on the device, sum over ranks."""
        import torch
        self.engine._resolve_pending()
        metas = gather_metas(owned_meta(self.engine.store), self.group,
                             self.device if self.nccl else "cpu")
        lay = merge_meta(metas)
        pos, nrm, ages, idx = fill_owned(self.engine.store, lay, self.rank, self.engine.frame_index,
                                         self.device)
        out = [self._sum_(x.view(torch_int_view(x))) for x in (pos, nrm, ages, idx)]
        return _to_mesh(out[0].view(torch.float64), out[1].view(torch.float64), out[2], out[3])


__all__ = ["PartitionedEngine", "StatsCombiner", "sum_stats", "allreduce_frame_stats", "export_blocks",
           "merge_stores", "merge_compact", "ADDITIVE", "HALO_MODES", "OwnedMeta", "GlobalLayout",
           "owned_meta", "merge_meta", "fill_owned", "compact_local", "gather_metas", "pack_meta",
           "unpack_meta"]
