"""Frame-by-frame reconstruction driver (mirror of reference pkg/src/voxmesh/engine.py).

``Engine.fuse_frame`` is ONE C-ABI call (``vm_fuse_frame``): depth upload,
then the whole per-frame kernel sequence on the device (collect -> integrate
-> scope/halo -> retype(+refine) -> place -> triangulate -> GC -> normals), and
a D2H read of the StatsRow counters.  The non-timing StatsRow columns match
the reference exactly; ``fusion_ms`` / ``meshing_ms`` are device times (the
kernels' own %globaltimer stamps: collect + integrate | retype + placement +
GC + normals) of the same two segments the reference times on the host
(engine.py:127-156).
"""
from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass, replace
from typing import Optional

import numpy as np

from . import _lib
from .errors import ConsistencyError
from .fusion import Intrinsics, Pose
from .mesher import STRATEGIES
from .refine import REGULAR_TYPES, RefineParams
from .store import CompactMesh, SpatialStore


@dataclass
class RunConfig:
    cube_size: float = 0.03
    trunc: Optional[float] = None        # defaults to 3 * cube_size
    epsilon: float = 0.1
    refine: bool = False
    strategy: str = "claim"
    baseline: bool = False
    max_range: float = 5.0
    frustum_only: bool = False
    workers: int = 0                     # accepted for API parity; the GPU ignores it
    seed: int = 0
    weight_cap: int = 128
    max_vertices: Optional[int] = None
    table_size: int = 1 << 20
    # device arena capacity hints (0 = defaults; arenas grow on demand)
    block_capacity: int = 0
    vertex_capacity: int = 0
    triangle_capacity: int = 0
    # spatial partition: this engine computes rank's tiles
    rank: int = 0
    nranks: int = 1
    tile_blocks: int = 8
    halo_exchange: bool = False          # margin blocks received from their owners (partition.py)
    # opt-in block GC (north star item 5; off = the reference's never-evict
    # store, store.py:14): every block_gc_age frames, evict blocks not
    # collected for that long that hold no vertex and no observed sample
    block_gc_age: int = 0

    def resolved(self) -> "RunConfig":
        cfg = replace(self)
        if cfg.trunc is None:
            cfg.trunc = 3.0 * cfg.cube_size
        if cfg.trunc < cfg.cube_size:
            raise ValueError("truncation band must be at least one cube")
        if cfg.workers <= 0:
            cfg.workers = os.cpu_count() or 1
        if cfg.strategy not in STRATEGIES:
            raise ValueError(f"unknown strategy {cfg.strategy!r}")
        if cfg.block_gc_age < 0:
            raise ValueError("block_gc_age must be >= 0")
        return cfg

    def to_dict(self) -> dict:
        return {k: getattr(self, k) for k in (
            "cube_size", "trunc", "epsilon", "refine", "strategy", "baseline", "max_range",
            "frustum_only", "workers", "seed", "weight_cap")}


@dataclass
class StatsRow:
    frame: int
    blocks_active: int
    vertices_live: int
    triangles_live: int
    vertices_allocated_total: int
    vertices_recycled_total: int
    irregular_cube_count: int
    fusion_ms: float
    meshing_ms: float
    compact_ms: float

    FIELDS = ("frame", "blocks_active", "vertices_live", "triangles_live",
              "vertices_allocated_total", "vertices_recycled_total",
              "irregular_cube_count", "fusion_ms", "meshing_ms", "compact_ms")


@dataclass
class AuditReport:
    vertices_live: int
    triangles_live: int
    refcount_mismatches: int
    duplicate_handles: int
    zero_ref_live: int
    conservation_ok: bool

    @property
    def ok(self) -> bool:
        return (self.refcount_mismatches == 0 and self.duplicate_handles == 0
                and self.zero_ref_live == 0 and self.conservation_ok)


_REGULAR_MASK = np.zeros(256, dtype=bool)
_REGULAR_MASK[list(REGULAR_TYPES)] = True


def _is_device_tensor(x) -> bool:
    return hasattr(x, "data_ptr") and getattr(x, "is_cuda", False)


_ROW_KEYS = ("blocks_active", "vertices_live", "triangles_live", "vertices_allocated_total",
             "vertices_recycled_total", "irregular_cube_count", "fusion_ms", "meshing_ms")


class _PendingRow(StatsRow):
    """StatsRow of a frame submitted in pipelined mode: its fields are filled
    when the frame completes -- at the engine's next call or on first access."""

    def __init__(self, engine: "Engine", frame: int):
        object.__setattr__(self, "_engine", engine)
        object.__setattr__(self, "_done", False)
        object.__setattr__(self, "frame", frame)

    def _fill(self, row: StatsRow) -> None:
        for k in StatsRow.FIELDS:
            object.__setattr__(self, k, getattr(row, k))
        object.__setattr__(self, "_done", True)

    def _fill_from(self, d: dict) -> None:
        """The row's columns from the frame's device stats (Engine._row_from's mapping)."""
        sa = object.__setattr__
        for k in _ROW_KEYS:
            sa(self, k, d[k])
        sa(self, "compact_ms", 0.0)
        sa(self, "_done", True)

    def __getattribute__(self, name):
        if name in StatsRow.FIELDS and name != "frame" and not object.__getattribute__(self, "_done"):
            object.__getattribute__(self, "_engine")._resolve_pending()
        return object.__getattribute__(self, name)

    def __repr__(self):
        return StatsRow.__repr__(self) if self._done else f"_PendingRow(frame={self.frame})"

    def __eq__(self, other):
        self.blocks_active   # resolve
        return StatsRow.__eq__(self, other)


class Engine:
    def __init__(self, config: RunConfig, intrinsics: Intrinsics, audit_every_frame: bool = False,
                 pipelined: bool = False):
        """pipelined=True: fuse_frame returns once the frame's work is queued
        (its StatsRow fills in when the frame completes) and the next frame's
        host->device depth copy overlaps this frame's kernels
        (vm_fuse_frame_submit).  Results are identical; an error of frame t
        surfaces at the engine's next call."""
        self.config = config.resolved()
        self.intrinsics = intrinsics
        c = self.config
        self.store = SpatialStore(c.cube_size, table_size=c.table_size,
                                  max_vertices=c.max_vertices, initial_blocks=c.block_capacity,
                                  initial_vertices=c.vertex_capacity,
                                  initial_triangles=c.triangle_capacity, rank=c.rank,
                                  nranks=c.nranks, tile_blocks=c.tile_blocks,
                                  halo_exchange=c.halo_exchange)
        self.frame_index = 0
        self.stats: list[StatsRow] = []
        self.device_stats: list[dict] = []
        self.audit_every_frame = audit_every_frame
        self._intr_c = _lib.intr_c(intrinsics)
        self._pose_c = _lib.PoseC()   # (reused: the C side copies the pose during the call)
        self._pose_v = np.frombuffer(self._pose_c, dtype=np.float64, count=12)
        self._stream_h = None         # the engine's CUDA stream handle (cached; set_stream resets it)
        self._order_ev = None
        self._fcfg = _lib.FrameConfig(float(c.trunc), float(c.max_range), float(c.epsilon),
                                      int(c.weight_cap), int(bool(c.refine)),
                                      int(bool(c.frustum_only)), _lib.STRATEGY_CODES[c.strategy],
                                      int(max(0, c.block_gc_age)))
        self._collected_n = 0
        self._collected_cache = None
        self.pipelined = bool(pipelined) and not audit_every_frame
        self._pending: Optional[_PendingRow] = None
        self._inflight = None   # CUDA tensor input of the frame in flight (kept alive until it completes)
        # the submit returns with the host copy in flight; fuse_frame waits for
        # it (vm_input_wait) after delivering the previous frame's row
        _lib.check(_lib.load().vm_set_deferred_input_wait(self.store._h, 1))

    # -- per-frame pipeline ---------------------------------------------------
    def _order_device_input(self, t) -> None:
        """A CUDA tensor input is read by kernels on the engine's stream: order
        that stream after the stream that produced it (torch's current stream).
        The tensor is kept referenced until its frame has completed (the
        pipelined paths hold it in ``_inflight``), so the caching allocator
        cannot hand its memory out while a queued frame still reads it."""
        import torch
        if self._stream_h is None:
            self._stream_h = self.stream_handle()
        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        producer = raw(t.device.index) if raw is not None else torch.cuda.current_stream(t.device).cuda_stream
        if producer != self._stream_h:   # (C side: a wait only if the producer's work is pending --
            _lib.check(_lib.load().vm_order_after(self.store._h, C.c_void_p(producer or None)))   # no overlap then)

    def _pose_arg(self, pose) -> "_lib.PoseC":
        v = self._pose_v
        v[:9] = pose.rotation.reshape(9) if isinstance(pose.rotation, np.ndarray) else np.asarray(pose.rotation,
                                                                                                    np.float64).reshape(9)
        v[9:] = pose.translation
        return self._pose_c

    def _depth_args(self, depth):
        if _is_device_tensor(depth):
            import torch
            if depth.dtype != torch.float64 or not depth.is_contiguous() or depth.dim() != 2:
                raise ValueError("device depth must be a contiguous 2-D float64 CUDA tensor")
            self._order_device_input(depth)
            return C.c_void_p(depth.data_ptr()), depth.shape[0], depth.shape[1], 1, depth
        d = np.ascontiguousarray(np.asarray(depth, dtype=np.float64))
        if d.ndim != 2:
            raise ValueError("depth must be a 2-D array")
        return _lib.ptr(d), d.shape[0], d.shape[1], 0, d

    def fuse_frame(self, depth, pose: Pose) -> StatsRow:
        ptr, h, w, on_dev, keep = self._depth_args(depth)
        self.store._touch()
        if self.pipelined:
            L = _lib.load()
            rc = L.vm_fuse_frame_submit(self.store._h, ptr, h, w, on_dev, C.byref(self._intr_c),
                                        C.byref(self._pose_arg(pose)), C.byref(self._fcfg), self.frame_index)
            try:   # (the previous frame's row is delivered while this frame's host buffer is copied)
                return self._after_submit(rc, keep if on_dev else None)
            finally:
                if not on_dev:
                    L.vm_input_wait(self.store._h)   # the caller may reuse its buffer on return
        st = _lib.Stats()
        _lib.check(_lib.load().vm_fuse_frame(self.store._h, ptr, h, w, on_dev,
                                              C.byref(self._intr_c), C.byref(self._pose_arg(pose)),
                                              C.byref(self._fcfg), self.frame_index, C.byref(st)))
        del keep
        return self._record(st)

    def fuse_frame_raw(self, raw, pose: Pose, depth_scale: float = 5000.0) -> StatsRow:
        """fuse_frame(read_depth-style raw / depth_scale, pose) from the raw 16-bit
        depth image (io_formats.py:41-84): the conversion runs on the device,
        bit-identical, and only the u16 image crosses PCIe.  `raw` is a (H, W)
        uint16 array (native byte order) or a contiguous uint16/int16 CUDA tensor."""
        if _is_device_tensor(raw):
            if raw.element_size() != 2 or not raw.is_contiguous() or raw.dim() != 2:
                raise ValueError("device raw depth must be a contiguous 2-D 16-bit CUDA tensor")
            ptr, h, w, on_dev, keep = C.c_void_p(raw.data_ptr()), raw.shape[0], raw.shape[1], 1, raw
        else:
            a = np.ascontiguousarray(np.asarray(raw, dtype=np.uint16))
            if a.ndim != 2:
                raise ValueError("raw depth must be a 2-D array")
            ptr, h, w, on_dev, keep = _lib.ptr(a), a.shape[0], a.shape[1], 0, a
        self.store._touch()
        if on_dev:
            self._order_device_input(raw)
        L = _lib.load()
        rc = L.vm_fuse_frame_submit_raw(self.store._h, ptr, h, w, on_dev, float(depth_scale),
                                        C.byref(self._intr_c), C.byref(self._pose_arg(pose)),
                                        C.byref(self._fcfg), self.frame_index)
        try:
            row = self._after_submit(rc, keep if on_dev else None)
        finally:
            if not on_dev:
                L.vm_input_wait(self.store._h)
        if not self.pipelined:
            self._resolve_pending()
        return row

    def _after_submit(self, rc: int, device_input=None) -> StatsRow:
        """Bookkeeping after vm_fuse_frame_submit[_raw].  An argument error
        (empty depth, bad config) queued nothing and left the frame in flight
        pending: its row stays pending.  Any other error completed the pending
        frame (it is the error reported) and dropped the new one."""
        if rc in (_lib.VM_ERR_INPUT, _lib.VM_ERR_VALUE):
            _lib.check(rc)
        prev, self._pending = self._pending, None
        self._inflight = None   # (the previous frame has completed on the device)
        _lib.check(rc)          # (an error of the previous frame surfaces here)
        self._inflight = device_input   # read by the frame now in flight
        if prev is not None:    # completed by the submit: deliver its stats
            self._deliver(prev)
        row = _PendingRow(self, self.frame_index)
        self._pending = row
        self.stats.append(row)
        self.frame_index += 1
        return row

    def _deliver(self, row: _PendingRow) -> None:
        st = _lib.Stats()
        _lib.check(_lib.load().vm_fuse_frame_result(self.store._h, C.byref(st)))
        d = st.as_dict()
        self.device_stats.append(d)
        self._collected_n = d["collected_blocks"]
        self._collected_cache = None
        row._fill_from(d)

    def _resolve_pending(self) -> None:
        """Complete the pipelined frame in flight, if any (every engine
        entry point settles it on the device side as well)."""
        row, self._pending = self._pending, None
        if row is not None:
            self._deliver(row)
        self._inflight = None

    @staticmethod
    def _row_from(frame: int, d: dict) -> StatsRow:
        return StatsRow(frame=frame, blocks_active=d["blocks_active"],
                        vertices_live=d["vertices_live"], triangles_live=d["triangles_live"],
                        vertices_allocated_total=d["vertices_allocated_total"],
                        vertices_recycled_total=d["vertices_recycled_total"],
                        irregular_cube_count=d["irregular_cube_count"],
                        fusion_ms=d["fusion_ms"], meshing_ms=d["meshing_ms"], compact_ms=0.0)

    def fuse_frame_enqueue(self, depth, pose: Pose):
        """Split form for device timing: enqueue only (see vm_fuse_frame_enqueue)."""
        self._resolve_pending()
        ptr, h, w, on_dev, keep = self._depth_args(depth)
        self.store._touch()
        _lib.check(_lib.load().vm_fuse_frame_enqueue(self.store._h, ptr, h, w, on_dev,
                                                      C.byref(self._intr_c),
                                                      C.byref(self._pose_arg(pose)),
                                                      C.byref(self._fcfg), self.frame_index))
        return keep

    def fuse_frame_finish(self) -> StatsRow:
        st = _lib.Stats()
        _lib.check(_lib.load().vm_fuse_frame_finish(self.store._h, C.byref(st)))
        return self._record(st)

    def _record(self, st) -> StatsRow:
        d = st.as_dict()
        self.device_stats.append(d)
        self._collected_n = d["collected_blocks"]
        self._collected_cache = None
        row = StatsRow(frame=self.frame_index, blocks_active=d["blocks_active"],
                       vertices_live=d["vertices_live"], triangles_live=d["triangles_live"],
                       vertices_allocated_total=d["vertices_allocated_total"],
                       vertices_recycled_total=d["vertices_recycled_total"],
                       irregular_cube_count=d["irregular_cube_count"],
                       fusion_ms=d["fusion_ms"], meshing_ms=d["meshing_ms"], compact_ms=0.0)
        self.stats.append(row)
        self.frame_index += 1
        if self.audit_every_frame:
            report = self.audit()
            if not report.ok:
                raise ConsistencyError(f"frame {row.frame} audit failed: {report}")
        return row

    @property
    def last_collected(self) -> list:
        self._resolve_pending()
        if self._collected_cache is None:
            n = self._collected_n
            out = np.zeros((n, 3), np.int32)
            if n:
                _lib.check(_lib.load().vm_get_collected(self.store._h, _lib.ptr(out), n))
            self._collected_cache = sorted((int(a), int(b), int(c)) for a, b, c in out)
        return self._collected_cache

    # -- derived quantities -----------------------------------------------------
    def irregular_cube_count(self) -> int:
        """engine.py:169-176 as a full device scan."""
        self._resolve_pending()
        return self.store.irregular_cube_count()

    def compact(self) -> CompactMesh:
        self._resolve_pending()
        t0 = time.perf_counter()
        mesh = self.store.compact_mesh(self.frame_index)
        if self.stats:
            self.stats[-1].compact_ms = (time.perf_counter() - t0) * 1e3
        return mesh

    def audit(self) -> AuditReport:
        """engine.py:187-230 as device reductions."""
        self._resolve_pending()
        a = _lib.AuditC()
        _lib.check(_lib.load().vm_audit(self.store._h, C.byref(a)))
        return AuditReport(vertices_live=int(a.vertices_live), triangles_live=int(a.triangles_live),
                           refcount_mismatches=int(a.refcount_mismatches),
                           duplicate_handles=int(a.duplicate_handles),
                           zero_ref_live=int(a.zero_ref_live),
                           conservation_ok=bool(a.conservation_ok))

    def set_profiling(self, on: bool = True) -> None:
        self._resolve_pending()
        _lib.check(_lib.load().vm_set_profiling(self.store._h, int(bool(on))))

    def phase_times(self) -> dict:
        """Per-kernel device ms of the last frame (requires set_profiling)."""
        self._resolve_pending()
        ms = np.zeros(len(PHASES))
        _lib.check(_lib.load().vm_phase_times(self.store._h, _lib.ptr(ms), len(PHASES)))
        return dict(zip(PHASES, (float(v) for v in ms)))

    def set_trace(self, buffer) -> None:
        """Diagnostics: per-CTA kernel phase timestamps into a CUDA u64 tensor of
        4 * 2048 * 32 entries (csrc/vm_device.cuh, kTraceCtas); None = off."""
        ptr = None if buffer is None else buffer.data_ptr()
        _lib.check(_lib.load().vm_set_trace(self.store._h, C.c_void_p(ptr)))

    def stream_handle(self) -> int:
        """The CUDA stream the engine queues its work on (cudaStream_t as int)."""
        h = C.c_void_p()
        _lib.check(_lib.load().vm_get_stream(self.store._h, C.byref(h)))
        return h.value or 0

    def set_stream(self, stream_handle: int) -> None:
        """Queue the engine's work on a caller's stream (0 / None: its own).
        Frame overlap needs the engine's own stream."""
        self._resolve_pending()
        _lib.check(_lib.load().vm_set_stream(self.store._h, C.c_void_p(stream_handle or None)))
        self._stream_h = None


PHASES = ("depth_stats", "collect", "fuse_blocks", "retype_place", "gc_normals")
