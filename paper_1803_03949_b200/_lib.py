"""ctypes binding of ``libvoxmesh_b200.so`` (C ABI: include/voxmesh_b200.h).

There is no CPU fallback: if the shared library is missing, or no CUDA device
is present when an engine is created, the call fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from .errors import CapacityError, ConsistencyError, InputError

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libvoxmesh_b200.so"


def lib_path() -> Path:
    """The product library, or the VOXMESH_B200_LIB override (the tracing build
    of tools/trace_frame.py), read when the library is first loaded."""
    env = os.environ.get("VOXMESH_B200_LIB")
    return Path(env) if env else LIB_PATH

VM_OK, VM_ERR_CAPACITY, VM_ERR_CONSISTENCY, VM_ERR_VALUE, VM_ERR_CUDA, VM_ERR_INPUT = range(6)
STRATEGY_CODES = {"serial": 0, "claim": 1, "partition": 2}
GHOST_RECORD = 6160   # VM_GHOST_RECORD: halo-exchange record bytes (coord + 512 tsdf + 512 weights)


class StoreConfig(C.Structure):
    _fields_ = [("cube_size", C.c_double), ("table_size", C.c_int64), ("max_vertices", C.c_int64),
                ("initial_blocks", C.c_int64), ("initial_vertices", C.c_int64),
                ("initial_triangles", C.c_int64), ("rank", C.c_int32), ("nranks", C.c_int32),
                ("tile_blocks", C.c_int32), ("halo_exchange", C.c_int32)]


class Intr(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32)]


class PoseC(C.Structure):
    _fields_ = [("rotation", C.c_double * 9), ("translation", C.c_double * 3)]


class FrameConfig(C.Structure):
    _fields_ = [("trunc", C.c_double), ("max_range", C.c_double), ("epsilon", C.c_double),
                ("weight_cap", C.c_int64), ("refine", C.c_int32), ("frustum_only", C.c_int32),
                ("strategy", C.c_int32), ("block_gc_age", C.c_int32)]


STATS_FIELDS = ("frame", "blocks_active", "vertices_live", "triangles_live",
                "vertices_allocated_total", "vertices_recycled_total", "irregular_cube_count",
                "valid_pixels", "nsteps", "collected_blocks", "new_blocks", "scope_blocks",
                "halo_blocks", "active_cubes", "edge_placements", "new_vertices", "changed_cubes",
                "triangles_freed", "triangles_allocated", "vertices_freed", "normals_computed",
                "fallback_normals", "refined_cubes", "resumes", "kernel_launches", "blocks_evicted",
                "overlapped")


class Stats(C.Structure):
    _fields_ = [(k, C.c_int64) for k in STATS_FIELDS] + [
        ("device_ms", C.c_double), ("fusion_ms", C.c_double), ("meshing_ms", C.c_double)]

    def as_dict(self) -> dict:
        # (one numpy view of the struct instead of a getattr per field: this
        # runs once per frame on the submission path)
        n = len(STATS_FIELDS)
        d = dict(zip(STATS_FIELDS, np.frombuffer(self, dtype=np.int64, count=n).tolist()))
        d.update(zip(("device_ms", "fusion_ms", "meshing_ms"),
                     np.frombuffer(self, dtype=np.float64, count=3, offset=8 * n).tolist()))
        return d


class AuditC(C.Structure):
    _fields_ = [(k, C.c_int64) for k in ("vertices_live", "triangles_live", "refcount_mismatches",
                                         "duplicate_handles", "zero_ref_live", "conservation_ok")]


COUNTER_FIELDS = ("block_count", "block_allocations", "vertex_count", "vertex_free",
                  "vertex_recycled_total", "vertex_allocation_events", "triangle_count",
                  "triangle_free", "triangle_recycled_total", "irregular_cube_count",
                  "block_capacity", "vertex_capacity", "triangle_capacity", "vertex_records",
                  "store_bytes", "device_bytes")


class CountersC(C.Structure):
    _fields_ = [(k, C.c_int64) for k in COUNTER_FIELDS]


# exported symbols (checked by tests/test_abi.py against include/voxmesh_b200.h)
_SIGS = {
    "vm_last_error": (C.c_char_p, []),
    "vm_version": (C.c_char_p, []),
    "vm_create": (C.c_int, [C.POINTER(StoreConfig), C.POINTER(C.c_void_p)]),
    "vm_destroy": (C.c_int, [C.c_void_p]),
    "vm_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "vm_get_stream": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "vm_order_after": (C.c_int, [C.c_void_p, C.c_void_p]),
    "vm_partition_collect_keys": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                            C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p,
                                            C.c_int64, C.POINTER(C.c_int64)]),
    "vm_partition_frame_begin_keys": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                                C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "vm_set_deferred_input_wait": (C.c_int, [C.c_void_p, C.c_int]),
    "vm_input_wait": (C.c_int, [C.c_void_p]),
    "vm_set_profiling": (C.c_int, [C.c_void_p, C.c_int]),
    "vm_phase_times": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    "vm_set_trace": (C.c_int, [C.c_void_p, C.c_void_p]),
    "vm_reserve": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int64]),
    "vm_fuse_frame": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                C.POINTER(Intr), C.POINTER(PoseC), C.POINTER(FrameConfig),
                                C.c_int64, C.POINTER(Stats)]),
    "vm_fuse_frame_enqueue": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                        C.POINTER(Intr), C.POINTER(PoseC), C.POINTER(FrameConfig),
                                        C.c_int64]),
    "vm_fuse_frame_finish": (C.c_int, [C.c_void_p, C.POINTER(Stats)]),
    "vm_fuse_frame_submit": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                       C.POINTER(Intr), C.POINTER(PoseC), C.POINTER(FrameConfig),
                                       C.c_int64]),
    "vm_fuse_frame_result": (C.c_int, [C.c_void_p, C.POINTER(Stats)]),
    "vm_fuse_frame_submit_raw": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                           C.c_double, C.POINTER(Intr), C.POINTER(PoseC),
                                           C.POINTER(FrameConfig), C.c_int64]),
    "vm_collect": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                             C.POINTER(Intr), C.POINTER(PoseC), C.c_double, C.c_double,
                             C.POINTER(C.c_int64)]),
    "vm_get_collected": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64]),
    "vm_integrate": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_int32,
                               C.c_int32, C.POINTER(Intr), C.POINTER(PoseC), C.c_double,
                               C.c_double, C.c_int64]),
    "vm_scope_halo": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.c_void_p, C.c_void_p,
                                C.POINTER(C.c_int64), C.c_void_p]),
    "vm_extract": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                             C.c_int64, C.c_int32, C.c_int32, C.c_double, C.c_void_p]),
    "vm_garbage_collect": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]),
    "vm_compute_normals": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64]),
    "vm_refine_eval": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                 C.c_double, C.c_void_p]),
    "vm_block_in_frustum": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(PoseC),
                                      C.POINTER(Intr), C.c_void_p]),
    "vm_set_blocks": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "vm_lookup": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "vm_counters": (C.c_int, [C.c_void_p, C.POINTER(CountersC)]),
    "vm_snapshot_blocks": (C.c_int, [C.c_void_p, C.c_int64] + [C.c_void_p] * 7),
    "vm_snapshot_vertices": (C.c_int, [C.c_void_p, C.c_int64] + [C.c_void_p] * 6),
    "vm_snapshot_triangles": (C.c_int, [C.c_void_p, C.c_int64] + [C.c_void_p] * 3),
    "vm_irregular_count": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "vm_compact": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "vm_compact_fetch": (C.c_int, [C.c_void_p] + [C.c_void_p] * 4),
    "vm_audit": (C.c_int, [C.c_void_p, C.POINTER(AuditC)]),
    "vm_export_blocks": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_int64)] + [C.c_void_p] * 8),
    "vm_import_blocks": (C.c_int, [C.c_void_p, C.c_int64] + [C.c_void_p] * 8),
    "vm_partition_frame_begin": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                           C.POINTER(Intr), C.POINTER(PoseC), C.POINTER(FrameConfig),
                                           C.c_int64, C.c_void_p, C.c_int64, C.POINTER(C.c_int64),
                                           C.POINTER(C.c_int64)]),
    "vm_partition_repack": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]),
    "vm_partition_frame_finish": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int64,
                                            C.POINTER(Stats)]),
    "vm_partition_compact_begin": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "vm_partition_compact_meta": (C.c_int, [C.c_void_p] + [C.c_void_p] * 4),
    "vm_partition_compact_fill": (C.c_int, [C.c_void_p] + [C.c_void_p] * 5 + [C.c_int64, C.c_void_p, C.c_int64]
                                  + [C.c_void_p] * 4),
}

EXPORTED = tuple(_SIGS)
_lib = None


def load():
    """Load the CUDA library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        path = lib_path()
        if not path.exists():
            raise RuntimeError(
                f"{path.name} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        L = C.CDLL(str(path))
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == VM_OK:
        return
    msg = load().vm_last_error().decode()
    if rc == VM_ERR_CAPACITY:
        raise CapacityError(msg)
    if rc == VM_ERR_CONSISTENCY:
        raise ConsistencyError(msg)
    if rc == VM_ERR_VALUE:
        raise ValueError(msg)
    if rc == VM_ERR_INPUT:
        raise InputError(msg)
    raise RuntimeError(f"CUDA error: {msg}")


def ptr(a) -> C.c_void_p | None:
    if a is None:
        return None
    return C.c_void_p(a.ctypes.data)


def intr_c(intr) -> Intr:
    return Intr(float(intr.fx), float(intr.fy), float(intr.cx), float(intr.cy),
                int(intr.width), int(intr.height))


def pose_c(pose, out: "PoseC | None" = None) -> PoseC:
    p = PoseC() if out is None else out
    v = np.frombuffer(p, dtype=np.float64, count=12)
    v[:9] = np.asarray(pose.rotation, np.float64).reshape(9)
    v[9:] = np.asarray(pose.translation, np.float64).reshape(3)
    return p


def coords_array(coords) -> np.ndarray:
    if coords is None:
        return np.zeros((0, 3), np.int32)
    a = np.asarray(list(coords) if not isinstance(coords, np.ndarray) else coords)
    return np.ascontiguousarray(a.reshape(-1, 3).astype(np.int32))
