"""GPU-vs-oracle state comparison (TEST INFRASTRUCTURE -- the checker).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` leg import this module.  It diffs a B200 ``Engine`` against an
``OracleEngine`` (oracle/oracle.py, the serial C restatement of the reference)
that consumed the same f64 depth frames and poses:

* the StatsRow columns the reference pins (engine.py:123-165), every frame;
* the block set and, per block, tsdf / weight / type_prev / type_curr
  (store.py:70-81, mesher.py:111-134) -- bit-exact;
* the compact mesh (store.py:388-425): positions, triangle indices and ages
  bit-exact, normals within ``NORMAL_ATOL`` (unit vectors; they are expected
  bit-exact too, the face-normal fallback sums in the reference's order).

The north star's tolerances (TSDF 1e-5 relative, positions 1e-4 voxel) are
looser than what is checked here; the measured differences are reported so
a regression shows how far off it is, not only that it failed.
"""
from __future__ import annotations

import numpy as np

NORMAL_ATOL = 1e-12
STAT_KEYS = ("frame", "blocks_active", "vertices_live", "triangles_live",
             "vertices_allocated_total", "vertices_recycled_total", "irregular_cube_count")


def stats_tuple_gpu(row) -> tuple:
    return tuple(int(getattr(row, k)) for k in STAT_KEYS)


def stats_tuple_oracle(row: dict) -> tuple:
    return tuple(int(row[k]) for k in STAT_KEYS)


def compare_rows(gpu_rows, oracle_rows) -> dict:
    """Per-frame StatsRow comparison; returns the first mismatching frame."""
    n = min(len(gpu_rows), len(oracle_rows))
    first = None
    for i in range(n):
        if stats_tuple_gpu(gpu_rows[i]) != stats_tuple_oracle(oracle_rows[i]):
            first = i
            break
    return {"frames": n, "match": first is None and len(gpu_rows) == len(oracle_rows),
            "first_mismatch": first}


def compare_state(engine, oracle_engine, *, blocks: bool = True) -> dict:
    """Final-state diff of a GPU engine and an oracle engine at the same frame.
    Returns a dict of named checks (bool) plus measured differences."""
    out: dict = {}
    mesh = engine.compact()
    pos, nrm, ages, idx = oracle_engine.compact()
    out["vertices"] = int(len(pos))
    out["triangles"] = int(len(idx))
    same_shape = mesh.positions.shape == pos.shape and mesh.indices.shape == idx.shape
    out["mesh_indices"] = bool(same_shape and np.array_equal(mesh.indices, idx))
    out["mesh_positions"] = bool(same_shape and np.array_equal(mesh.positions, pos))
    out["mesh_ages"] = bool(same_shape and np.array_equal(mesh.ages, ages))
    if same_shape and len(pos):
        d = float(np.abs(mesh.normals - nrm).max())
        out["normal_max_abs_diff"] = d
        out["mesh_normals"] = bool(d <= NORMAL_ATOL)
        out["position_max_abs_diff_voxels"] = float(np.abs(mesh.positions - pos).max()
                                                    / engine.store.cube_size)
    else:
        out["mesh_normals"] = bool(same_shape)
    if blocks:
        g = engine.store.snapshot_arrays()
        o = oracle_engine.store.snapshot_blocks()
        out["blocks"] = int(len(o["coords"]))
        same = g["coords"].shape == o["coords"].shape and np.array_equal(g["coords"], o["coords"])
        out["block_set"] = bool(same)
        for k in ("tsdf", "weight", "type_prev", "type_curr"):
            out[k] = bool(same and np.array_equal(g[k], o[k]))
        if same and len(o["coords"]):
            den = np.maximum(np.abs(o["tsdf"]), 1e-12)
            out["tsdf_max_rel_diff"] = float((np.abs(g["tsdf"] - o["tsdf"]) / den).max())
    checks = [v for k, v in out.items() if isinstance(v, bool)]
    out["match"] = bool(all(checks))
    return out


__all__ = ["NORMAL_ATOL", "STAT_KEYS", "compare_rows", "compare_state", "stats_tuple_gpu",
           "stats_tuple_oracle"]
