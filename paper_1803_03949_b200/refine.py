"""Hamming-distance cube-type refinement: parameters and scalar rule.

The per-cube rule runs on the device inside ``k_retype``
(csrc/vm_device.cuh: refine_type); this module keeps the reference's public
names (pkg/src/voxmesh/refine.py:29-140).  ``detect_disturbance`` is the
reference's scalar statement of Eq. 3-5 and is what the exhaustive KAT
compares the device kernel against
(tests/test_gpu_reference_suite.py::test_refine_kernel_exhaustive_eq3_5).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .mc_tables import CORNER_OFFSETS

HAMMING_RADIUS = 3


def _regular_types():
    out = []
    for axis in range(3):
        for side in (0, 1):
            out.append(sum(1 << k for k, off in enumerate(CORNER_OFFSETS) if off[axis] == side))
    return tuple(out)


# face-parallel split types, ordered (x-, x+, y-, y+, z-, z+)
REGULAR_TYPES = _regular_types()
_POPCOUNT = np.array([bin(i).count("1") for i in range(256)], dtype=np.int64)


@dataclass
class RefineParams:
    """epsilon is in normalised tsdf units, so it scales with cube size."""

    epsilon: float = 0.1
    enabled: bool = True


def hamming(a: int, b: int) -> int:
    """Number of differing bits between two 8-bit cube types."""
    return int(_POPCOUNT[(a ^ b) & 0xFF])


def detect_disturbance(t_curr: int, t_prev: int, corner_tsdf, params: RefineParams):
    """Regular type to snap to, or None (temporal, proximity and magnitude gates)."""
    if not params.enabled or hamming(t_curr, t_prev) > HAMMING_RADIUS:
        return None
    c = np.asarray(corner_tsdf, dtype=np.float64)
    best, best_dist = None, HAMMING_RADIUS + 1
    for reg in REGULAR_TYPES:
        dist = hamming(t_curr, reg)
        if dist > HAMMING_RADIUS or dist >= best_dist:
            continue
        diff = t_curr ^ reg
        if all(abs(float(c[k])) < params.epsilon for k in range(8) if (diff >> k) & 1):
            best, best_dist = reg, dist
    return best
