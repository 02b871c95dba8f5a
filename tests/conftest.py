"""Shared pytest configuration.

Markers: ``gpu`` = needs a CUDA device (run on the B200 box via gpurun);
everything else runs on CPU in the builder container.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def load_golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


ENGINE_SCENES = ("wall", "sphere_orbit", "tilted_refine", "room_noise_refine", "room_frustum",
                 "gc_carve", "sphere_box")
FIELD_SCENES = ("fields_s0_r0", "fields_s7_r1")


def cfg_from_golden(g: dict) -> dict:
    c = g["cfg"]
    return dict(cube_size=float(c[0]), trunc=float(c[1]), epsilon=float(c[2]),
                refine=bool(c[3]), max_range=float(c[4]), frustum_only=bool(c[5]),
                weight_cap=int(c[6]), table_size=int(c[7]))


@pytest.fixture
def golden():
    return load_golden


def edge_use_counts(indices) -> dict:
    """Undirected edge -> number of incident triangles (reference conftest.py:47-54)."""
    counts: dict = {}
    for a, b, c in np.asarray(indices):
        for e in ((a, b), (b, c), (c, a)):
            key = (min(e), max(e))
            counts[key] = counts.get(key, 0) + 1
    return counts
