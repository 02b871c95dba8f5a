"""CPU-only checks of the C ABI library and the host-side logic (no GPU).

* the library loads and exports every entry point declared in
  include/voxmesh_b200.h (no compute calls: there is no device here);
* the __constant__ tables baked into csrc/vm_device.cuh agree with the
  geometry derived from the reference's corner/edge numbering;
* host helpers with reference semantics (hash_block, detect_disturbance,
  block_in_frustum, truncate) agree with the CPU oracle.
"""
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _header_symbols():
    text = (ROOT / "include" / "voxmesh_b200.h").read_text()
    return sorted(set(re.findall(r"^(?:int|const char \*)\s*(vm_\w+)\(", text, re.M)))


def test_library_exports_every_header_symbol():
    from paper_1803_03949_b200 import _lib
    L = _lib.load()
    syms = _header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTED)
    assert L.vm_version().decode().startswith("voxmesh-b200")


def test_engine_creation_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1803_03949_b200 import SpatialStore
    with pytest.raises(RuntimeError, match="CUDA"):
        SpatialStore(0.03)


def test_library_is_sm100a():
    import subprocess
    so = ROOT / "paper_1803_03949_b200" / "libvoxmesh_b200.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _cuh_array(name):
    text = (ROOT / "paper_1803_03949_b200" / "csrc" / "vm_device.cuh").read_text()
    m = re.search(name + r"\[\d+\] = \{([^}]*)\}", text)
    return [int(v, 0) for v in m.group(1).replace(" ", "").split(",")]


def test_device_edge_tables_match_geometry():
    from paper_1803_03949_b200.mc_tables import (EDGE_AXIS, EDGE_END_CORNER,
                                                 EDGE_OWNER_OFFSET, EDGE_START_CORNER, pack_offset)
    assert _cuh_array("c_e_own") == [pack_offset(o) for o in EDGE_OWNER_OFFSET]
    assert _cuh_array("c_e_axis") == list(EDGE_AXIS)
    assert _cuh_array("c_e_start") == list(EDGE_START_CORNER)
    assert _cuh_array("c_e_end") == list(EDGE_END_CORNER)
    from paper_1803_03949_b200.refine import REGULAR_TYPES
    assert tuple(_cuh_array("c_regular")) == REGULAR_TYPES == (0x99, 0x66, 0x33, 0xCC, 0x0F, 0xF0)


def test_tables_integrity():
    """reference tests/test_mesher.py:34-63 on the packed tables."""
    from paper_1803_03949_b200.mc_tables import EDGE_CORNERS, EDGE_TABLE, TRI_TABLE, mc_lookup
    for t in range(256):
        mask = 0
        for e, (a, b) in enumerate(EDGE_CORNERS):
            if ((t >> a) & 1) != ((t >> b) & 1):
                mask |= 1 << e
        assert EDGE_TABLE[t] == mask
        used = 0
        for tri in TRI_TABLE[t]:
            assert len(tri) == 3
            for e in tri:
                used |= 1 << e
        assert used == mask and len(TRI_TABLE[t]) <= 5
    assert mc_lookup(0) == (0, ()) and mc_lookup(255) == (0, ())


def test_hash_block_matches_oracle():
    from oracle.oracle import hash_block as ohash
    from paper_1803_03949_b200.store import hash_block
    rng = np.random.default_rng(0)
    for c in rng.integers(-5000, 5000, size=(500, 3)):
        for ts in (1 << 20, 1 << 21, 1000003, 8):
            assert hash_block(tuple(c), ts) == ohash(tuple(c), ts)


def test_detect_disturbance_matches_oracle_exhaustive():
    """Criterion 10 case set (reference tests/test_acceptance.py:327-373)."""
    from oracle.oracle import detect_disturbance as odet
    from paper_1803_03949_b200.refine import REGULAR_TYPES, RefineParams, detect_disturbance
    from refine_cases import refine_cases
    params = RefineParams(epsilon=0.1)
    n = 0
    for tc, tp, corners in refine_cases():
        assert detect_disturbance(tc, tp, corners, params) == odet(tc, tp, corners, 0.1)
        n += 1
    assert n > 12000


def test_block_in_frustum_host_matches_oracle():
    from oracle.oracle import block_in_frustum as ofr
    from paper_1803_03949_b200.fusion import Intrinsics, block_in_frustum
    from paper_1803_03949_b200.synth import static_pose
    intr = Intrinsics(64.0, 64.0, 32.0, 24.0, 64, 48)
    rng = np.random.default_rng(1)
    pose = static_pose((0.1, -0.2, 0.05), (0.3, 0.1, 1.0))
    for c in rng.integers(-6, 7, size=(400, 3)):
        assert block_in_frustum(tuple(c), pose, intr, 0.24) == ofr(c, pose.rotation, pose.translation,
                                                                   (64, 64, 32, 24, 64, 48), 0.24)


def test_truncate():
    from paper_1803_03949_b200.fusion import truncate
    assert truncate(0.0, 0.06) == 0.0
    assert truncate(0.03, 0.06) == pytest.approx(0.5)
    assert truncate(-0.2, 0.06) == -1.0 and truncate(0.2, 0.06) == 1.0


def test_bench_byte_model_is_positive():
    import bench
    ds = dict(collected_blocks=1400, new_blocks=100, scope_blocks=1500, halo_blocks=1550,
              edge_placements=290000, new_vertices=30000, changed_cubes=58000,
              triangles_freed=46000, triangles_allocated=81000, normals_computed=78000,
              vertices_freed=12000, fallback_normals=1000)
    b = bench.phase_bytes(ds, 480, 640)
    assert all(v > 0 for v in b.values())
    assert 20e6 < sum(b.values()) < 200e6
