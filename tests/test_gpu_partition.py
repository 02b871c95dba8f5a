"""Spatial partition on one GPU: N engines,
one per simulated rank, each fed the same frames.  The combined per-frame
StatsRow and the merged compaction must equal the reference's golden output
(and a single engine's) bit for bit, for every tile size and rank count --
including tile_blocks=1, where every block borders another rank's tile.
"""
import numpy as np
import pytest

from conftest import ENGINE_SCENES, cfg_from_golden, load_golden
from test_gpu_parity import NORMAL_ATOL, _check_mesh, _pose, _stats_tuple

pytestmark = pytest.mark.gpu


def _rank_engines(g, nranks, tile_blocks):
    from paper_1803_03949_b200 import Engine, Intrinsics, RunConfig
    cfg = cfg_from_golden(g)
    i6 = g["intr6"]
    intr = Intrinsics(float(i6[0]), float(i6[1]), float(i6[2]), float(i6[3]), int(i6[4]), int(i6[5]))
    return [Engine(RunConfig(rank=r, nranks=nranks, tile_blocks=tile_blocks, **cfg), intr)
            for r in range(nranks)]


def _combined_rows(engines, combiner, frame):
    from paper_1803_03949_b200.partition import sum_stats
    g = combiner.combine(sum_stats([e.device_stats[-1] for e in engines]))
    return (frame, g["blocks_active"], g["vertices_live"], g["triangles_live"],
            g["vertices_allocated_total"], g["vertices_recycled_total"], g["irregular_cube_count"])


def _merged_mesh(engines):
    from paper_1803_03949_b200.partition import export_blocks, merge_compact
    parts = [export_blocks(e.store) for e in engines]
    return parts, merge_compact(parts, engines[0].store.cube_size, engines[0].frame_index)


@pytest.mark.parametrize("name", ENGINE_SCENES)
@pytest.mark.parametrize("nranks,tile_blocks", [(2, 1), (3, 2), (4, 8)])
def test_partitioned_engines_match_reference_golden(name, nranks, tile_blocks):
    from paper_1803_03949_b200.partition import StatsCombiner
    g = load_golden(name)
    engines = _rank_engines(g, nranks, tile_blocks)
    comb = StatsCombiner()
    for i in range(len(g["depth"])):
        for e in engines:
            e.fuse_frame(g["depth"][i], _pose(g, i))
        assert _combined_rows(engines, comb, i) == tuple(g["stats"][i]), (name, i)
    parts, mesh = _merged_mesh(engines)
    # owned blocks partition the reference's block set
    coords = np.concatenate([p["coords"] for p in parts])
    assert len(coords) == len(g["coords"])
    order = np.lexsort((coords[:, 2], coords[:, 1], coords[:, 0]))
    assert np.array_equal(coords[order], g["coords"])
    _check_mesh(mesh, g)


def test_partitioned_room_prefix_matches_single_engine():
    """C2-shaped room (640x480, 8 mm) prefix: partition of 2 and 3 ranks vs one engine."""
    from paper_1803_03949_b200 import Engine, RunConfig
    from paper_1803_03949_b200.partition import StatsCombiner
    from paper_1803_03949_b200.synth import camera_pose, config_spec, render_depth
    spec, cfg = config_spec("C2")
    intr = spec.intrinsics()
    single = Engine(RunConfig(**cfg), intr)
    groups = {n: [Engine(RunConfig(rank=r, nranks=n, tile_blocks=4, **cfg), intr) for r in range(n)]
              for n in (2, 3)}
    combs = {n: StatsCombiner() for n in groups}
    for i in range(0, 40, 4):
        pose = camera_pose(spec, i)
        d = render_depth(spec, pose)
        row = single.fuse_frame(d, pose)
        for n, engines in groups.items():
            for e in engines:
                e.fuse_frame(d, pose)
            assert _combined_rows(engines, combs[n], row.frame) == _stats_tuple(row), (n, i)
    ref = single.compact()
    for n, engines in groups.items():
        _, mesh = _merged_mesh(engines)
        assert np.array_equal(mesh.indices, ref.indices)
        assert np.array_equal(mesh.positions, ref.positions)
        assert np.array_equal(mesh.ages, ref.ages)
        assert np.allclose(mesh.normals, ref.normals, rtol=0, atol=NORMAL_ATOL)


# ---- halo exchange + distributed compaction (in-process ranks) -------------
from partition_sim import fuse_all, rank_engines  # noqa: E402


def _intr_of(g):
    from paper_1803_03949_b200 import Intrinsics
    i6 = g["intr6"]
    return Intrinsics(float(i6[0]), float(i6[1]), float(i6[2]), float(i6[3]), int(i6[4]), int(i6[5]))


@pytest.mark.parametrize("name", ENGINE_SCENES)
@pytest.mark.parametrize("halo", ["margin", "exchange", "exchange-shard"])
@pytest.mark.parametrize("nranks,tile_blocks", [(2, 1), (3, 2), (4, 8)])
def test_distributed_compaction_and_halo_exchange_match_reference_golden(name, halo, nranks, tile_blocks):
    """Halo exchange (owners integrate; boundary blocks all-gathered and
    adopted by the ranks whose margin they are in, before meshing) and the
    distributed compaction (owned-block metadata merged by key, each rank
    fills its global ranges, ranges summed): rows and mesh equal the
    reference's golden output bit for bit."""
    from paper_1803_03949_b200.partition import StatsCombiner, compact_local, sum_stats
    g = load_golden(name)
    engines = rank_engines(cfg_from_golden(g), _intr_of(g), nranks, tile_blocks, halo)
    comb = StatsCombiner()
    log = []
    for i in range(len(g["depth"])):
        rows = fuse_all(engines, g["depth"][i], _pose(g, i), halo, log)
        c = comb.combine(sum_stats(rows))
        got = (i, c["blocks_active"], c["vertices_live"], c["triangles_live"],
               c["vertices_allocated_total"], c["vertices_recycled_total"], c["irregular_cube_count"])
        assert got == tuple(g["stats"][i]), (name, i)
    if halo != "margin" and tile_blocks == 1:
        assert sum(map(sum, log)) > 0                  # records actually crossed ranks
    _check_mesh(compact_local([e.store for e in engines], engines[0].frame_index), g)


def test_halo_exchange_integrates_owned_blocks_only():
    """In exchange mode a rank's band walk collects only its owned blocks and
    the margin arrives by the exchange: the collected set (owned + adopted
    margin) equals margin mode's, rows and the mesh are identical, and
    records did cross ranks."""
    from paper_1803_03949_b200.synth import camera_pose, config_spec, render_depth
    spec, cfg = config_spec("C2")
    spec.width, spec.height, spec.fx, spec.fy = 320, 240, 262.5, 262.5
    intr = spec.intrinsics()
    m = rank_engines(cfg, intr, 2, 8, "margin")
    x = rank_engines(cfg, intr, 2, 8, "exchange")
    xs = rank_engines(cfg, intr, 2, 8, "exchange-shard")
    log = []
    for i in range(0, 12, 3):
        pose = camera_pose(spec, i)
        d = render_depth(spec, pose)
        rm = fuse_all(m, d, pose, "margin")
        rx = fuse_all(x, d, pose, "exchange", log)
        rs = fuse_all(xs, d, pose, "exchange-shard")
        for a, b in zip(rx, rs):   # (the sharded band walk collects the same blocks)
            assert a["collected_blocks"] == b["collected_blocks"]
            for k in ("blocks_active", "vertices_live", "triangles_live", "irregular_cube_count"):
                assert a[k] == b[k], k
        for a, b in zip(rm, rx):
            assert b["collected_blocks"] == a["collected_blocks"]      # owned + adopted margin
            for k in ("blocks_active", "vertices_live", "triangles_live", "irregular_cube_count"):
                assert a[k] == b[k], k
    assert all(sum(c) > 0 for c in log)
    from paper_1803_03949_b200.partition import compact_local
    ma = compact_local([e.store for e in m], m[0].frame_index)
    mb = compact_local([e.store for e in x], x[0].frame_index)
    assert np.array_equal(ma.indices, mb.indices) and np.array_equal(ma.positions, mb.positions)
    assert np.array_equal(ma.normals, mb.normals)


@pytest.mark.slow
@pytest.mark.parametrize("halo", ["margin", "exchange", "exchange-shard"])
def test_c2_halo_modes_full_resolution_match_oracle(halo):
    """C2 (640x480, 8 mm), 2 and 4 ranks, 16 frames: rows every frame and the
    distributed compaction against the CPU oracle."""
    import torch
    from oracle.oracle import OracleEngine
    from oracle.parity import NORMAL_ATOL, stats_tuple_oracle
    from paper_1803_03949_b200.partition import StatsCombiner, compact_local, sum_stats
    from paper_1803_03949_b200.synth import camera_pose, config_spec, render_depth_torch
    spec, cfg = config_spec("C2")
    intr = spec.intrinsics()
    groups = {n: rank_engines(cfg, intr, n, 8, halo) for n in (2, 4)}
    combs = {n: StatsCombiner() for n in groups}
    ora = OracleEngine(cfg, (intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height))
    for i in range(16):
        pose = camera_pose(spec, i)
        d = render_depth_torch(spec, pose)
        torch.cuda.synchronize()
        ref = stats_tuple_oracle(ora.fuse_frame(d.cpu().numpy(), pose.rotation, pose.translation))
        for n, engines in groups.items():
            c = combs[n].combine(sum_stats(fuse_all(engines, d, pose, halo)))
            got = (i, c["blocks_active"], c["vertices_live"], c["triangles_live"],
                   c["vertices_allocated_total"], c["vertices_recycled_total"], c["irregular_cube_count"])
            assert got == ref, (n, i)
    pos, nrm, ages, idx = ora.compact()
    for n, engines in groups.items():
        mesh = compact_local([e.store for e in engines], 16)
        assert np.array_equal(mesh.indices, idx), n
        assert np.array_equal(mesh.positions, pos), n
        assert np.array_equal(mesh.ages, ages), n
        assert np.allclose(mesh.normals, nrm, rtol=0, atol=NORMAL_ATOL), n
