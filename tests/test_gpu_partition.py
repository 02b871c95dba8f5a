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
