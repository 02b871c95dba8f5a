"""Frame overlap: pipelined submission of device-resident
frames on the engine's own stream launches frame t+1's k_collect right behind
frame t's k_gc_normals, which lets it start (cudaTriggerProgrammaticLaunchCompletion)
once its collect counters are saved; the collect skips the grid-dependency wait
and runs the work that depends on frame t (fallback records, record ranges,
the snapshot publish) after frame t's commit.

Every result must be the synchronous engine's and the oracle's, bit for bit:
StatsRow columns and unit counts per frame, the final state and the compact
mesh -- also when frames resume after heap / record growth and when a
collect-time CapacityError is raised while the previous frame's gc runs.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROW_KEYS = ("frame", "blocks_active", "vertices_live", "triangles_live", "vertices_allocated_total",
            "vertices_recycled_total", "irregular_cube_count", "valid_pixels", "nsteps", "collected_blocks",
            "new_blocks", "scope_blocks", "halo_blocks", "active_cubes", "edge_placements", "new_vertices",
            "changed_cubes", "triangles_freed", "triangles_allocated", "vertices_freed", "normals_computed",
            "fallback_normals", "refined_cubes")


def _frames(config, n):
    import torch
    from paper_1803_03949_b200.synth import camera_pose, config_spec, render_depth_torch
    spec, cfg = config_spec(config)
    poses = [camera_pose(spec, i) for i in range(n)]
    depths = [render_depth_torch(spec, p, device="cuda") for p in poses]
    torch.cuda.synchronize()
    return spec, cfg, poses, depths


def _run(spec, cfg, poses, depths, pipelined, **over):
    from paper_1803_03949_b200 import Engine, RunConfig
    eng = Engine(RunConfig(**cfg, **over), spec.intrinsics(), pipelined=pipelined)
    for d, p in zip(depths, poses):
        eng.fuse_frame(d, p)
    eng.stats[-1].blocks_active   # (completes the frame in flight)
    return eng


def _rows(eng):
    return [tuple(d[k] for k in ROW_KEYS) for d in eng.device_stats]


def _same_mesh(a, b):
    ma, mb = a.compact(), b.compact()
    assert np.array_equal(ma.indices, mb.indices)
    assert np.array_equal(ma.positions, mb.positions)
    assert np.array_equal(ma.ages, mb.ages)
    assert np.array_equal(ma.normals, mb.normals)
    return len(ma.positions)


@pytest.mark.parametrize("config", ["C2", "C3"])
def test_overlapped_frames_match_synchronous_engine(config):
    """C2 / C3 (refinement) at 640x480, 40 frames back to back."""
    spec, cfg, poses, depths = _frames(config, 40)
    caps = dict(block_capacity=30_000, vertex_capacity=12_000_000)   # (no arena growth: no resumes)
    ov = _run(spec, cfg, poses, depths, pipelined=True, **caps)
    sync = _run(spec, cfg, poses, depths, pipelined=False)
    flags = [d["overlapped"] for d in ov.device_stats]
    assert flags[0] == 0 and all(flags[1:]), flags      # every frame after the first overlapped
    assert sum(d["overlapped"] for d in sync.device_stats) == 0
    assert _rows(ov) == _rows(sync)
    assert _same_mesh(ov, sync) > 100_000
    assert ov.audit().ok


def test_overlapped_frames_match_oracle():
    """The overlapped engine against the CPU oracle directly (C2, 16 frames)."""
    from oracle.oracle import OracleEngine
    from oracle.parity import compare_rows, compare_state
    spec, cfg, poses, depths = _frames("C2", 16)
    intr = spec.intrinsics()
    ov = _run(spec, cfg, poses, depths, pipelined=True, block_capacity=30_000, vertex_capacity=12_000_000)
    ora = OracleEngine(cfg, (intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height))
    for d, p in zip(depths, poses):
        ora.fuse_frame(d.cpu().numpy(), p.rotation, p.translation)
    r = compare_rows(ov.stats, ora.stats)
    assert r["match"], r
    s = compare_state(ov, ora)
    assert s["match"], s
    assert sum(d["overlapped"] for d in ov.device_stats) >= 14


@pytest.mark.parametrize("caps", [dict(block_capacity=64), dict(vertex_capacity=2048),
                                  dict(block_capacity=300, vertex_capacity=50_000)])
def test_overlapped_frames_resume_after_growth(caps):
    """Tiny arenas: frames stop at the heap / record guards (a queued,
    overlapped k_collect sees the guard and writes nothing), the host grows
    the arena, resumes the frame and launches the queued one again."""
    spec, cfg, poses, depths = _frames("C2", 12)
    ov = _run(spec, cfg, poses, depths, pipelined=True, **caps)
    sync = _run(spec, cfg, poses, depths, pipelined=False)
    assert sum(d["resumes"] for d in ov.device_stats) > 0
    assert _rows(ov) == _rows(sync)
    _same_mesh(ov, sync)


def test_collect_capacity_error_raised_for_its_own_frame():
    """A table that fills up at frame k: the overlapped k_collect of frame k
    raises while frame k-1's gc still runs -- frame k-1 must still complete
    with its own row, and the error belong to frame k, as in the synchronous
    engine."""
    from paper_1803_03949_b200 import CapacityError, Engine, RunConfig
    spec, cfg, poses, depths = _frames("C2", 30)
    table = 2 * 3000
    sync = Engine(RunConfig(**cfg, table_size=table), spec.intrinsics())
    k = None
    for i, (d, p) in enumerate(zip(depths, poses)):
        try:
            sync.fuse_frame(d, p)
        except CapacityError:
            k = i
            break
    assert k is not None and k >= 2, k
    ov = Engine(RunConfig(**cfg, table_size=table), spec.intrinsics(), pipelined=True)
    raised_at = None
    for i, (d, p) in enumerate(zip(depths[:k + 2], poses[:k + 2])):
        try:
            ov.fuse_frame(d, p)
        except CapacityError:
            raised_at = i
            break
    if raised_at is None:
        with pytest.raises(CapacityError):
            ov.stats[-1].blocks_active
        raised_at = k + 2
    # (pipelined: frame k's error surfaces at the next call)
    assert raised_at == k + 1, (raised_at, k)
    assert [tuple(d[q] for q in ROW_KEYS) for d in ov.device_stats[:k]] == _rows(sync)[:k]
    assert ov.store.block_count == sync.store.block_count


@pytest.mark.parametrize("raw", [False, True])
def test_host_copied_frames_overlap_and_match(raw):
    """Host frames (pinned f64, or raw u16 as read_depth would decode them):
    the copy stream posts a per-slot flag that k_collect waits for, so these
    frames overlap too; rows and mesh equal the synchronous engine's."""
    import torch
    from paper_1803_03949_b200 import Engine, RunConfig
    spec, cfg, poses, depths = _frames("C2", 24)
    caps = dict(block_capacity=30_000, vertex_capacity=12_000_000)
    host = [d.cpu().numpy() for d in depths]
    if raw:
        host = [np.clip(np.rint(h * 5000.0), 0, 65535).astype(np.uint16) for h in host]
        conv = [torch.from_numpy(h.astype(np.float64) / 5000.0).cuda() for h in host]
    ov = Engine(RunConfig(**cfg, **caps), spec.intrinsics(), pipelined=True)
    for h, p in zip(host, poses):
        buf = h.copy()
        (ov.fuse_frame_raw if raw else ov.fuse_frame)(buf, p)
        buf[...] = 0   # (the engine must be done reading it on return)
    ov.stats[-1].blocks_active
    sync = _run(spec, cfg, poses, conv if raw else depths, pipelined=False)
    flags = [d["overlapped"] for d in ov.device_stats]
    assert flags[0] == 0 and sum(flags[1:]) >= len(flags) - 2, flags
    assert _rows(ov) == _rows(sync)
    _same_mesh(ov, sync)


def test_overlap_with_depth_stats_pass_c4():
    """C4 (4 mm, 40 mm band): the band step count depends on the frame's
    valid pixels, so k_depth_stats runs first -- it too starts under the
    previous gc, and the collect waits for its CTAs on a counter."""
    spec, cfg, poses, depths = _frames("C4", 12)
    caps = dict(block_capacity=80_000, vertex_capacity=24_000_000)
    ov = _run(spec, cfg, poses, depths, pipelined=True, **caps)
    sync = _run(spec, cfg, poses, depths, pipelined=False)
    flags = [d["overlapped"] for d in ov.device_stats]
    assert flags[0] == 0 and all(flags[1:]), flags
    assert _rows(ov) == _rows(sync)
    _same_mesh(ov, sync)
