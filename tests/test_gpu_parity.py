"""GPU parity: the CUDA path (through the C ABI) against the reference's own
golden fixtures and against the CPU oracle on identical inputs.

Bit-exact: block sets, TSDF and weights, cube types, triangle topology (compact
indices), vertex positions and ages, StatsRow non-timing columns.  Normals are
also expected bit-exact (the fallback reproduces the reference's summation
order); the written tolerance is 1e-12 (unit vectors).
"""
import numpy as np
import pytest

from conftest import ENGINE_SCENES, FIELD_SCENES, cfg_from_golden, load_golden

pytestmark = pytest.mark.gpu

NORMAL_ATOL = 1e-12


def _engine_from_golden(g, pipelined=False, **over):
    from paper_1803_03949_b200 import Engine, Intrinsics, RunConfig
    cfg = cfg_from_golden(g)
    cfg.update(over)
    i6 = g["intr6"]
    intr = Intrinsics(float(i6[0]), float(i6[1]), float(i6[2]), float(i6[3]), int(i6[4]), int(i6[5]))
    return Engine(RunConfig(**cfg), intr, pipelined=pipelined)


def _pose(g, i):
    from paper_1803_03949_b200 import Pose
    return Pose(g["rot"][i], g["trans"][i])


def _stats_tuple(row):
    return (row.frame, row.blocks_active, row.vertices_live, row.triangles_live,
            row.vertices_allocated_total, row.vertices_recycled_total, row.irregular_cube_count)


def _check_blocks(store, g):
    blocks = list(store.blocks())
    coords = np.array([b.coord for b in blocks], np.int32).reshape(-1, 3)
    assert np.array_equal(coords, g["coords"])
    for k in ("tsdf", "weight", "type_prev", "type_curr"):
        got = np.stack([getattr(b, k) for b in blocks]) if blocks else np.zeros((0,))
        assert np.array_equal(got, g[k]), k
    # slot occupancy pattern (handles differ: GPU allocation order is free)
    ev = np.stack([b.edge_vertex for b in blocks])
    tr = np.stack([b.triangles for b in blocks])
    assert np.array_equal(ev >= 0, g["edge_vertex"] >= 0)
    assert np.array_equal(tr >= 0, g["triangles"] >= 0)


def _check_mesh(mesh, g):
    assert np.array_equal(mesh.indices, g["m_indices"])
    assert np.array_equal(mesh.positions, g["m_positions"])
    assert np.array_equal(mesh.ages, g["m_ages"])
    assert np.allclose(mesh.normals, g["m_normals"], rtol=0, atol=NORMAL_ATOL)


@pytest.mark.parametrize("name", ENGINE_SCENES)
@pytest.mark.parametrize("strategy", ["claim", "partition"])
def test_engine_matches_reference_golden(name, strategy):
    g = load_golden(name)
    eng = _engine_from_golden(g, strategy=strategy)
    for i in range(len(g["depth"])):
        row = eng.fuse_frame(g["depth"][i], _pose(g, i))
        assert _stats_tuple(row) == tuple(g["stats"][i]), (name, i)
        assert eng.audit().ok
    assert eng.irregular_cube_count() == int(g["stats"][-1][6])
    assert sorted(eng.last_collected) == sorted(map(tuple, g["last_collected"].tolist()))
    _check_blocks(eng.store, g)
    _check_mesh(eng.compact(), g)
    a = eng.audit()
    assert [a.vertices_live, a.triangles_live, a.refcount_mismatches, a.duplicate_handles,
            a.zero_ref_live, int(a.conservation_ok)] == list(g["audit"])
    c = eng.store._counters()
    # arena accounting that the reference pins (VertexPool.count/free/recycled/events,
    # TrianglePool live count and recycled total)
    assert c["vertex_count"] == g["counters"][2]
    assert c["vertex_free"] == g["counters"][3]
    assert c["vertex_recycled_total"] == g["counters"][4]
    assert c["vertex_allocation_events"] == g["counters"][5]
    assert c["triangle_count"] - c["triangle_free"] == g["counters"][6] - g["counters"][7]
    assert c["triangle_recycled_total"] == g["counters"][8]
    # pool views: refcounts derived from cube types equal the reference's
    vp = eng.store.vertices
    ref_live = np.sort(g["v_refcount"][g["v_alive"]])
    assert np.array_equal(np.sort(vp.refcount[:vp.live_count]), ref_live)


@pytest.mark.parametrize("name", ENGINE_SCENES)
def test_engine_resume_after_arena_growth(name):
    """Tiny initial arenas force every capacity guard to trip and the frame to
    resume after growth; results must be unchanged."""
    g = load_golden(name)
    eng = _engine_from_golden(g, block_capacity=4, vertex_capacity=16, triangle_capacity=16)
    resumes = 0
    for i in range(len(g["depth"])):
        row = eng.fuse_frame(g["depth"][i], _pose(g, i))
        resumes += eng.device_stats[-1]["resumes"]
        assert _stats_tuple(row) == tuple(g["stats"][i]), (name, i)
    if g["coords"].shape[0] > 16:
        assert resumes > 0
    _check_mesh(eng.compact(), g)


@pytest.mark.parametrize("name", ENGINE_SCENES)
@pytest.mark.parametrize("tiny", [False, True])
def test_pipelined_engine_matches_reference_golden(name, tiny):
    """Pipelined submission (vm_fuse_frame_submit: frame t+1's depth copy
    overlaps frame t's kernels, rows fill in lazily): identical rows, blocks and
    mesh; with tiny arenas every frame also resumes after growth, and a store
    access between frames completes the frame in flight."""
    g = load_golden(name)
    over = dict(block_capacity=4, vertex_capacity=16, triangle_capacity=16) if tiny else {}
    eng = _engine_from_golden(g, pipelined=True, **over)
    rows = []
    for i in range(len(g["depth"])):
        depth = np.array(g["depth"][i])       # a fresh host buffer, overwritten after the call
        rows.append(eng.fuse_frame(depth, _pose(g, i)))
        depth[:] = -1.0                         # the engine must not read it after returning
        if i == 1:
            eng.store._counters()               # completes frame 1 on the device side
    for i, row in enumerate(rows):
        assert _stats_tuple(row) == tuple(g["stats"][i]), (name, i)
    _check_blocks(eng.store, g)
    _check_mesh(eng.compact(), g)
    assert eng.audit().ok


@pytest.mark.parametrize("name", FIELD_SCENES)
@pytest.mark.parametrize("strategy", ["serial", "claim", "partition"])
@pytest.mark.parametrize("tiny", [False, True])
def test_extract_fields_match_reference(name, strategy, tiny):
    """extract_frame through the phase API; with a 16-record vertex arena the
    retype stops at its capacity check and resumes after growth."""
    from paper_1803_03949_b200 import RefineParams, SpatialStore
    from paper_1803_03949_b200.mesher import extract_frame
    g = load_golden(name)
    cfg = cfg_from_golden(g)
    st = SpatialStore(cfg["cube_size"], initial_vertices=16 if tiny else 0)
    coords = [tuple(c) for c in g["in_coords"].tolist()]
    st.set_block_samples(coords, g["in_tsdf"], g["in_weight"])
    scope = [(c, None) for c in sorted(coords)]
    rp = RefineParams(epsilon=cfg["epsilon"], enabled=cfg["refine"])
    r1 = extract_frame(st, scope, 0, strategy=strategy, refine_params=rp, halo=sorted(coords))
    st.set_block_samples(coords, g["in_tsdf2"], None)
    r2 = extract_frame(st, scope, 1, strategy=strategy, refine_params=rp, halo=sorted(coords))
    assert [r1["refined"], r1["freed"], r2["refined"], r2["freed"]] == list(g["extract_out"])
    _check_blocks(st, g)
    _check_mesh(st.compact_mesh(2), g)


def _run_oracle_and_gpu(spec, cfg, frames, strategy="claim", rng=None, pose_fn=None):
    from oracle.oracle import OracleEngine
    from paper_1803_03949_b200 import Engine, RunConfig
    from paper_1803_03949_b200.synth import camera_pose, render_depth
    intr = spec.intrinsics()
    eng = Engine(RunConfig(strategy=strategy, **cfg), intr)
    ora = OracleEngine(cfg, (intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height))
    for i in range(frames):
        pose = (pose_fn or camera_pose)(spec, i)
        d = render_depth(spec, pose, rng)
        row = eng.fuse_frame(d, pose)
        ref = ora.fuse_frame(d, pose.rotation, pose.translation)
        assert _stats_tuple(row) == tuple(ref[k] for k in (
            "frame", "blocks_active", "vertices_live", "triangles_live",
            "vertices_allocated_total", "vertices_recycled_total", "irregular_cube_count")), i
    return eng, ora


def _compare_final(eng, ora):
    m = eng.compact()
    pos, nrm, ages, idx = ora.compact()
    assert np.array_equal(m.indices, idx)
    assert np.array_equal(m.positions, pos)
    assert np.array_equal(m.ages, ages)
    assert np.allclose(m.normals, nrm, rtol=0, atol=NORMAL_ATOL)
    snap = ora.store.snapshot_blocks()
    blocks = list(eng.store.blocks())
    assert np.array_equal(np.array([b.coord for b in blocks], np.int32), snap["coords"])
    assert np.array_equal(np.stack([b.tsdf for b in blocks]), snap["tsdf"])
    assert np.array_equal(np.stack([b.type_curr for b in blocks]), snap["type_curr"])


def test_c1_sphere_box_prefix_matches_oracle():
    """BASELINE config C1 (sphere+box, 320x240, 8 mm), first 4 frames."""
    from paper_1803_03949_b200.synth import config_spec
    spec, cfg = config_spec("C1")
    eng, ora = _run_oracle_and_gpu(spec, cfg, 4)
    _compare_final(eng, ora)


def test_c3_refine_room_prefix_matches_oracle():
    """C3-style refine run at reduced resolution (160x120, 8 mm), 6 frames."""
    from paper_1803_03949_b200.synth import config_spec
    spec, cfg = config_spec("C3")
    spec.width, spec.height, spec.fx, spec.fy = 160, 120, 131.25, 131.25
    eng, ora = _run_oracle_and_gpu(spec, cfg, 6)
    _compare_final(eng, ora)


def test_noisy_partition_matches_oracle():
    from paper_1803_03949_b200.synth import SceneSpec
    spec = SceneSpec(scene="room", room_size=(2.0, 2.0, 1.4), orbit_radius=0.3, look="outward",
                     elevation_amp_deg=30.0, angular_step_deg=20.0, frames=8, width=96, height=72,
                     fx=70.0, fy=70.0, noise_sigma=0.003)
    eng, ora = _run_oracle_and_gpu(spec, dict(cube_size=0.02, refine=True), 8,
                                   strategy="partition", rng=np.random.default_rng(5))
    _compare_final(eng, ora)


def test_run_to_run_and_strategy_determinism():
    from paper_1803_03949_b200.synth import SceneSpec
    spec = SceneSpec(scene="sphere", sphere_radius=0.3, orbit_radius=0.9, elevation_amp_deg=60.0,
                     angular_step_deg=18.0, frames=6, width=96, height=72, fx=80.0, fy=80.0)
    meshes = []
    for strategy in ("serial", "claim", "partition", "claim"):
        eng, _ = _run_oracle_and_gpu(spec, dict(cube_size=0.025), 6, strategy=strategy)
        meshes.append(eng.compact())
    for m in meshes[1:]:
        assert np.array_equal(m.positions, meshes[0].positions)
        assert np.array_equal(m.indices, meshes[0].indices)
        assert np.array_equal(m.normals, meshes[0].normals)


def test_c4_fine_resolution_prefix_matches_oracle():
    """BASELINE config C4 (4 mm cubes, 40 mm band: 8 ray steps) at 320x240, 3 frames."""
    from paper_1803_03949_b200.synth import config_spec
    spec, cfg = config_spec("C4")
    spec.width, spec.height, spec.fx, spec.fy = 320, 240, 262.5, 262.5
    eng, ora = _run_oracle_and_gpu(spec, cfg, 3)
    assert eng.device_stats[-1]["nsteps"] >= 8
    _compare_final(eng, ora)


def test_c5_multiroom_prefix_matches_oracle():
    """BASELINE config C5 (20 x 20 m multi-room, table 2^21) at 320x240, 4 frames."""
    from paper_1803_03949_b200.synth import config_spec, multiroom_pose
    spec, cfg = config_spec("C5")
    spec.width, spec.height, spec.fx, spec.fy = 320, 240, 262.5, 262.5
    eng, ora = _run_oracle_and_gpu(spec, cfg, 4, pose_fn=multiroom_pose)
    _compare_final(eng, ora)


@pytest.mark.parametrize("cube", [0.002, 0.02])
def test_scattered_depth_overflows_collect_set_matches_oracle(cube):
    """Uniform random depth at fine cubes and a wide band: a 64x8-pixel region
    touches far more distinct blocks than k_collect's shared-memory key set
    holds (its overflow list, then the direct-probe pass); at 2 cm the set does
    not overflow.  Block set, TSDF and mesh must equal the oracle's."""
    from oracle.oracle import OracleEngine
    from paper_1803_03949_b200 import Engine, Intrinsics, Pose, RunConfig
    rng = np.random.default_rng(7)
    w, h = 64, 32
    intr = Intrinsics(40.0, 40.0, (w - 1) / 2, (h - 1) / 2, w, h)
    cfg = dict(cube_size=cube, trunc=max(0.03, 2 * cube), table_size=1 << 22)
    eng = Engine(RunConfig(**cfg), intr)
    ora = OracleEngine(cfg, (intr.fx, intr.fy, intr.cx, intr.cy, w, h))
    for i in range(2):
        d = rng.uniform(0.3, 3.0, size=(h, w))
        d[rng.random((h, w)) < 0.05] = 0.0
        pose = Pose(np.eye(3), np.array([0.01 * i, 0.0, 0.0]))
        row = eng.fuse_frame(d, pose)
        ref = ora.fuse_frame(d, pose.rotation, pose.translation)
        assert _stats_tuple(row) == tuple(ref[k] for k in (
            "frame", "blocks_active", "vertices_live", "triangles_live",
            "vertices_allocated_total", "vertices_recycled_total", "irregular_cube_count")), i
    _compare_final(eng, ora)


@pytest.mark.parametrize("config", ["C1", "C4"])
@pytest.mark.parametrize("pipelined", [False, True])
def test_raw_u16_depth_matches_converted_frames(config, pipelined):
    """fuse_frame_raw (device-side read_depth conversion, io_formats.py:84) is
    bit-identical to fuse_frame on the host-converted f64 frames; C4's band
    step count depends on the depth, so its raw frame is converted by
    k_depth_stats, C1's by k_collect."""
    from paper_1803_03949_b200 import Engine, RunConfig
    from paper_1803_03949_b200.synth import camera_pose, config_spec, render_depth
    spec, cfg = config_spec(config)
    spec.width, spec.height = 160, 120
    spec.fx = spec.fy = 131.25 if config == "C4" else 65.6
    scale = 5000.0
    intr = spec.intrinsics()
    a = Engine(RunConfig(**cfg), intr)
    b = Engine(RunConfig(**cfg), intr, pipelined=pipelined)
    rows_b = []
    for i in range(3):
        pose = camera_pose(spec, i)
        raw = np.clip(np.rint(render_depth(spec, pose) * scale), 0, 65535).astype(np.uint16)
        ra = a.fuse_frame(raw.astype(np.float64) / scale, pose)
        rows_b.append(b.fuse_frame_raw(raw, pose, depth_scale=scale))
        assert _stats_tuple(rows_b[-1]) == _stats_tuple(ra), i
    ma, mb = a.compact(), b.compact()
    assert np.array_equal(ma.indices, mb.indices) and np.array_equal(ma.positions, mb.positions)
    assert np.array_equal(ma.normals, mb.normals)
    ba, bb = list(a.store.blocks()), list(b.store.blocks())
    assert np.array_equal(np.stack([x.tsdf for x in ba]), np.stack([x.tsdf for x in bb]))


@pytest.mark.parametrize("name", ["sphere_orbit", "room_noise_refine"])
def test_halo_shard_spill_matches_reference_golden(name, monkeypatch):
    """The frame's halo list is appended into 32 sharded sub-lists; a full
    shard spills into the general list.  With 3-entry shards nearly every
    append spills: rows, blocks and mesh stay identical, and the pipelined
    rows carry the kernels' own device time."""
    monkeypatch.setenv("VOXMESH_B200_HALO_SHARD_CAP", "3")
    g = load_golden(name)
    eng = _engine_from_golden(g, pipelined=True)
    rows = [eng.fuse_frame(g["depth"][i], _pose(g, i)) for i in range(len(g["depth"]))]
    for i, row in enumerate(rows):
        assert _stats_tuple(row) == tuple(g["stats"][i]), (name, i)
    assert all(d["device_ms"] > 0 for d in eng.device_stats)
    _check_blocks(eng.store, g)
    _check_mesh(eng.compact(), g)


@pytest.mark.parametrize("cap", ["0", "5"])
@pytest.mark.parametrize("name", ["sphere_orbit", "room_noise_refine", "gc_carve"])
def test_fallback_ring_overflow_applied_inline_matches_reference_golden(name, cap, monkeypatch):
    """Face-normal fallback records live in a bounded ring until the next
    frame applies them; records past it are applied inline by k_gc_normals.
    With a 0- or 5-record ring (all or nearly all inline) every row, block and
    the mesh, normals included, stay identical -- pipelined and synchronous."""
    monkeypatch.setenv("VOXMESH_B200_FALLBACK_CAP", cap)
    g = load_golden(name)
    for pipelined in (False, True):
        eng = _engine_from_golden(g, pipelined=pipelined)
        rows = [eng.fuse_frame(g["depth"][i], _pose(g, i)) for i in range(len(g["depth"]))]
        for i, row in enumerate(rows):
            assert _stats_tuple(row) == tuple(g["stats"][i]), (name, i)
        assert sum(d["fallback_normals"] for d in eng.device_stats) > int(cap)   # (the inline path ran)
        _check_blocks(eng.store, g)
        _check_mesh(eng.compact(), g)


def test_vertex_records_are_compact_and_accounted():
    """Birth and normal live in a vertex-record arena indexed by a per-slot
    handle: a slot gets a record when first occupied and keeps it.  Records in
    use cover the live vertices and stay far below 1536 per block; the store's
    HBM accounting is blocks x per-block bytes + records x 32 B."""
    g = load_golden("gc_carve")
    eng = _engine_from_golden(g)
    for i in range(len(g["depth"])):
        eng.fuse_frame(g["depth"][i], _pose(g, i))
    c = eng.store._counters()
    live = eng.stats[-1].vertices_live
    assert live <= c["vertex_records"] <= c["vertex_allocation_events"]
    assert c["vertex_records"] < 0.25 * 1536 * c["block_count"]
    per_block = 8 * 512 + 4 * 512 + 64 + 2 * 512 + 8 * 1536 + 4 * 1536 + 3 * 192 + 64
    assert c["store_bytes"] == c["block_count"] * per_block + 32 * c["vertex_records"]
    assert c["device_bytes"] >= c["store_bytes"]
