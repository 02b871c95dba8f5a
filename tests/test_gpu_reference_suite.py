"""The reference's own test suite (pkg/tests/*.py) ported to the CUDA path.

Each test cites the reference test it mirrors.  Known-answer values are the
reference's (fusion KATs, table/type KATs, sharing counts, Euler
characteristic, acceptance criteria).
"""
import numpy as np
import pytest

from conftest import edge_use_counts

pytestmark = pytest.mark.gpu

B = 8


def _intr():
    from paper_1803_03949_b200 import Intrinsics
    return Intrinsics(fx=64.0, fy=64.0, cx=32.0, cy=24.0, width=64, height=48)


def _single_pixel(depth_value, u=32, v=24):
    from paper_1803_03949_b200 import DepthFrame
    px = np.zeros((48, 64))
    px[v, u] = depth_value
    return DepthFrame(px)


# ---------------------------------------------------------------- fusion (test_fusion.py)
def test_collect_single_pixel_band():            # test_fusion.py:50-60
    from paper_1803_03949_b200 import Pose, SpatialStore
    from paper_1803_03949_b200.fusion import collect_blocks
    st = SpatialStore(cube_size=0.03)
    got = collect_blocks(st, _single_pixel(1.0), Pose.identity(), _intr(), trunc=0.06)
    assert set(got) == {(0, 0, 3), (0, 0, 4)}


def test_collect_all_invalid_and_out_of_range():  # test_fusion.py:63-76
    from paper_1803_03949_b200 import DepthFrame, Pose, SpatialStore
    from paper_1803_03949_b200.fusion import collect_blocks
    st = SpatialStore(cube_size=0.03)
    assert collect_blocks(st, DepthFrame(np.zeros((48, 64))), Pose.identity(), _intr(), 0.06) == []
    assert st.block_count == 0
    assert collect_blocks(st, _single_pixel(3.5), Pose.identity(), _intr(), 0.06, max_range=2.0) == []


def test_collect_idempotent():                    # test_fusion.py:79-85
    from paper_1803_03949_b200 import Pose, SpatialStore
    from paper_1803_03949_b200.fusion import collect_blocks
    st = SpatialStore(cube_size=0.03)
    a = collect_blocks(st, _single_pixel(1.0), Pose.identity(), _intr(), trunc=0.06)
    n = st.block_allocations
    assert collect_blocks(st, _single_pixel(1.0), Pose.identity(), _intr(), trunc=0.06) == a
    assert st.block_allocations == n


def test_integrate_first_write_and_running_average():   # test_fusion.py:90-113
    from paper_1803_03949_b200 import Pose, SpatialStore
    from paper_1803_03949_b200.fusion import collect_blocks, integrate_frame
    st = SpatialStore(cube_size=0.03)
    f1, f2 = _single_pixel(1.0), _single_pixel(0.92)
    b1 = collect_blocks(st, f1, Pose.identity(), _intr(), trunc=0.08)
    integrate_frame(st, b1, f1, Pose.identity(), _intr(), trunc=0.08)
    d, w = st.corner_sample((0, 0, 32))
    assert w == 1 and d == pytest.approx(0.5, abs=1e-12)
    b2 = collect_blocks(st, f2, Pose.identity(), _intr(), trunc=0.08)
    integrate_frame(st, b2, f2, Pose.identity(), _intr(), trunc=0.08)
    d, w = st.corner_sample((0, 0, 32))
    assert w == 2 and d == pytest.approx(0.0, abs=1e-15)


def test_integrate_wall_corner_and_weight_cap():       # test_fusion.py:116-143
    from paper_1803_03949_b200 import DepthFrame, Intrinsics, Pose, SpatialStore
    from paper_1803_03949_b200.fusion import collect_blocks, integrate_frame
    intr = Intrinsics(50.0, 50.0, 24.0, 24.0, 48, 48)
    st = SpatialStore(cube_size=0.025)
    frame = DepthFrame(np.full((48, 48), 1.0))
    for _ in range(10):
        b = collect_blocks(st, frame, Pose.identity(), intr, trunc=0.075)
        integrate_frame(st, b, frame, Pose.identity(), intr, trunc=0.075)
    d, w = st.corner_sample((0, 0, 40))
    assert w == 10 and abs(d) <= 1e-6
    st = SpatialStore(cube_size=0.03)
    last = 0
    for _ in range(6):
        b = collect_blocks(st, _single_pixel(1.0), Pose.identity(), _intr(), trunc=0.08)
        integrate_frame(st, b, _single_pixel(1.0), Pose.identity(), _intr(), trunc=0.08, weight_cap=4)
        _, w = st.corner_sample((0, 0, 32))
        assert w >= last
        last = w
    assert last == 4


def test_untouched_beyond_band():                      # test_fusion.py:175-191
    from paper_1803_03949_b200 import Pose, SpatialStore
    from paper_1803_03949_b200.fusion import collect_blocks, integrate_frame
    st = SpatialStore(cube_size=0.03)
    b = collect_blocks(st, _single_pixel(1.0), Pose.identity(), _intr(), trunc=0.08)
    integrate_frame(st, b, _single_pixel(1.0), Pose.identity(), _intr(), trunc=0.08)
    for blk in st.blocks():
        for x, y, z in np.argwhere(blk.weight > 0):
            assert (blk.coord[2] * 8 + z) * 0.03 <= 1.0 + 0.08 + 1e-9
    assert st.corner_sample((0, 0, 37))[1] == 0


def test_order_insensitive_below_saturation():         # test_fusion.py:194-215
    from paper_1803_03949_b200 import DepthFrame, Intrinsics, SpatialStore
    from paper_1803_03949_b200.fusion import collect_blocks, integrate_frame
    from paper_1803_03949_b200.synth import static_pose
    intr = Intrinsics(50.0, 50.0, 24.0, 24.0, 48, 48)
    pose = static_pose((0, 0, 0), (0, 0, 1))
    frames = [DepthFrame(np.full((48, 48), 1.0)), DepthFrame(np.full((48, 48), 1.02))]

    def fuse(order):
        st = SpatialStore(cube_size=0.025)
        for f in order:
            b = collect_blocks(st, f, pose, intr, trunc=0.075)
            integrate_frame(st, b, f, pose, intr, trunc=0.075)
        return {blk.coord: (blk.tsdf.copy(), blk.weight.copy()) for blk in st.blocks()}

    ab, ba = fuse(frames), fuse(frames[::-1])
    assert ab.keys() == ba.keys()
    for k in ab:
        assert np.array_equal(ab[k][1], ba[k][1])
        assert np.allclose(ab[k][0], ba[k][0], atol=1e-12, rtol=0)


def test_frustum_device_matches_host():               # test_fusion.py:238-252 + engine filter
    from paper_1803_03949_b200 import SpatialStore
    from paper_1803_03949_b200.fusion import block_in_frustum, block_in_frustum_device
    from paper_1803_03949_b200.synth import static_pose
    st = SpatialStore(cube_size=0.03)
    pose = static_pose((0.1, -0.2, 0.05), (0.3, 0.1, 1.0))
    coords = np.random.default_rng(1).integers(-6, 7, size=(600, 3))
    dev = block_in_frustum_device(st, coords, pose, _intr())
    host = np.array([block_in_frustum(tuple(c), pose, _intr(), 0.24) for c in coords])
    assert np.array_equal(dev, host)
    from paper_1803_03949_b200 import Pose
    assert block_in_frustum_device(st, [(0, 0, 0), (0, 0, -50), (0, 0, 4)], Pose.identity(),
                                   _intr()).tolist() == [True, False, True]


# ---------------------------------------------------------------- store (test_store.py)
def test_capacity_error_block_table():                 # test_store.py:102-107
    from paper_1803_03949_b200 import CapacityError, SpatialStore
    st = SpatialStore(cube_size=0.03, table_size=8)
    st.set_block_samples([(i, 0, 0) for i in range(4)])
    assert st.block_count == 4
    with pytest.raises(CapacityError):
        st.set_block_samples([(9, 9, 9)])


def test_capacity_error_vertex_pool():                 # store.py:150-152
    from paper_1803_03949_b200 import CapacityError, Engine, RunConfig
    from paper_1803_03949_b200.synth import SceneSpec, static_pose, render_depth
    spec = SceneSpec(scene="plane", width=48, height=48, fx=40.0, fy=40.0)
    pose = static_pose((0, 0, 0), (0, 0, 1))
    eng = Engine(RunConfig(cube_size=0.02, max_vertices=50), spec.intrinsics())
    with pytest.raises(CapacityError):
        eng.fuse_frame(render_depth(spec, pose), pose)


def test_capacity_error_vertex_pool_pipelined():       # store.py:150-152, pipelined submission
    """The failing frame's error surfaces at the next call; the frame queued
    behind it is dropped (its kernels stop at the guard) and raises nothing twice."""
    from paper_1803_03949_b200 import CapacityError, Engine, RunConfig
    from paper_1803_03949_b200.synth import SceneSpec, static_pose, render_depth
    spec = SceneSpec(scene="plane", width=48, height=48, fx=40.0, fy=40.0)
    pose = static_pose((0, 0, 0), (0, 0, 1))
    depth = render_depth(spec, pose)
    eng = Engine(RunConfig(cube_size=0.02, max_vertices=50), spec.intrinsics(), pipelined=True)
    eng.fuse_frame(depth, pose)                        # queued; fails on the device
    with pytest.raises(CapacityError):
        eng.fuse_frame(depth, pose)                    # queues frame 1, settles frame 0
    assert eng._pending is None                        # frame 1 was dropped, not left in flight
    from paper_1803_03949_b200 import _lib
    import ctypes as C
    st = _lib.Stats()
    assert _lib.load().vm_fuse_frame_result(eng.store._h, C.byref(st)) != 0   # nothing submitted


def test_hash_table_heavy_load_no_dropped_inserts():   # test_store.py:40-57 (load 50%)
    from paper_1803_03949_b200 import SpatialStore
    st = SpatialStore(cube_size=0.03, table_size=1 << 14)
    rng = np.random.default_rng(3)
    coords = {tuple(int(v) for v in r) for r in rng.integers(-200, 200, size=(20000, 3))}
    coords = sorted(coords)[: (1 << 13) - 1]
    st.set_block_samples(coords)
    st.set_block_samples(coords)                       # idempotent
    assert st.block_count == len(coords)
    assert st.contains(coords).all()
    assert not st.contains([(999, 999, 999)]).any()
    assert set(st.block_coords()) == set(coords)


# ---------------------------------------------------------------- mesher (test_mesher.py)
def _store_with_field(fn, blocks=((0, 0, 0),), l=0.03):
    from paper_1803_03949_b200 import SpatialStore
    st = SpatialStore(cube_size=l)
    grid = np.stack(np.meshgrid(*[np.arange(B)] * 3, indexing="ij"), axis=-1).reshape(-1, 3)
    tsdf = [fn((np.asarray(c) * B + grid) * l).reshape(8, 8, 8) for c in blocks]
    st.set_block_samples(list(blocks), np.stack(tsdf), np.ones((len(blocks), 8, 8, 8), np.int32))
    return st


ALL8 = [(x, y, z) for x in (0, 1) for y in (0, 1) for z in (0, 1)]


def _plane_store(l=0.03):
    return _store_with_field(lambda p: (p[:, 2] - 3.5 * l) / (3 * l), ALL8, l)


def test_type_kats():                                   # test_mesher.py:81-111
    from paper_1803_03949_b200.mesher import extract_frame
    st = _store_with_field(lambda p: np.full(len(p), 0.5), ALL8)
    extract_frame(st, [((0, 0, 0), None)], 0)
    assert st.get_block((0, 0, 0)).type_curr[3, 3, 3] == 0
    st = _store_with_field(lambda p: np.full(len(p), -0.5))
    extract_frame(st, [((0, 0, 0), None)], 0)
    assert st.get_block((0, 0, 0)).type_curr[2, 2, 2] == 255
    st = _plane_store()
    extract_frame(st, [((0, 0, 0), None)], 0)
    assert st.get_block((0, 0, 0)).type_curr[3, 3, 3] == 0x0F


def test_adjacent_cubes_share_edge_vertex():           # test_mesher.py:174-182
    from paper_1803_03949_b200.mesher import extract_frame
    st = _plane_store()
    mask = np.zeros((B,) * 3, dtype=bool)
    mask[2, 2, 3] = True
    mask[3, 2, 3] = True
    extract_frame(st, [((0, 0, 0), mask)], 0, halo=[])
    assert st.vertices.allocation_events == 6


def test_replacement_is_lazy_and_strategies_agree():    # test_mesher.py:185-209
    from paper_1803_03949_b200.mesher import extract_frame
    counts = {}
    for strategy in ("serial", "claim", "partition"):
        st = _plane_store()
        scope = [(c, None) for c in st.block_coords()]
        extract_frame(st, scope, 0, strategy=strategy)
        ev = st.vertices.allocation_events
        extract_frame(st, scope, 1, strategy=strategy)
        assert st.vertices.allocation_events == ev
        counts[strategy] = (ev, st.vertices.live_count)
    assert len(set(counts.values())) == 1


def test_triangulation_refcounts_match_tally():        # test_mesher.py:221-296
    from paper_1803_03949_b200 import Engine
    from paper_1803_03949_b200.mesher import extract_frame
    st = _plane_store()
    extract_frame(st, [(c, None) for c in st.block_coords()], 0)
    vp, tp = st.vertices, st.triangles
    tally = np.zeros(vp.count, np.int64)
    for blk in st.blocks():
        th = blk.triangles.reshape(-1)
        th = th[th >= 0]
        tally += np.bincount(tp.vertices[th].reshape(-1), minlength=vp.count)
    assert np.array_equal(tally, vp.refcount)
    blk = st.get_block((0, 0, 0))
    assert (blk.triangles[2, 2, 3, :2] >= 0).all() and (blk.triangles[2, 2, 3, 2:] == -1).all()


def test_gc_untouched_frees_nothing():                 # test_mesher.py:309-313
    from paper_1803_03949_b200.mesher import extract_frame, garbage_collect
    st = _plane_store()
    extract_frame(st, [(c, None) for c in st.block_coords()], 0)
    assert garbage_collect(st, st.block_coords()) == 0


def test_degenerate_gradient_falls_back_to_face_normal():   # test_mesher.py:368-385
    from paper_1803_03949_b200.mc_tables import CORNER_OFFSETS
    from paper_1803_03949_b200.mesher import extract_frame
    l = 0.03
    grid = np.stack(np.meshgrid(*[np.arange(B)] * 3, indexing="ij"), axis=-1).reshape(-1, 3)
    tsdf = ((grid * l)[:, 2] - 3.5 * l) / (3 * l)
    keep = np.zeros((B,) * 3, dtype=bool)
    for off in CORNER_OFFSETS:
        keep[3 + off[0], 3 + off[1], 3 + off[2]] = True
    from paper_1803_03949_b200 import SpatialStore
    st = SpatialStore(cube_size=l)
    st.set_block_samples([(0, 0, 0)], tsdf.reshape(1, 8, 8, 8), keep.astype(np.int32)[None])
    extract_frame(st, [((0, 0, 0), None)], 0)
    blk = st.get_block((0, 0, 0))
    hs = blk.edge_vertex[blk.edge_vertex >= 0]
    assert hs.size > 0
    nrm = st.vertices.normal
    for h in hs:
        assert np.linalg.norm(nrm[h]) == pytest.approx(1.0)
        assert nrm[h][2] > 0.9


def test_single_isolated_triangle():                    # test_mesher.py:396-410
    from paper_1803_03949_b200 import SpatialStore
    from paper_1803_03949_b200.mc_tables import CORNER_OFFSETS
    from paper_1803_03949_b200.mesher import extract_frame
    tsdf = np.zeros((8, 8, 8))
    w = np.zeros((8, 8, 8), np.int32)
    for k, off in enumerate(CORNER_OFFSETS):
        loc = (3 + off[0], 3 + off[1], 3 + off[2])
        tsdf[loc] = -0.5 if k == 0 else 0.5
        w[loc] = 1
    st = SpatialStore(cube_size=0.03)
    st.set_block_samples([(0, 0, 0)], tsdf[None], w[None])
    extract_frame(st, [((0, 0, 0), None)], 0)
    assert st.triangles.live_count == 1 and st.vertices.live_count == 3


def test_extract_empty_scope_noop():                   # test_mesher.py:481-484
    from paper_1803_03949_b200 import SpatialStore
    from paper_1803_03949_b200.mesher import extract_frame
    assert extract_frame(SpatialStore(cube_size=0.03), [], 0) == {"refined": 0, "freed": 0}


def test_watertight_euler_on_analytic_sphere():        # test_mesher.py:494-518
    from paper_1803_03949_b200 import SpatialStore
    from paper_1803_03949_b200.mesher import extract_frame
    r, l = 0.25, 0.025
    ext = l * B
    n = int(np.ceil((r + 6 * l) / ext)) + 1
    grid = np.stack(np.meshgrid(*[np.arange(B)] * 3, indexing="ij"), axis=-1).reshape(-1, 3)
    coords, fields = [], []
    for bx in range(-n, n + 1):
        for by in range(-n, n + 1):
            for bz in range(-n, n + 1):
                ctr = (np.array([bx, by, bz]) + 0.5) * ext
                if abs(np.linalg.norm(ctr) - r) < ext * 1.4:
                    pts = (np.array([bx, by, bz]) * B + grid) * l
                    coords.append((bx, by, bz))
                    fields.append(np.clip((np.linalg.norm(pts, axis=1) - r) / (3 * l), -1, 1))
    st = SpatialStore(cube_size=l)
    st.set_block_samples(coords, np.stack(fields), np.ones((len(coords), 8, 8, 8), np.int32))
    extract_frame(st, [(c, None) for c in st.block_coords()], 0)
    mesh = st.compact_mesh()
    counts = edge_use_counts(mesh.indices)
    assert all(v == 2 for v in counts.values())
    assert len(mesh.positions) - len(counts) + len(mesh.indices) == 2


# ---------------------------------------------------------------- refine
def test_refine_kernel_exhaustive_eq3_5():              # test_acceptance.py:327-373
    import ctypes as C
    from paper_1803_03949_b200 import SpatialStore, _lib
    from paper_1803_03949_b200.refine import RefineParams, detect_disturbance
    from refine_cases import refine_cases
    cases = list(refine_cases())
    tc = np.array([c[0] for c in cases], np.uint8)
    tp = np.array([c[1] for c in cases], np.uint8)
    corners = np.ascontiguousarray(np.stack([c[2] for c in cases]).astype(np.float64))
    out = np.zeros(len(cases), np.int32)
    st = SpatialStore(cube_size=0.03)
    _lib.check(_lib.load().vm_refine_eval(st._h, _lib.ptr(tc), _lib.ptr(tp), _lib.ptr(corners),
                                          len(cases), 0.1, _lib.ptr(out)))
    want = [detect_disturbance(a, b, c, RefineParams(0.1)) for a, b, c in cases]
    got = [None if v < 0 else int(v) for v in out]
    assert got == want and len(cases) == 12680


# ---------------------------------------------------------------- acceptance
def _wall(width=96, fx=75.0, offset=-1.0):
    from paper_1803_03949_b200.synth import SceneSpec
    return SceneSpec(scene="plane", plane_normal=(0, 0, -1), plane_offset=offset, width=width,
                     height=width, fx=fx, fy=fx)


def test_wall_normals_and_temporal_stability():         # test_mesher.py:338-346, :413-427; criterion 8
    from paper_1803_03949_b200 import Engine, RunConfig
    from paper_1803_03949_b200.synth import render_depth, static_pose
    spec = _wall()
    pose = static_pose((0.0, 0.0, 0.0), (0.0, 0.0, 1.0))
    depth = render_depth(spec, pose)
    eng = Engine(RunConfig(cube_size=0.02), spec.intrinsics(), audit_every_frame=True)
    eng.fuse_frame(depth, pose)
    m1 = eng.compact()
    ev, tc = eng.store.vertices.allocation_events, eng.store.triangles.count
    eng.fuse_frame(depth, pose)
    m2 = eng.compact()
    assert eng.store.vertices.allocation_events == ev and eng.store.triangles.count == tc
    assert np.array_equal(m1.positions, m2.positions) and np.array_equal(m1.normals, m2.normals)
    assert np.array_equal(m1.indices, m2.indices)
    eng.fuse_frame(depth, pose)
    mesh = eng.compact()
    ang = np.degrees(np.arccos(np.clip(-mesh.normals[:, 2], -1, 1)))
    assert ang.max() <= 2.0
    assert np.allclose(np.linalg.norm(mesh.normals, axis=1), 1.0)


def test_criterion_4_memory_reduction():                # test_acceptance.py:153-177
    from paper_1803_03949_b200 import Engine, RunConfig
    from paper_1803_03949_b200.synth import render_depth, static_pose
    l = 0.02
    spec = _wall(width=116)
    pose = static_pose((0, 0, 0), (0, 0, 1))
    depth = render_depth(spec, pose)
    eng = Engine(RunConfig(cube_size=l), spec.intrinsics(), audit_every_frame=True)
    for _ in range(3):
        row = eng.fuse_frame(depth, pose)
    mesh = eng.compact()
    cols_x = np.unique(np.floor(mesh.positions[:, 0] / l).astype(int))
    assert len(cols_x) >= 64
    assert row.vertices_live / (3 * row.triangles_live) <= 0.25
    assert abs(row.triangles_live / row.vertices_live - 1.939) <= 0.1


def test_criterion_5_watertight_orbit():                # test_acceptance.py:180-188
    from paper_1803_03949_b200 import Engine, RunConfig
    from paper_1803_03949_b200.synth import SceneSpec, camera_pose, render_depth
    spec = SceneSpec(scene="sphere", sphere_radius=0.3, orbit_radius=0.9, elevation_amp_deg=60.0,
                     angular_step_deg=6.0, frames=60, width=128, height=96, fx=110.0, fy=110.0)
    eng = Engine(RunConfig(cube_size=0.02), spec.intrinsics(), audit_every_frame=True)
    for i in range(spec.frames):
        p = camera_pose(spec, i)
        eng.fuse_frame(render_depth(spec, p), p)
    mesh = eng.compact()
    counts = edge_use_counts(mesh.indices)
    assert sum(1 for v in counts.values() if v != 2) == 0
    assert len(mesh.positions) - len(counts) + len(mesh.indices) == 2


def test_criterion_6_garbage_collection():              # test_acceptance.py:191-238
    from paper_1803_03949_b200 import Engine, RunConfig
    from paper_1803_03949_b200.synth import render_depth, static_pose
    l = 0.02
    cfg = RunConfig(cube_size=l, weight_cap=8)
    wall, receded = _wall(), _wall(offset=-(1.0 + 1.5 * l))
    pose = static_pose((0, 0, 0), (0, 0, 1))
    d_wall, d_empty = render_depth(wall, pose), render_depth(receded, pose)
    eng = Engine(cfg, wall.intrinsics(), audit_every_frame=True)
    eng.fuse_frame(d_wall, pose)
    zcut = 1.0 + l

    def region_live():
        n = 0
        pos = eng.store.vertices.position
        for blk in eng.store.blocks():
            occ = blk.edge_vertex.reshape(-1)
            occ = occ[occ >= 0]
            n += int((pos[occ][:, 2] < zcut).sum())
        return n

    before = region_live()
    pool = eng.store.vertices
    live0, ev0, rec0 = pool.live_count, pool.allocation_events, pool.recycled_total
    for _ in range(cfg.weight_cap):
        eng.fuse_frame(d_empty, pose)
    after = region_live()
    pool = eng.store.vertices
    freed = live0 + pool.allocation_events - ev0 - pool.live_count
    arena = pool.count
    assert before > 1000 and after == 0 and pool.recycled_total - rec0 == freed
    for _ in range(cfg.weight_cap + 2):
        eng.fuse_frame(d_wall, pose)
    assert eng.store.vertices.count == arena and region_live() > 0


def test_criterion_7_refinement_efficacy():             # test_acceptance.py:241-265
    from paper_1803_03949_b200 import Engine, RunConfig
    from paper_1803_03949_b200.synth import render_depth, static_pose, tilted_plane_spec
    l = 0.02
    spec = tilted_plane_spec(8.0, distance=1.0, width=128, height=96)
    spec.fx = spec.fy = 90.0
    pose = static_pose((0.0, 0.0, 0.0), (0.0, 0.0, 1.0))
    depth = render_depth(spec, pose)
    n = np.asarray(spec.plane_normal) / np.linalg.norm(spec.plane_normal)
    out = {}
    for refine in (False, True):
        eng = Engine(RunConfig(cube_size=l, refine=refine), spec.intrinsics(), audit_every_frame=True)
        for _ in range(8):
            row = eng.fuse_frame(depth, pose)
        assert row.irregular_cube_count == eng.irregular_cube_count()
        mesh = eng.compact()
        out[refine] = (row.irregular_cube_count,
                       float(np.sqrt(((mesh.positions @ n - spec.plane_offset) ** 2).mean())))
    assert out[True][0] <= 0.5 * out[False][0]
    assert out[False][1] <= 0.5 * l and out[True][1] <= 0.5 * l


def test_blank_frame_is_noop():                         # test_mesher.py:481-491
    from paper_1803_03949_b200 import Engine, RunConfig
    from paper_1803_03949_b200.synth import render_depth, static_pose
    spec = _wall()
    pose = static_pose((0.0, 0.0, 0.0), (0.0, 0.0, 1.0))
    depth = render_depth(spec, pose)
    eng = Engine(RunConfig(cube_size=0.02), spec.intrinsics(), audit_every_frame=True)
    first = eng.fuse_frame(depth, pose)
    row = eng.fuse_frame(np.zeros_like(depth), pose)
    assert (row.blocks_active, row.vertices_live, row.triangles_live, row.vertices_allocated_total) == \
        (first.blocks_active, first.vertices_live, first.triangles_live, first.vertices_allocated_total)


def test_device_resident_depth_matches_host_depth():
    import torch
    from paper_1803_03949_b200 import Engine, RunConfig
    from paper_1803_03949_b200.synth import SceneSpec, camera_pose, render_depth
    spec = SceneSpec(scene="sphere", sphere_radius=0.3, orbit_radius=0.9, elevation_amp_deg=60.0,
                     angular_step_deg=18.0, frames=4, width=96, height=72, fx=80.0, fy=80.0)
    e1 = Engine(RunConfig(cube_size=0.025), spec.intrinsics())
    e2 = Engine(RunConfig(cube_size=0.025), spec.intrinsics())
    for i in range(4):
        p = camera_pose(spec, i)
        d = render_depth(spec, p)
        e1.fuse_frame(d, p)
        e2.fuse_frame(torch.tensor(d, device="cuda"), p)
    m1, m2 = e1.compact(), e2.compact()
    assert np.array_equal(m1.positions, m2.positions) and np.array_equal(m1.indices, m2.indices)


def test_store_usable_after_block_table_capacity_error():   # store.py:296-320, 304-306
    """A frame that fills the block table raises CapacityError; the device
    flag is then cleared and the partially updated store stays usable as the
    reference's does: the block count is the reference's (table_size / 2,
    allocation stopped at 2n >= table_size), the blocks it allocated are empty
    ones, compaction / audit / snapshots work, and a later frame that needs a
    new block raises again."""
    from oracle.oracle import OracleCapacityError, OracleEngine
    from paper_1803_03949_b200 import CapacityError, Engine, RunConfig
    from paper_1803_03949_b200.synth import SceneSpec, camera_pose, render_depth
    spec = SceneSpec(scene="sphere", sphere_radius=0.3, orbit_radius=0.9, elevation_amp_deg=60.0,
                     angular_step_deg=18.0, frames=3, width=64, height=48, fx=55.0, fy=55.0)
    intr = spec.intrinsics()
    cfg = dict(cube_size=0.025, table_size=48)          # frame 0 needs 32 blocks, the table holds 24
    eng = Engine(RunConfig(**cfg), intr)
    ora = OracleEngine(cfg, (intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height))
    pose = camera_pose(spec, 0)
    d = render_depth(spec, pose)
    with pytest.raises(CapacityError):
        eng.fuse_frame(d, pose)
    with pytest.raises(OracleCapacityError):
        ora.fuse_frame(d, pose.rotation, pose.translation)
    assert eng.store.block_count == ora.store.block_count() == 24
    m = eng.compact()                                  # no stale error re-raised
    assert len(m.indices) == 0 and len(m.positions) == 0
    assert eng.audit().ok
    snap = eng.store.snapshot_arrays()
    assert (snap["weight"] == 0).all() and (snap["tsdf"] == 0).all()
    with pytest.raises(CapacityError):                # a block of frame 0 it could not allocate
        eng.fuse_frame(d, pose)
    with pytest.raises(OracleCapacityError):
        ora.fuse_frame(d, pose.rotation, pose.translation)
    assert eng.store.block_count == ora.store.block_count() == 24


def test_pipelined_engine_continues_after_capacity_error():
    """After a pipelined frame's CapacityError the engine is not wedged: the
    dropped frame can be submitted again and compaction works."""
    from paper_1803_03949_b200 import CapacityError, Engine, RunConfig
    from paper_1803_03949_b200.synth import SceneSpec, static_pose, render_depth
    spec = SceneSpec(scene="plane", width=48, height=48, fx=40.0, fy=40.0)
    pose = static_pose((0, 0, 0), (0, 0, 1))
    depth = render_depth(spec, pose)
    eng = Engine(RunConfig(cube_size=0.02, max_vertices=50), spec.intrinsics(), pipelined=True)
    eng.fuse_frame(depth, pose)
    with pytest.raises(CapacityError):
        eng.fuse_frame(depth, pose)
    eng.compact()                                      # the partial store can be read
    # the pool stays over its limit (the failing frame's vertices were placed),
    # so every later frame reports CapacityError again -- never the wedge
    # "previous frame's result was not taken"
    for _ in range(2):
        eng.fuse_frame(np.zeros_like(depth), pose)
        with pytest.raises(CapacityError):
            eng.fuse_frame(np.zeros_like(depth), pose)
        assert eng._pending is None


def test_pipelined_empty_depth_keeps_pending_frame():
    """An argument error (empty depth) queues nothing: the frame in flight
    keeps its row and later submissions proceed (the engine is not wedged)."""
    from paper_1803_03949_b200 import Engine, InputError, RunConfig
    from paper_1803_03949_b200.synth import SceneSpec, static_pose, render_depth
    spec = SceneSpec(scene="plane", width=48, height=48, fx=40.0, fy=40.0)
    pose = static_pose((0, 0, 0), (0, 0, 1))
    depth = render_depth(spec, pose)
    a = Engine(RunConfig(cube_size=0.02), spec.intrinsics(), pipelined=True)
    b = Engine(RunConfig(cube_size=0.02), spec.intrinsics())
    r0 = a.fuse_frame(depth, pose)
    with pytest.raises(InputError):
        a.fuse_frame(np.zeros((0, 48)), pose)
    r1 = a.fuse_frame(depth, pose)
    s0, s1 = b.fuse_frame(depth, pose), b.fuse_frame(depth, pose)
    assert (r0.vertices_live, r1.vertices_live) == (s0.vertices_live, s1.vertices_live)
    assert r1.frame == 1


def test_device_depth_from_another_stream_is_ordered():
    """A CUDA depth tensor produced on a side stream (torch's current stream
    at the call) is ordered before the engine's kernels and kept alive for
    them (record_stream): rows equal the host-input engine's."""
    import torch
    from paper_1803_03949_b200 import Engine, RunConfig
    from paper_1803_03949_b200.synth import SceneSpec, camera_pose, render_depth
    spec = SceneSpec(scene="sphere", sphere_radius=0.3, orbit_radius=0.9, elevation_amp_deg=60.0,
                     angular_step_deg=18.0, frames=4, width=96, height=72, fx=80.0, fy=80.0)
    intr = spec.intrinsics()
    a = Engine(RunConfig(cube_size=0.025), intr, pipelined=True)
    b = Engine(RunConfig(cube_size=0.025), intr)
    side = torch.cuda.Stream()
    rows = []
    for i in range(spec.frames):
        pose = camera_pose(spec, i)
        d = render_depth(spec, pose)
        with torch.cuda.stream(side):
            big = torch.randn(4096, 4096, device="cuda")
            for _ in range(4):
                big = big @ big.T / 4096.0          # keep the side stream busy
            dev = torch.from_numpy(d).to("cuda") + big[0, 0].clamp(-1.0, 1.0) * 0.0
            rows.append(a.fuse_frame(dev, pose))
            del dev                                     # freed while the frame may still read it
        b.fuse_frame(d, pose)
    for ra, rb in zip(rows, b.stats):
        assert (ra.blocks_active, ra.vertices_live, ra.triangles_live) == \
               (rb.blocks_active, rb.vertices_live, rb.triangles_live)
