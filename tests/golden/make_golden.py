"""Generate golden fixtures by running the REFERENCE ``voxmesh`` itself.

Run in the builder container only (needs /root/reference):

    python tests/golden/make_golden.py [/root/reference/pkg/src]

For each scene it stores (npz, compressed): the f64 depth frames and poses fed
in, the reference's per-frame StatsRow non-timing columns, and the final state:
sorted block coordinates with tsdf/weight/type_prev/type_curr/edge_vertex/
triangles, the vertex pool (position/normal/refcount/birth/alive), the compact
mesh (engine.py:178 -> store.py:388-425) and the audit report.  The oracle
(tests/test_oracle_golden.py) and, through the oracle, the CUDA path are pinned
to these.  Scenes follow the reference's own test fixtures
(pkg/tests/conftest.py, test_acceptance.py, test_mesher.py) at small sizes.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent


def _ref(src):
    sys.path.insert(0, src)
    import voxmesh  # noqa: F401
    from voxmesh import Engine, RunConfig, SpatialStore  # noqa: F401
    from voxmesh import synth
    from voxmesh.mesher import extract_frame  # noqa: F401
    return sys.modules["voxmesh"], synth


def engine_scene(vm, name, spec_frames, cfg_kw, intr):
    """spec_frames: list of (depth, pose)."""
    cfg = vm.RunConfig(strategy="serial", workers=1, **cfg_kw)
    eng = vm.Engine(cfg, intr, audit_every_frame=True)
    stats = []
    for depth, pose in spec_frames:
        row = eng.fuse_frame(depth, pose)
        stats.append([row.frame, row.blocks_active, row.vertices_live, row.triangles_live,
                      row.vertices_allocated_total, row.vertices_recycled_total,
                      row.irregular_cube_count])
    out = dict(kind="engine", name=name)
    out["depth"] = np.stack([d for d, _ in spec_frames]).astype(np.float64)
    out["rot"] = np.stack([p.rotation for _, p in spec_frames])
    out["trans"] = np.stack([p.translation for _, p in spec_frames])
    out["intr6"] = np.array([intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height])
    c = eng.config
    out["cfg"] = np.array([c.cube_size, c.trunc, c.epsilon, float(c.refine), c.max_range,
                           float(c.frustum_only), float(c.weight_cap), float(c.table_size)])
    out["stats"] = np.array(stats, np.int64)
    out["last_collected"] = np.array(eng.last_collected, np.int32).reshape(-1, 3)
    dump_state(eng.store, out, eng.frame_index)
    rep = eng.audit()
    out["audit"] = np.array([rep.vertices_live, rep.triangles_live, rep.refcount_mismatches,
                             rep.duplicate_handles, rep.zero_ref_live, int(rep.conservation_ok)])
    return out


def dump_state(store, out, frame):
    blocks = list(store.blocks())
    out["coords"] = np.array([b.coord for b in blocks], np.int32).reshape(-1, 3)
    for k in ("tsdf", "weight", "type_prev", "type_curr", "edge_vertex", "triangles"):
        arr = [getattr(b, k) for b in blocks]
        out[k] = np.stack(arr) if arr else np.zeros((0,), np.int32)
    vp = store.vertices
    n = vp.count
    out["v_position"] = vp.position[:n].copy()
    out["v_normal"] = vp.normal[:n].copy()
    out["v_refcount"] = vp.refcount[:n].copy()
    out["v_birth"] = vp.birth_frame[:n].copy()
    out["v_alive"] = vp.alive[:n].copy()
    out["counters"] = np.array([store.block_count, store.block_allocations, vp.count,
                                len(vp.free), vp.recycled_total, vp.allocation_events,
                                store.triangles.count, len(store.triangles.free),
                                store.triangles.recycled_total], np.int64)
    m = store.compact_mesh(frame)
    out["m_positions"], out["m_normals"] = m.positions, m.normals
    out["m_ages"], out["m_indices"] = m.ages, m.indices


def random_field_scene(vm, seed, refine, scale=1.0):
    """test_mesher.py:436-478 style: random corner field over 8 blocks, partial
    observation, one extract_frame over the full scope (serial)."""
    from voxmesh.mesher import extract_frame
    from voxmesh.refine import RefineParams
    B = 8
    l = 0.03
    rng = np.random.default_rng(seed)
    store = vm.SpatialStore(cube_size=l)
    blocks = [(x, y, z) for x in (0, 1) for y in (0, 1) for z in (0, 1)]
    tsdf, weight = [], []
    for coord in blocks:
        blk = store.get_or_allocate_block(coord)
        blk.tsdf.reshape(-1)[:] = rng.normal(size=512) * scale
        blk.weight[:] = 1
        mask = np.random.default_rng(seed + 1).random((B, B, B)) < 0.85
        blk.weight[~mask] = 0
        tsdf.append(blk.tsdf.copy())
        weight.append(blk.weight.copy())
    scope = [(c, None) for c in store.block_coords()]
    # two frames: a second, perturbed field exercises re-typing / retriangulation / GC
    rp = RefineParams(epsilon=0.1, enabled=refine)
    r1 = extract_frame(store, scope, 0, strategy="serial", refine_params=rp,
                       halo=store.block_coords())
    tsdf2 = []
    for coord in blocks:
        blk = store.get_block(coord)
        blk.tsdf.reshape(-1)[:] += rng.normal(size=512) * 0.05 * scale
        tsdf2.append(blk.tsdf.copy())
    r2 = extract_frame(store, scope, 1, strategy="serial", refine_params=rp,
                       halo=store.block_coords())
    out = dict(kind="fields", name=f"fields_s{seed}_r{int(refine)}")
    out["in_coords"] = np.array(blocks, np.int32)
    out["in_tsdf"] = np.stack(tsdf)
    out["in_tsdf2"] = np.stack(tsdf2)
    out["in_weight"] = np.stack(weight)
    out["cfg"] = np.array([l, 0.0, 0.1, float(refine), 0, 0, 0, float(1 << 20)])
    out["extract_out"] = np.array([r1["refined"], r1["freed"], r2["refined"], r2["freed"]], np.int64)
    dump_state(store, out, 2)
    return out


def main(src="/root/reference/pkg/src"):
    vm, synth = _ref(src)
    SceneSpec, camera_pose, render_depth = synth.SceneSpec, synth.camera_pose, synth.render_depth
    static_pose, tilted_plane_spec = synth.static_pose, synth.tilted_plane_spec
    scenes = []

    # 1. wall (conftest.py:12-30)
    spec = SceneSpec(scene="plane", plane_normal=(0, 0, -1), plane_offset=-1.0,
                     width=64, height=64, fx=50.0, fy=50.0)
    pose = static_pose((0.0, 0.0, 0.0), (0.0, 0.0, 1.0))
    d = render_depth(spec, pose)
    scenes.append(engine_scene(vm, "wall", [(d, pose)] * 3, dict(cube_size=0.02),
                               spec.intrinsics()))

    # 2. sphere orbit (conftest.py:33-44, smaller)
    spec = SceneSpec(scene="sphere", sphere_radius=0.3, orbit_radius=0.9,
                     elevation_amp_deg=60.0, angular_step_deg=18.0, frames=6,
                     width=64, height=48, fx=55.0, fy=55.0)
    fr = [(render_depth(spec, camera_pose(spec, i)), camera_pose(spec, i)) for i in range(6)]
    scenes.append(engine_scene(vm, "sphere_orbit", fr, dict(cube_size=0.025), spec.intrinsics()))

    # 3. tilted plane with refinement (test_acceptance.py:241-265, smaller)
    spec = tilted_plane_spec(8.0, distance=1.0, width=64, height=48)
    spec.fx = spec.fy = 60.0
    pose = static_pose((0.0, 0.0, 0.0), (0.0, 0.0, 1.0))
    d = render_depth(spec, pose)
    scenes.append(engine_scene(vm, "tilted_refine", [(d, pose)] * 4,
                               dict(cube_size=0.02, refine=True), spec.intrinsics()))

    # 4. noisy box room with refinement (test_acceptance.py:56-62 room, + noise)
    spec = SceneSpec(scene="room", room_size=(2.0, 2.0, 1.4), orbit_radius=0.3,
                     look="outward", elevation_amp_deg=30.0, angular_step_deg=36.0,
                     frames=5, width=64, height=48, fx=45.0, fy=45.0,
                     noise_sigma=0.002, seed=3)
    rng = np.random.default_rng(3)
    fr = [(render_depth(spec, camera_pose(spec, i), rng), camera_pose(spec, i)) for i in range(5)]
    scenes.append(engine_scene(vm, "room_noise_refine", fr,
                               dict(cube_size=0.025, refine=True, epsilon=0.15),
                               spec.intrinsics()))

    # 5. frustum-only scope filter (engine.py:135-138) + max_range clipping
    spec = SceneSpec(scene="room", room_size=(2.0, 2.0, 1.4), orbit_radius=0.3,
                     look="outward", elevation_amp_deg=30.0, angular_step_deg=36.0,
                     frames=4, width=64, height=48, fx=45.0, fy=45.0)
    fr = [(render_depth(spec, camera_pose(spec, i)), camera_pose(spec, i)) for i in range(4)]
    scenes.append(engine_scene(vm, "room_frustum", fr,
                               dict(cube_size=0.025, frustum_only=True, max_range=1.3),
                               spec.intrinsics()))

    # 6. GC carve / refuse (test_acceptance.py:191-238, smaller)
    l = 0.02
    wall = SceneSpec(scene="plane", plane_normal=(0, 0, -1), plane_offset=-1.0,
                     width=48, height=48, fx=40.0, fy=40.0)
    rec = SceneSpec(scene="plane", plane_normal=(0, 0, -1), plane_offset=-(1.0 + 1.5 * l),
                    width=48, height=48, fx=40.0, fy=40.0)
    pose = static_pose((0, 0, 0), (0, 0, 1))
    dw, de = render_depth(wall, pose), render_depth(rec, pose)
    fr = [(dw, pose)] + [(de, pose)] * 4 + [(dw, pose)] * 6 + [(np.zeros_like(dw), pose)]
    scenes.append(engine_scene(vm, "gc_carve", fr, dict(cube_size=l, weight_cap=4),
                               wall.intrinsics()))

    # 7. sphere+box composite (SURVEY.md 8d C1 scene, reduced)
    orig = synth.scene_sdf

    def sdf(spec_, pts):
        pts = np.asarray(pts, dtype=np.float64)
        room = (np.array([1.5, 1.5, 1.0]) - np.abs(pts)).min(axis=-1)
        sph = np.linalg.norm(pts - np.array([0.9, 0.0, -0.4]), axis=-1) - 0.4
        q = np.abs(pts - np.array([-0.8, 0.5, -0.6])) - 0.25
        box = (np.linalg.norm(np.maximum(q, 0.0), axis=-1)
               + np.minimum(np.max(q, axis=-1), 0.0))
        return np.minimum(room, np.minimum(sph, box))
    synth.scene_sdf = sdf
    try:
        spec = SceneSpec(scene="room", orbit_radius=0.3, look="outward",
                         elevation_amp_deg=20.0, elevation_rings=3, angular_step_deg=9.0,
                         frames=3, width=80, height=60, fx=65.625, fy=65.625)
        fr = [(render_depth(spec, camera_pose(spec, i)), camera_pose(spec, i)) for i in range(3)]
    finally:
        synth.scene_sdf = orig
    scenes.append(engine_scene(vm, "sphere_box", fr, dict(cube_size=0.016), spec.intrinsics()))

    # 8. random fields through extract_frame (all cube types)
    scenes.append(random_field_scene(vm, 0, False))
    scenes.append(random_field_scene(vm, 7, True, scale=0.12))

    total = 0
    for sc in scenes:
        path = HERE / f"{sc['name']}.npz"
        arrays = {k: v for k, v in sc.items() if k not in ("kind", "name")}
        arrays["kind"] = np.array(sc["kind"])
        np.savez_compressed(path, **arrays)
        total += path.stat().st_size
        print(f"{path.name}: {path.stat().st_size / 1e3:.0f} kB")
    print(f"total {total / 1e6:.2f} MB")


if __name__ == "__main__":
    main(*sys.argv[1:])
