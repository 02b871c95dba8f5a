"""Opt-in block GC (north star item 5; csrc/vm_kernels.cuh k_block_gc).

The reference never evicts a block (store.py:14), so parity mode keeps block
GC off.  With ``RunConfig.block_gc_age = K`` a block not collected for K
frames that holds no vertex and no observed sample is evicted: its index goes
to a free list that allocations pop first, its hash entry keeps the key
(value "evicted"), its neighbours' rows are unlinked.  Such a block is read by
meshing exactly like an absent one, so everything but ``blocks_active`` stays
identical -- rows, mesh, normals -- and a re-observed key is allocated again.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rows(eng):
    return [(r.vertices_live, r.triangles_live, r.vertices_allocated_total, r.vertices_recycled_total,
             r.irregular_cube_count) for r in eng.stats]


@pytest.mark.parametrize("config,nframes", [("C2", 90), ("C5", 150)])
def test_block_gc_evicts_and_reallocates_with_identical_mesh(config, nframes):
    import torch
    from paper_1803_03949_b200 import Engine, RunConfig
    from paper_1803_03949_b200.synth import camera_pose, config_spec, multiroom_pose, render_depth_torch
    spec, cfg = config_spec(config)
    spec.width, spec.height, spec.fx, spec.fy = 320, 240, 262.5, 262.5
    pose_fn = multiroom_pose if config == "C5" else camera_pose
    intr = spec.intrinsics()
    a = Engine(RunConfig(**cfg), intr)
    b = Engine(RunConfig(block_gc_age=8, **cfg), intr, pipelined=True)
    # forward, then back over the first frames (re-observation of evicted keys)
    order = list(range(nframes)) + list(range(24))
    for i in order:
        p = pose_fn(spec, i)
        d = render_depth_torch(spec, p)
        a.fuse_frame(d, p)
        b.fuse_frame(d, p)
    torch.cuda.synchronize()
    assert _rows(a) == _rows(b)
    ev = b.device_stats[-1]["blocks_evicted"]
    assert ev > 0
    assert all(rb.blocks_active <= ra.blocks_active for ra, rb in zip(a.stats, b.stats))
    assert b.stats[-1].blocks_active < a.stats[-1].blocks_active
    # evicted keys seen again were allocated again (frames after the turn-around)
    new_a = sum(d["new_blocks"] for d in a.device_stats[nframes:])
    new_b = sum(d["new_blocks"] for d in b.device_stats[nframes:])
    assert new_b > new_a
    ma, mb = a.compact(), b.compact()
    assert np.array_equal(ma.indices, mb.indices)
    assert np.array_equal(ma.positions, mb.positions)
    assert np.array_equal(ma.ages, mb.ages)
    assert np.array_equal(ma.normals, mb.normals)
    assert b.audit().ok
    # the snapshot lists live blocks only, all of them present in the never-evicting store
    sa, sb = a.store.snapshot_arrays(), b.store.snapshot_arrays()
    assert len(sb["coords"]) == b.stats[-1].blocks_active
    ka = {tuple(c) for c in sa["coords"].tolist()}
    assert {tuple(c) for c in sb["coords"].tolist()} <= ka
    print(config, "evicted", ev, "blocks", a.stats[-1].blocks_active, "->", b.stats[-1].blocks_active)


def test_block_gc_off_is_parity_mode():
    """block_gc_age = 0 (default) never evicts."""
    from paper_1803_03949_b200 import Engine, RunConfig
    from paper_1803_03949_b200.synth import camera_pose, config_spec, render_depth
    spec, cfg = config_spec("C2")
    spec.width, spec.height, spec.fx, spec.fy = 160, 120, 131.25, 131.25
    e = Engine(RunConfig(**cfg), spec.intrinsics())
    for i in range(0, 60, 3):
        p = camera_pose(spec, i)
        e.fuse_frame(render_depth(spec, p), p)
    assert e.device_stats[-1]["blocks_evicted"] == 0
    assert e.stats[-1].blocks_active == e.store.block_count
