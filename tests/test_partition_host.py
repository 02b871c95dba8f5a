"""Host logic of the spatial partition (CPU): global StatsRow reconstruction
from per-rank counters, and the same reconstruction through a gloo
world_size-2 process group (the NCCL path on the GPU box runs this code)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1803_03949_b200.partition import ADDITIVE, StatsCombiner, sum_stats


def _rank_streams(seed=0, frames=12, nranks=2):
    """Per-rank, per-frame counters with consistent live/alloc/free bookkeeping."""
    rng = np.random.default_rng(seed)
    out = [[] for _ in range(nranks)]
    for r in range(nranks):
        live = 0
        rec = 0
        for f in range(frames):
            alloc = int(rng.integers(0, 500))
            free = int(rng.integers(0, live + alloc + 1))
            live += alloc - free
            rec += free
            d = {k: int(rng.integers(0, 1000)) for k in ADDITIVE}
            d.update(new_vertices=alloc, vertices_freed=free, vertices_live=live,
                     vertices_recycled_total=rec)
            out[r].append(d)
    return out


def test_high_water_is_global_not_sum_of_rank_high_waters():
    # rank 0 frees everything while rank 1 allocates: global peak < sum of peaks
    r0 = [dict.fromkeys(ADDITIVE, 0), dict.fromkeys(ADDITIVE, 0)]
    r1 = [dict.fromkeys(ADDITIVE, 0), dict.fromkeys(ADDITIVE, 0)]
    r0[0].update(new_vertices=10, vertices_live=10)
    r0[1].update(new_vertices=0, vertices_freed=10, vertices_live=0)
    r1[0].update(new_vertices=0, vertices_live=0)
    r1[1].update(new_vertices=6, vertices_live=6)
    c = StatsCombiner()
    assert c.combine(sum_stats([r0[0], r1[0]]))["vertices_allocated_total"] == 10
    # frame 1: all allocations precede all frees -> peak = 10 + 6
    assert c.combine(sum_stats([r0[1], r1[1]]))["vertices_allocated_total"] == 16


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, streams, q):
    import torch.distributed as dist
    from paper_1803_03949_b200.partition import allreduce_frame_stats
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = StatsCombiner()
        rows = [c.combine(allreduce_frame_stats(d)) for d in streams[rank]]
        q.put((rank, rows))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_allreduce_matches_in_process_combination():
    streams = _rank_streams()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, streams, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    c = StatsCombiner()
    want = [c.combine(sum_stats([streams[0][f], streams[1][f]])) for f in range(len(streams[0]))]
    assert got[0] == want and got[1] == want


# ---- distributed compaction: metadata merge (CPU) --------------------------
def _random_metas(nranks=3, nblocks=200, seed=1):
    from paper_1803_03949_b200.partition import OwnedMeta
    rng = np.random.default_rng(seed)
    coords = rng.integers(-50, 50, size=(nblocks * 2, 3))
    coords = np.unique(coords, axis=0)[:nblocks]
    off = 1 << 20
    keys = (((coords[:, 0] + off) << 42) | ((coords[:, 1] + off) << 21) | (coords[:, 2] + off)).astype(np.uint64)
    owner = rng.integers(0, nranks, size=len(keys))
    occ = rng.integers(0, 2 ** 32, size=(len(keys), 48), dtype=np.uint64).astype(np.uint32)
    occ[rng.random(len(keys)) < 0.3] = 0
    vcnt = np.bitwise_count(occ).sum(axis=1).astype(np.int32)
    tcnt = rng.integers(0, 900, size=len(keys)).astype(np.int32)
    metas = []
    for r in range(nranks):
        sel = np.where(owner == r)[0]
        sel = sel[np.argsort(keys[sel])]
        metas.append(OwnedMeta(keys[sel], vcnt[sel], tcnt[sel], occ[sel]))
    return metas, coords, keys, vcnt, tcnt, occ


def test_merge_meta_is_the_sorted_block_order_with_exact_bases():
    """k-way merge by packed key == the reference's lexicographic block order
    (store.py:396-406); vertex / triangle bases are exclusive scans in that
    order; each rank's blocks land at their global positions."""
    from paper_1803_03949_b200.partition import merge_meta
    metas, coords, keys, vcnt, tcnt, occ = _random_metas()
    lay = merge_meta(metas)
    order = np.lexsort((coords[:, 2], coords[:, 1], coords[:, 0]))
    assert np.array_equal(lay.keys, keys[order])
    assert np.array_equal(lay.vbase, np.concatenate([[0], np.cumsum(vcnt[order])[:-1]]))
    assert np.array_equal(lay.tbase, np.concatenate([[0], np.cumsum(tcnt[order])[:-1]]))
    assert lay.nv == vcnt.sum() and lay.nt == tcnt.sum()
    for r, m in enumerate(metas):
        assert np.array_equal(lay.keys[lay.my_global[r]], m.keys)
    # slot index of a set bit = vbase + prefix popcount within the block
    g = 7
    w = 5
    expect = sum(bin(int(x)).count("1") for x in lay.occ[g, :w])
    assert lay.occ_pre[g, w] == expect


def test_merge_meta_rejects_a_block_owned_twice():
    from paper_1803_03949_b200.partition import merge_meta
    metas, *_ = _random_metas(nranks=2)
    with pytest.raises(RuntimeError):
        merge_meta([metas[0], metas[0]])


def _gather_worker(rank, world, port, metas, q):
    import torch.distributed as dist
    from paper_1803_03949_b200.partition import gather_metas, merge_meta
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        got = gather_metas(metas[rank])
        lay = merge_meta(got)
        q.put((rank, lay.keys.tolist(), lay.vbase.tolist(), lay.my_global[rank].tolist(),
               [m.occ.tolist() for m in got]))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_gather_metas_reassembles_every_rank():
    """The padded all-gather of owned-block metadata (PartitionedEngine.compact)
    over a gloo world_size-2 group gives every rank the same merged layout as
    the in-process merge."""
    from paper_1803_03949_b200.partition import merge_meta
    metas, *_ = _random_metas(nranks=2, nblocks=150, seed=4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, metas, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in procs:
        r, *rest = q.get(timeout=120)
        got[r] = rest
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    lay = merge_meta(metas)
    for r in (0, 1):
        keys, vbase, mine, occs = got[r]
        assert keys == lay.keys.tolist() and vbase == lay.vbase.tolist()
        assert mine == lay.my_global[r].tolist()
        assert all(np.array_equal(np.asarray(o, np.uint32), m.occ) for o, m in zip(occs, metas))
