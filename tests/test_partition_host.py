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
