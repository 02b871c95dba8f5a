"""In-process simulation of a partitioned reconstruction on one GPU (test
helper): N rank engines fed the same frames; in halo-exchange mode the
all-gather of the ranks' boundary-block records is done here, on the device,
exactly as partition.PartitionedEngine does it over torch.distributed.
halo "exchange-shard" also shards the band walk: rank r walks its slice of
pixel rows and lists the block keys it meets, the lists are concatenated (the
all-gather) and every rank collects its blocks from the union."""
import ctypes as C

import numpy as np


def rank_engines(cfg: dict, intr, nranks: int, tile_blocks: int, halo: str):
    from paper_1803_03949_b200 import Engine, RunConfig
    return [Engine(RunConfig(rank=r, nranks=nranks, tile_blocks=tile_blocks,
                             halo_exchange=halo.startswith("exchange"), **cfg), intr) for r in range(nranks)]


def fuse_all(engines, depth, pose, halo: str, log=None):
    """One frame on every rank engine; returns their device_stats rows."""
    if not halo.startswith("exchange"):
        for e in engines:
            e.fuse_frame(depth, pose)
        return [e.device_stats[-1] for e in engines]
    import torch
    from paper_1803_03949_b200 import _lib
    L = _lib.load()
    rec = _lib.GHOST_RECORD
    sends, counts = [], []
    allk = None
    if halo == "exchange-shard":
        nr = len(engines)
        lists = []
        for r, e in enumerate(engines):
            ptr, h, w, on_dev, keep = e._depth_args(depth)
            rows = [(h * q // nr) // 8 * 8 for q in range(nr)] + [h]
            keys = torch.empty(1 << 20, dtype=torch.int64, device="cuda")
            nk = C.c_int64(0)
            _lib.check(L.vm_partition_collect_keys(e.store._h, ptr, h, w, on_dev, C.byref(e._intr_c),
                                                   C.byref(_lib.pose_c(pose)), C.byref(e._fcfg),
                                                   e.frame_index, rows[r], rows[r + 1],
                                                   C.c_void_p(keys.data_ptr()), keys.numel(), C.byref(nk)))
            lists.append(keys[: nk.value])
        allk = torch.cat(lists)
        torch.cuda.synchronize()
    for e in engines:
        ptr, h, w, on_dev, keep = e._depth_args(depth)
        cap = 1024
        buf = torch.empty(cap * rec, dtype=torch.uint8, device="cuda")
        n, nown = C.c_int64(), C.c_int64()
        if allk is not None:
            _lib.check(L.vm_partition_frame_begin_keys(e.store._h, C.c_void_p(allk.data_ptr()), allk.numel(),
                                                       C.c_void_p(buf.data_ptr()), cap, C.byref(n), C.byref(nown)))
        else:
            _lib.check(L.vm_partition_frame_begin(e.store._h, ptr, h, w, on_dev, C.byref(e._intr_c),
                                                  C.byref(_lib.pose_c(pose)), C.byref(e._fcfg), e.frame_index,
                                                  C.c_void_p(buf.data_ptr()), cap, C.byref(n), C.byref(nown)))
        if n.value > cap:
            cap = n.value + 7
            buf = torch.empty(cap * rec, dtype=torch.uint8, device="cuda")
            _lib.check(L.vm_partition_repack(e.store._h, C.c_void_p(buf.data_ptr()), cap, C.byref(n)))
        sends.append(buf)
        counts.append(n.value)
    maxc = max(counts)
    counts_a = np.asarray(counts, np.int32)
    recv = torch.cat([s[: maxc * rec] for s in sends]) if maxc else None
    torch.cuda.synchronize()
    if log is not None:
        log.append(list(counts))
    for e in engines:
        st = _lib.Stats()
        _lib.check(L.vm_partition_frame_finish(e.store._h, C.c_void_p(recv.data_ptr()) if recv is not None
                                               else None, _lib.ptr(counts_a), len(engines), maxc,
                                               C.byref(st)))
        e._record(st)
    return [e.device_stats[-1] for e in engines]
