"""Host vs device in the back-to-back stream (bench.py's `value` path):
per-frame period of Engine.fuse_frame (pipelined, device-resident frames,
engine's own stream), the C submit split (VOXMESH_B200_HOST_PROF: enqueue =
kernel launches, settle = waiting for the previous frame), and the same
frames through the bare C call.  Diagnostics; needs a GPU."""
import ctypes as C
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

os.environ["VOXMESH_B200_HOST_PROF"] = "1"
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_1803_03949_b200 import Engine, RunConfig, _lib  # noqa: E402
from paper_1803_03949_b200.synth import config_spec  # noqa: E402

W, N = 5, 295
spec, cfg = config_spec(os.environ.get("VM_CONFIG", "C2"))
dev = torch.device("cuda", 0)
poses, depths = bench.make_frames(spec, W + N, dev)
caps = dict(block_capacity=int(os.environ.get("VM_BLOCKS", 30_000)), vertex_capacity=int(os.environ.get("VM_RECORDS", 12_000_000)))


def run(label, bare):
    eng = Engine(RunConfig(**cfg, **caps), spec.intrinsics(), pipelined=True)
    for i in range(W):
        eng.fuse_frame(depths[i], poses[i])
    eng.stats[-1].blocks_active
    torch.cuda.synchronize()
    est = torch.cuda.ExternalStream(eng.stream_handle(), device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lib = _lib.load()
    pcs = [_lib.pose_c(p) for p in poses]
    st = _lib.Stats()
    e0.record(est)
    t0 = time.perf_counter()
    if bare:
        for i in range(W, W + N):
            rc = lib.vm_fuse_frame_submit(eng.store._h, C.c_void_p(depths[i].data_ptr()), spec.height, spec.width, 1,
                                          C.byref(eng._intr_c), C.byref(pcs[i]), C.byref(eng._fcfg), i)
            lib.vm_fuse_frame_result(eng.store._h, C.byref(st))
    else:
        for i in range(W, W + N):
            eng.fuse_frame(depths[i], poses[i])
    e1.record(est)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    print(f"{label}: wall {1e6 * wall / N:6.1f} us/frame, device {1e3 * e0.elapsed_time(e1) / N:6.1f} us/frame",
          flush=True)
    eng.store.__del__()
    del eng


run("Engine.fuse_frame", False)
run("bare C submit", True)
