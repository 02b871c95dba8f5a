"""Python-side cost of Engine.fuse_frame on the pipelined device-input path,
split by step (diagnostics; needs a GPU): argument checks + stream ordering,
pose conversion, the C call (incl. its wait for the previous frame), and the
row bookkeeping after it.  usage: python tools/py_overhead.py"""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_1803_03949_b200 import Engine, RunConfig, _lib  # noqa: E402
from paper_1803_03949_b200.synth import config_spec  # noqa: E402

W, N = 5, 200
spec, cfg = config_spec("C2")
dev = torch.device("cuda", 0)
poses, depths = bench.make_frames(spec, W + N, dev)
eng = Engine(RunConfig(block_capacity=30_000, vertex_capacity=12_000_000, **cfg), spec.intrinsics(), pipelined=True)
for i in range(W):
    eng.fuse_frame(depths[i], poses[i])
eng.stats[-1].blocks_active
torch.cuda.synchronize()
lib = _lib.load()
T = np.zeros((N, 5))
for k in range(N):
    i = W + k
    t0 = time.perf_counter_ns()
    ptr, h, w, on_dev, keep = eng._depth_args(depths[i])
    eng.store._touch()
    t1 = time.perf_counter_ns()
    pc = C.byref(_lib.pose_c(poses[i], eng._pose_c))
    t2 = time.perf_counter_ns()
    rc = lib.vm_fuse_frame_submit(eng.store._h, ptr, h, w, on_dev, C.byref(eng._intr_c), pc, C.byref(eng._fcfg),
                                  eng.frame_index)
    t3 = time.perf_counter_ns()
    eng._after_submit(rc, keep)
    t4 = time.perf_counter_ns()
    T[k] = (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0)
eng.stats[-1].blocks_active
torch.cuda.synchronize()
med = np.median(T, axis=0) / 1e3
print(f"median us: depth args + ordering {med[0]:.1f}, pose {med[1]:.1f}, C submit {med[2]:.1f}, "
      f"after submit {med[3]:.1f}, total {med[4]:.1f}")
t0 = time.perf_counter_ns()
for _ in range(1000):
    torch.cuda.current_stream(dev)
t1 = time.perf_counter_ns()
for _ in range(1000):
    torch._C._cuda_getCurrentRawStream(0)
t2 = time.perf_counter_ns()
ev = torch.cuda.Event()
s = torch.cuda.current_stream(dev)
for _ in range(1000):
    ev.record(s)
    ev.query()
t3 = time.perf_counter_ns()
st = _lib.Stats()
for _ in range(1000):
    st.as_dict()
t4 = time.perf_counter_ns()
print(f"current_stream {(t1 - t0) / 1e6:.2f} us, raw stream {(t2 - t1) / 1e6:.2f} us, "
      f"event record+query {(t3 - t2) / 1e6:.2f} us, Stats.as_dict {(t4 - t3) / 1e6:.2f} us")
