"""Host-side cost of the pipelined submission path (diagnostics, needs a GPU):
per-frame wall time of Engine.fuse_frame split into the C submit call and the
Python around it, for pinned host f64 depth, raw u16 and device-resident depth."""
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

W, N = 40, 100
spec, cfg = config_spec("C2")
spec.frames = W + N
dev = torch.device("cuda", 0)
poses, depths = bench.make_frames(spec, W + N, dev)
host = [torch.empty(d.shape, dtype=torch.float64, pin_memory=True) for d in depths]
for hd, d in zip(host, depths):
    hd.copy_(d)
host_np = [h.numpy() for h in host]
raws = [torch.from_numpy(np.clip(np.rint(h * 5000.0), 0, 65535).astype(np.uint16)).pin_memory().numpy()
        for h in host_np]

lib = _lib.load()
orig = lib.vm_fuse_frame_submit
for name, src, fn in [("f64 pinned", host_np, "fuse_frame"), ("device f64", depths, "fuse_frame"),
                      ("raw u16", raws, "fuse_frame_raw")]:
    eng = Engine(RunConfig(**cfg), spec.intrinsics(), pipelined=True)
    f = getattr(eng, fn)
    for i in range(W):
        f(src[i], poses[i])
    torch.cuda.synchronize()
    t_call = []
    t0 = time.perf_counter()
    for i in range(W, W + N):
        a = time.perf_counter()
        f(src[i], poses[i])
        t_call.append(time.perf_counter() - a)
    eng.stats[-1].blocks_active
    torch.cuda.synchronize()
    tot = time.perf_counter() - t0
    print(f"{name:11s}: period {1e6 * tot / N:6.1f} us/frame  call mean {1e6 * np.mean(t_call):6.1f} "
          f"median {1e6 * np.median(t_call):6.1f} us")

# the C call alone (submit + settle inside), device depth, no Python wrapper work
eng = Engine(RunConfig(**cfg), spec.intrinsics(), pipelined=True)
for i in range(W):
    eng.fuse_frame(depths[i], poses[i])
torch.cuda.synchronize()
import ctypes as C  # noqa: E402
st = _lib.Stats()
ts = []
t0 = time.perf_counter()
for i in range(W, W + N):
    pc = _lib.pose_c(poses[i])
    a = time.perf_counter()
    rc = lib.vm_fuse_frame_submit(eng.store._h, C.c_void_p(depths[i].data_ptr()), spec.height, spec.width, 1,
                                  C.byref(eng._intr_c), C.byref(pc), C.byref(eng._fcfg), i)
    b = time.perf_counter()
    lib.vm_fuse_frame_result(eng.store._h, C.byref(st))
    ts.append((b - a, time.perf_counter() - b))
    assert rc == 0
torch.cuda.synchronize()
tot = time.perf_counter() - t0
ts = np.array(ts) * 1e6
print(f"raw C submit (device depth): period {1e6 * tot / N:6.1f} us/frame, submit {ts[:, 0].mean():6.1f} "
      f"(median {np.median(ts[:, 0]):6.1f}), result {ts[:, 1].mean():5.1f} us")
