"""Per-frame kernel spans in the e2e setting (pipelined Engine, pinned host
depth, no L2 flush): for frames W..W+N of C2, the gap from one frame's last
kernel end to the next frame's first kernel start, and each kernel's span.
Diagnostics build (-DVM_TRACE: block-0 start / latest CTA end per kernel and
frame in a ring).  usage: python tools/trace_gaps.py [first=40] [n=40]"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1803_03949_b200 import build as _build  # noqa: E402
os.environ["VOXMESH_B200_LIB"] = str(_build.build(trace=True))
import bench  # noqa: E402
from paper_1803_03949_b200 import Engine, RunConfig  # noqa: E402
from paper_1803_03949_b200.synth import config_spec  # noqa: E402

FIRST = int(sys.argv[1]) if len(sys.argv) > 1 else 40
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
CTAS, SLOTS = 2048, 32
spec, cfg = config_spec("C2")
spec.frames = FIRST + N
dev = torch.device("cuda", 0)
poses, depths = bench.make_frames(spec, FIRST + N, dev)
host = [torch.empty(d.shape, dtype=torch.float64, pin_memory=True) for d in depths]
for hd, d in zip(host, depths):
    hd.copy_(d)
host_np = [h.numpy() for h in host]
eng = Engine(RunConfig(**cfg), spec.intrinsics(), pipelined=True)
buf = torch.zeros(4 * CTAS * SLOTS + 256 * 8, dtype=torch.int64, device=dev)
for i in range(FIRST):
    eng.fuse_frame(host_np[i], poses[i])
torch.cuda.synchronize()
eng.set_trace(buf)
for i in range(FIRST, FIRST + N):
    eng.fuse_frame(host_np[i], poses[i])
eng.stats[-1].blocks_active
torch.cuda.synchronize()
ring = buf[4 * CTAS * SLOTS:].view(256, 8).cpu().numpy().astype(np.int64)
rows = [ring[f & 255] for f in range(FIRST, FIRST + N)]
names = ["collect", "fuse", "retype", "gc"]
spans = {n: [] for n in names}
gaps = {n: [] for n in names}   # start of kernel k - end of the previous kernel
for j, r in enumerate(rows):
    for k, n in enumerate(names):
        spans[n].append((r[2 * k + 1] - r[2 * k]) / 1e3)
        prev_end = r[2 * k - 1] if k > 0 else (rows[j - 1][7] if j > 0 else 0)
        if prev_end:
            gaps[n].append((r[2 * k] - prev_end) / 1e3)
frame = [(rows[j + 1][0] - rows[j][0]) / 1e3 for j in range(len(rows) - 1)]
print(f"frames {FIRST}..{FIRST + N - 1}: frame period mean {np.mean(frame):.2f} us (median {np.median(frame):.2f})")
for n in names:
    print(f"  {n:8s} span mean {np.mean(spans[n]):6.2f}  gap before mean {np.mean(gaps[n]):6.2f} "
          f"median {np.median(gaps[n]):6.2f} max {np.max(gaps[n]):6.2f} us")
