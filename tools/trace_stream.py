"""Per-CTA kernel timelines of consecutive frames of a back-to-back stream
(pipelined submission of device-resident frames on the engine's own stream,
i.e. the `value` path of bench.py with frame overlap), on one time base.
Diagnostics; needs a GPU.  usage: python tools/trace_stream.py [first=150] [n=3] [config=C2]
Runs the trajectory to frame `first`, traces `n` consecutive frames into one
buffer each and prints, per frame and kernel: the CTA start / end spread
(first start, median end, last end) and the gaps between kernels."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1803_03949_b200 import build as _build  # noqa: E402
os.environ["VOXMESH_B200_LIB"] = str(_build.build(trace=True))   # the -DVM_TRACE variant
import bench  # noqa: E402
from paper_1803_03949_b200 import Engine, RunConfig  # noqa: E402
from paper_1803_03949_b200.synth import config_spec  # noqa: E402

FIRST = int(sys.argv[1]) if len(sys.argv) > 1 else 150
N = int(sys.argv[2]) if len(sys.argv) > 2 else 3
CONF = sys.argv[3] if len(sys.argv) > 3 else "C2"
NAMES = ["collect", "fuse", "retype", "gc"]
CTAS, SLOTS = 2048, 32

spec, cfg = config_spec(CONF)
spec.frames = FIRST + N
dev = torch.device("cuda", 0)
poses, depths = bench.make_frames(spec, FIRST + N, dev)
eng = Engine(RunConfig(block_capacity=60_000, vertex_capacity=16_000_000, **cfg), spec.intrinsics(),
             pipelined=True)
for i in range(FIRST):
    eng.fuse_frame(depths[i], poses[i])
bufs = [torch.zeros(4 * CTAS * SLOTS, dtype=torch.int64, device=dev) for _ in range(N)]
torch.cuda.synchronize()
for k in range(N):
    eng.set_trace(bufs[k])
    eng.fuse_frame(depths[FIRST + k], poses[FIRST + k])
eng.set_trace(None)
eng.stats[-1].blocks_active
torch.cuda.synchronize()
trs = [b.view(4, CTAS, SLOTS).cpu().numpy().astype(np.int64) for b in bufs]
t0 = min(tr[k][:, 0][tr[k][:, 0] > 0].min() for tr in trs for k in range(4) if (tr[k][:, 0] > 0).any())
print(f"{CONF} frames {FIRST}..{FIRST + N - 1}, back to back; overlapped:",
      [d["overlapped"] for d in eng.device_stats[FIRST:FIRST + N]])
prev_end = None
for f, tr in enumerate(trs):
    print(f"frame {FIRST + f}:", {k: eng.device_stats[FIRST + f][k] for k in
                                   ("collected_blocks", "halo_blocks", "normals_computed")})
    for k, name in enumerate(NAMES):
        m = tr[k]
        m = m[m[:, 0] > 0]
        if not len(m):
            continue
        st, en = (m[:, 0] - t0) / 1e3, (m[:, 31] - t0) / 1e3
        gap = f" (starts {st.min() - prev_end:+.2f} us after the previous kernel's last CTA)" if prev_end else ""
        print(f"  {name:7s} {len(m):5d} CTAs  first start {st.min():8.2f}  start p50 {np.percentile(st, 50):8.2f}  "
              f"first end {en.min():8.2f}  end p50 {np.percentile(en, 50):8.2f}  last end {en.max():8.2f}{gap}")
        prev_end = en.max()
