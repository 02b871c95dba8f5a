"""Per-CTA timeline of one C2 frame (diagnostics; needs a GPU).
usage: python tools/trace_frame.py [frame=40] [config=C2]
Runs frames 0..frame-1, traces frame `frame` (csrc/vm_device.cuh kTraceCtas
layout) and prints, per kernel: the CTA start/end spread, the distribution of
CTA durations, items per CTA, and the phase split of the slowest CTAs."""
import sys
from pathlib import Path

import os

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1803_03949_b200 import build as _build  # noqa: E402
os.environ["VOXMESH_B200_LIB"] = str(_build.build(trace=True))   # the -DVM_TRACE variant
import bench  # noqa: E402
from paper_1803_03949_b200 import Engine, RunConfig  # noqa: E402

FRAME = int(sys.argv[1]) if len(sys.argv) > 1 else 40
CONF = sys.argv[2] if len(sys.argv) > 2 else "C2"
NAMES = ["collect", "fuse_blocks", "retype_place", "gc_normals"]
CTAS, SLOTS = 2048, 32

from paper_1803_03949_b200.synth import config_spec  # noqa: E402
spec, cfg = config_spec(CONF)
spec.frames = FRAME + 1
dev = torch.device("cuda", 0)
poses, depths = bench.make_frames(spec, FRAME + 1, dev)
eng = Engine(RunConfig(**cfg), spec.intrinsics())
for i in range(FRAME):
    eng.fuse_frame(depths[i], poses[i])
buf = torch.zeros(4 * CTAS * SLOTS, dtype=torch.int64, device=dev)
flush = torch.empty(256 << 18, dtype=torch.int32, device=dev)
flush.zero_()
torch.cuda.synchronize()
eng.set_trace(buf)
eng.fuse_frame(depths[FRAME], poses[FRAME])
eng.set_trace(None)
torch.cuda.synchronize()
tr = buf.view(4, CTAS, SLOTS).cpu().numpy().astype(np.int64)
print("frame", FRAME, {k: v for k, v in eng.device_stats[-1].items()
                       if k in ("collected_blocks", "scope_blocks", "halo_blocks", "normals_computed",
                                "fallback_normals", "edge_placements", "device_ms")})
t0 = min(tr[k][:, 0][tr[k][:, 0] > 0].min() for k in range(4) if (tr[k][:, 0] > 0).any())
for k, name in enumerate(NAMES):
    m = tr[k]
    live = m[:, 0] > 0
    if not live.any():
        continue
    m = m[live]
    st, en = (m[:, 0] - t0) / 1e3, (m[:, 31] - t0) / 1e3
    dur = en - st
    items = m[:, 27]
    print(f"\n{name}: {live.sum()} CTAs  start {st.min():.2f}..{st.max():.2f} us  end {en.min():.2f}..{en.max():.2f} us"
          f"  dur p50 {np.percentile(dur, 50):.2f} p90 {np.percentile(dur, 90):.2f} max {dur.max():.2f}"
          f"  items/CTA {np.bincount(items.clip(0, 10)).tolist()}")
    pro = (m[:, 1] - m[:, 0]) / 1e3
    print(f"  prologue p50 {np.percentile(pro, 50):.2f} max {pro.max():.2f} us")
    order = list(np.argsort(-en)[:3])
    if (m[:, 28] > 0).any():   # + the CTAs whose item loop finished last
        order += [i for i in np.argsort(-m[:, 28])[:2] if i not in order]
    for idx in order:
        row = m[idx]
        segs = []
        for it in range(min(int(row[27]), 5)):
            ts = [row[2 + 4 * it + p] for p in range(4)]
            prev = ts[0]
            parts = []
            for p in range(1, 4):
                if ts[p] > 0:
                    parts.append(f"{(ts[p] - prev) / 1e3:.2f}")
                    prev = ts[p]
            segs.append(f"[{(ts[0] - t0) / 1e3:.2f}: {'/'.join(parts)}]")
        extra = " ".join(f"s{p}={(row[p] - t0) / 1e3:.2f}" for p in (22, 23, 24, 25, 26, 28, 29, 30) if row[p] > 0)
        print(f"  slow CTA end {(row[31] - t0) / 1e3:.2f} items {row[27]} {' '.join(segs)} {extra}")

# per-SM view of gc: items and the latest item end on each SM
m = tr[3]
live = (m[:, 0] > 0) & (m[:, 27] > 0)
if live.any():
    sm = m[live, 24]
    en = (m[live, 28] - t0) / 1e3
    nv = m[live, 25]
    import collections
    per = collections.defaultdict(list)
    for a, e, v in zip(sm, en, nv):
        per[int(a)].append((e, int(v)))
    worst = sorted(per.items(), key=lambda kv: -max(e for e, _ in kv[1]))[:5]
    print("\ngc per SM (items, sum nv, latest item end):")
    for s_, L in worst:
        print(f"  sm {s_}: {len(L)} items, nv {sum(v for _, v in L)}, latest {max(e for e, _ in L):.2f} us")
    allsm = [(len(L), sum(v for _, v in L)) for L in per.values()]
    print("  SMs:", len(per), "items/SM min/max", min(a for a, _ in allsm), max(a for a, _ in allsm),
          "nv/SM min/max", min(b for _, b in allsm), max(b for _, b in allsm))
    print("  SM of gc CTAs 0..39:", [int(x) for x in m[:40, 24]] if len(m) >= 40 else [])
