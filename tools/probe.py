"""Quick GPU probe: C2 frames, per-kernel times (profiled engine) and whole-frame
device time (unprofiled engine, PDL overlap intact).  Development aid."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_1803_03949_b200 import Engine, RunConfig
from paper_1803_03949_b200.synth import config_spec, camera_pose, render_depth_torch

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
nf = int(sys.argv[2]) if len(sys.argv) > 2 else 30
spec, cfg = config_spec(name)
poses = [camera_pose(spec, i) for i in range(nf)]
depths = [render_depth_torch(spec, p) for p in poses]
torch.cuda.synchronize()
prof = Engine(RunConfig(**cfg, block_capacity=16384), spec.intrinsics())
prof.set_profiling(True)
plain = Engine(RunConfig(**cfg, block_capacity=16384), spec.intrinsics())
tot_p, tot = 0.0, 0.0
acc = None
for i in range(nf):
    prof.fuse_frame(depths[i], poses[i])
    ph = prof.phase_times()
    row = plain.fuse_frame(depths[i], poses[i])
    if i >= 5:
        tot += plain.device_stats[-1]["device_ms"]
        tot_p += prof.device_stats[-1]["device_ms"]
        acc = {k: acc.get(k, 0) + v for k, v in ph.items()} if acc else dict(ph)
m = nf - 5
print("per-kernel mean ms (profiled):", {k: round(v / m, 4) for k, v in acc.items()})
print(f"frame device ms: profiled {tot_p / m:.4f}  unprofiled {tot / m:.4f}  "
      f"(blocks {row.blocks_active} V {row.vertices_live} T {row.triangles_live})")
