"""Quick GPU probe: C2 frames timed per phase (development aid)."""
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
t0 = time.time()
poses = [camera_pose(spec, i) for i in range(nf)]
depths = [render_depth_torch(spec, p) for p in poses]
torch.cuda.synchronize()
print(f"rendered {nf} frames in {time.time()-t0:.1f}s", flush=True)
eng = Engine(RunConfig(**cfg), spec.intrinsics())
eng.set_profiling(True)
tot = 0.0
for i in range(nf):
    row = eng.fuse_frame(depths[i], poses[i])
    ds = eng.device_stats[-1]
    ph = eng.phase_times()
    if i < 3 or i % 10 == 0 or i == nf - 1:
        print(i, f"dev {ds['device_ms']:.3f} ms", {k: round(v, 3) for k, v in ph.items()},
              {k: ds[k] for k in ("collected_blocks", "new_blocks", "scope_blocks", "halo_blocks",
                                  "active_cubes", "new_vertices", "changed_cubes", "triangles_allocated",
                                  "vertices_freed", "fallback_normals", "resumes")}, flush=True)
    if i >= 3:
        tot += ds["device_ms"]
print(f"mean device ms/frame (frames 3..): {tot/(nf-3):.3f}  blocks {row.blocks_active} V {row.vertices_live} T {row.triangles_live}")
