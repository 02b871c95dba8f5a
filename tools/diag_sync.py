"""Diagnostics: sync vs pipelined engine rows on device-tensor input (C2 at 320x240)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch
from paper_1803_03949_b200 import Engine, RunConfig
from paper_1803_03949_b200.synth import camera_pose, config_spec, render_depth_torch
spec, cfg = config_spec("C2")
spec.width, spec.height, spec.fx, spec.fy = 320, 240, 262.5, 262.5
intr = spec.intrinsics()
for mode in ("sync_dev", "sync_dev_synced", "sync_host", "pipe_dev"):
    e = Engine(RunConfig(**cfg), intr, pipelined=mode.startswith("pipe"))
    rows = []
    for i in range(4):
        p = camera_pose(spec, i)
        d = render_depth_torch(spec, p)
        if mode == "sync_dev_synced":
            torch.cuda.synchronize()
        if mode == "sync_host":
            d = d.cpu().numpy()
        e.fuse_frame(d, p)
    torch.cuda.synchronize()
    print(mode, [(r.blocks_active, r.vertices_live, r.triangles_live) for r in e.stats],
          [(s["valid_pixels"], s["collected_blocks"], s["nsteps"]) for s in e.device_stats], flush=True)
