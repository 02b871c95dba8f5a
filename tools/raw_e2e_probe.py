"""Per-frame wall times of the e2e legs (f64 host depth and raw u16) at the
driver's short setting (--steps 20 --warmup 5), to find one-time costs inside
the timed window.  usage: python tools/raw_e2e_probe.py [steps] [warmup] [repeats]"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import make_frames  # noqa: E402
from paper_1803_03949_b200 import Engine, RunConfig  # noqa: E402
from paper_1803_03949_b200.synth import config_spec  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
warmup = int(sys.argv[2]) if len(sys.argv) > 2 else 5
repeats = int(sys.argv[3]) if len(sys.argv) > 3 else 3
spec, cfg = config_spec("C2")
n = steps + warmup
dev = torch.device("cuda", 0)
poses, depths = make_frames(spec, n, dev)
host = [d.cpu().pin_memory().numpy() for d in depths]
raws = [torch.from_numpy(np.clip(np.rint(h * 5000.0), 0, 65535).astype(np.uint16)).pin_memory().numpy() for h in host]
caps = dict(block_capacity=60000)
for rep in range(repeats):
    for kind in ("f64", "raw"):
        e = Engine(RunConfig(**cfg, **caps), spec.intrinsics(), pipelined=True)
        call = (lambda i: e.fuse_frame(host[i], poses[i])) if kind == "f64" else \
               (lambda i: e.fuse_frame_raw(raws[i], poses[i]))
        for i in range(warmup):
            call(i)
        torch.cuda.synchronize()
        ts = []
        t0 = time.perf_counter()
        for k in range(steps):
            a = time.perf_counter()
            call(warmup + k)
            ts.append((time.perf_counter() - a) * 1e6)
        torch.cuda.synchronize()
        tot = time.perf_counter() - t0
        e.stats[-1].blocks_active
        print(f"rep {rep} {kind}: {steps / tot:.0f} frames/s, per-call us: "
              + " ".join(f"{t:.0f}" for t in ts), flush=True)
        del e
