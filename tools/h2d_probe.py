"""Host->device bandwidth of one C2 depth frame (2.46 MB, pinned), as one copy
and split over several streams; also the raw u16 frame.  Diagnostics for the
e2e leg.  usage: python tools/h2d_probe.py"""
import time

import torch

n = 640 * 480
for dtype, name in ((torch.float64, "f64"), (torch.uint16, "u16")):
    host = torch.empty(n, dtype=dtype).pin_memory()
    dev = torch.empty(n, dtype=dtype, device="cuda")
    nbytes = host.numel() * host.element_size()
    for parts in (1, 2, 4, 8):
        streams = [torch.cuda.Stream() for _ in range(parts)]
        chunk = (n + parts - 1) // parts
        for rep in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for it in range(200):
                for p, st in enumerate(streams):
                    with torch.cuda.stream(st):
                        dev[p * chunk:(p + 1) * chunk].copy_(host[p * chunk:(p + 1) * chunk], non_blocking=True)
                for st in streams:
                    st.synchronize()
            dt = (time.perf_counter() - t0) / 200
        print(f"{name} {nbytes / 1e6:.2f} MB, {parts} stream(s): {dt * 1e6:.1f} us/frame = {nbytes / dt / 1e9:.1f} GB/s",
              flush=True)
