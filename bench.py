#!/usr/bin/env python
"""Benchmark: depth frames/sec of integrate + incremental mesh update (+GC) on
BASELINE.json configs[1] = C2 (synthetic room, 300-frame trajectory, 640x480,
8 mm voxels), one step = one depth frame through ``Engine.fuse_frame``.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl reference]

Arms
* default: the B200 path.  ``value`` = K / sum of per-frame device times
  (CUDA events on the engine's stream = torch's current stream; depth already
  in HBM; L2 flushed with a 256 MiB write between frames, outside the events).
  ``e2e`` = the same frames through the public API with pinned host depth
  (H2D every frame) and the StatsRow D2H, wall clock.  ``roofline`` = the
  dominant kernel's algorithmic bytes / its mean event-timed duration against
  MEASURED_PEAKS.json hbm_gbs.  ``cpu_baseline`` = the CPU oracle port
  (oracle/, serial C restatement of the reference) on a bounded prefix.
* --impl reference: the reference CPU algorithm (the oracle port, 1 core) on
  the same frames, and next to it the reference itself (pure-Python voxmesh
  from baseline/_ref) at serial/1 and claim/os.cpu_count() for a bounded
  prefix.  ``parity`` (default arm): a fresh B200 engine over the oracle
  leg's frames, diffed against the oracle's rows and final state.
Multi-GPU (torchrun, NCCL): default ``--mode partition`` -- one reconstruction
spatially partitioned across the ranks (hashed tiles of --tile-blocks^3
blocks), every rank fed the same frame; strong scaling,
value = K / sum over frames of the max-over-ranks frame device time; the
per-frame global StatsRow is one NCCL int64 all-reduce (inside e2e).
``--mode replicas``: independent replicas (weak scaling).
"""
from __future__ import annotations

import argparse
import gc
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "depth frames/sec (integrate+mesh) at 640x480, 8mm voxels; % of HBM roofline"
FLUSH_BYTES = 256 << 20

# Algorithmic bytes per unit of the current device layout:
# a corner sample is tsdf f64 + weight i32 (12 B); cube types 2 x u8; an edge
# slot is occupancy 1 bit + birth i32 + coordinate f64 + normal 3 x f64; a hash
# probe reads one 128-B bucket.
SAMPLE = 12
OCC = 1536 // 8        # occupancy bitmap bytes per block
BUCKET = 128


def phase_bytes(ds: dict, h: int, w: int) -> dict:
    """Compulsory bytes per kernel for one frame's unit counts (each touched
    byte once; re-reads that hit L2 are not counted)."""
    depth = h * w * 8
    coll, new, scope, halo = ds["collected_blocks"], ds["new_blocks"], ds["scope_blocks"], ds["halo_blocks"]
    old = coll - new
    return {
        "depth_stats": depth,
        # depth + one bucket probe and stamp per collected block + new-block records
        "collect": depth + coll * (BUCKET + 8) + new * 40,
        # old state read + new state written, init of new blocks (samples, types,
        # births, occupancy), depth gathers, neighbour rows + stamps
        "fuse_blocks": old * 512 * SAMPLE + coll * 512 * SAMPLE + new * (512 * (SAMPLE + 2) + 1536 * 4 + OCC)
        + min(coll * 512, h * w) * 8 + coll * 27 * 12,
        # (B+1)^3 sample tile, types read + written, per placement coordinate +
        # occupancy word, new vertex birth + normal
        "retype_place": scope * (729 * SAMPLE + 1024 + 1024) + ds["edge_placements"] * (8 + 4)
        + ds["new_vertices"] * (4 + 24),
        # occupancy + 9^3 type tile, 12-sample stencil + normal per vertex,
        # freed births, fallback records and incident vertex coordinates
        "gc_normals": halo * (OCC + 729) + ds["normals_computed"] * (12 * SAMPLE + 24)
        + ds["vertices_freed"] * 4 + ds["fallback_normals"] * (16 + 27 * 4 + 20 * 3 * 8 + 24),
    }


# ---------------------------------------------------------------- helpers
def measured_peak_gbs():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[2:6]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def make_frames(spec, nframes, device):
    from paper_1803_03949_b200.synth import camera_pose, multiroom_pose, render_depth, render_depth_torch
    pose_fn = multiroom_pose if spec.scene == "multiroom" else camera_pose
    poses = [pose_fn(spec, i) for i in range(nframes)]
    if device is not None:
        depths = [render_depth_torch(spec, p, device=device) for p in poses]
    else:
        depths = [render_depth(spec, p) for p in poses]
    return poses, depths


def oracle_run(spec, cfg, depths_host, poses, budget_s, warmup=0, return_engine=False):
    """Time the CPU oracle (serial C port of the reference) frame by frame."""
    from oracle.oracle import OracleEngine
    intr = spec.intrinsics()
    eng = OracleEngine(cfg, (intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height))
    for i in range(min(warmup, len(depths_host))):
        eng.fuse_frame(depths_host[i], poses[i].rotation, poses[i].translation)
    t_total, n = 0.0, 0
    for i in range(warmup, len(depths_host)):
        t0 = time.perf_counter()
        eng.fuse_frame(depths_host[i], poses[i].rotation, poses[i].translation)
        t_total += time.perf_counter() - t0
        n += 1
        if t_total > budget_s:
            break
    return (n, t_total, eng) if return_engine else (n, t_total)


REF_PKG = ROOT / "baseline" / "_ref"


def python_reference_run(spec, cfg, depths_host, poses, strategy, workers, budget_s):
    """The reference itself (pure-Python ``voxmesh``, installed unmodified into
    baseline/_ref by `pip install --target`), timed with its own StatsRow
    fusion_ms + meshing_ms (engine.py:123-165) over frames 0.. until the budget
    is spent.  Returns None when the install is absent."""
    if not (REF_PKG / "voxmesh").is_dir():
        return None
    if str(REF_PKG) not in sys.path:
        sys.path.insert(0, str(REF_PKG))
    import voxmesh
    intr = spec.intrinsics()
    rc = voxmesh.RunConfig(strategy=strategy, workers=workers, **cfg)
    eng = voxmesh.Engine(rc, voxmesh.Intrinsics(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height))
    ms, n = 0.0, 0
    for i in range(len(depths_host)):
        row = eng.fuse_frame(depths_host[i], voxmesh.Pose(poses[i].rotation, poses[i].translation))
        ms += row.fusion_ms + row.meshing_ms
        n += 1
        if ms / 1e3 > budget_s:
            break
    cores = eng.config.workers if strategy != "serial" else 1
    return {"value": n / (ms / 1e3), "unit": "frames/s", "cores": int(cores), "strategy": strategy,
            "workers": int(eng.config.workers), "kind": "reference (pure-Python voxmesh, baseline/_ref)",
            "sample": f"{n} frames (0..{n - 1}), engine's own fusion_ms + meshing_ms = {ms / 1e3:.1f} s"}


def python_reference_legs(spec, cfg, depths_host, poses, budget_s):
    """serial/1 (fastest, one core busy) and the default claim/os.cpu_count()
    (SURVEY.md 8d timing)."""
    out = []
    for strategy, workers in (("serial", 1), ("claim", 0)):
        r = python_reference_run(spec, cfg, depths_host, poses, strategy, workers, budget_s)
        if r is None:
            return [{"unavailable": "baseline/_ref/voxmesh not installed"}]
        out.append(r)
    return out


def parity_vs_oracle(spec, cfg, depths_dev, poses, ora, n, strategy):
    """A fresh B200 engine over the oracle leg's frames 0..n-1 (device depth),
    diffed against the oracle's rows and final state (oracle/parity.py)."""
    from oracle.parity import compare_rows, compare_state
    from paper_1803_03949_b200 import Engine, RunConfig
    eng = Engine(RunConfig(strategy=strategy, **cfg), spec.intrinsics())
    for i in range(n):
        eng.fuse_frame(depths_dev[i], poses[i])
    rows = compare_rows(eng.stats, ora.stats)
    st = compare_state(eng, ora)
    return {"frames": n, "match": bool(rows["match"] and st["match"]), "rows": rows,
            "state": {k: v for k, v in st.items() if k != "match"},
            "checked": "StatsRow every frame; final block set, tsdf, weight, type_prev, type_curr, "
                       "compact positions / indices / ages bit-exact, normals <= 1e-12"}


# ---------------------------------------------------------------- arms
def run_reference(args, spec, cfg, rank, world):
    import torch
    if rank != 0:
        return
    nframes = args.warmup + args.steps
    dev = "cuda" if torch.cuda.is_available() else None
    poses, depths = make_frames(spec, nframes, dev)
    host = [d.cpu().numpy() if dev else d for d in depths]
    n, t = oracle_run(spec, cfg, host, poses, budget_s=args.ref_budget, warmup=args.warmup)
    v = n / t if t > 0 else 0.0
    sample = (f"{args.config} frames {args.warmup}..{args.warmup + n - 1} after {args.warmup} "
              f"untimed warm-up frames (time cap {args.ref_budget:.0f} s)")
    pyref = python_reference_legs(spec, cfg, host, poses, args.pyref_budget)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "frames/s", "n_gpus": world,
            "steps": n, "warmup": args.warmup, "ms_per_step": 1e3 * t / max(n, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (sphere-traced analytic scene)", "config": workload(args, spec, cfg),
            "cpu_baseline": {"value": v, "unit": "frames/s", "cores": 1, "kind": "port",
                             "sample": sample},
            # the reference itself (pure Python) next to its C port, same frames from 0
            "python_reference": pyref,
            "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


CONFIG_TEXT = {
    "C1": "BASELINE.json configs[0] synthetic sphere+box scene",
    "C2": "BASELINE.json configs[1] synthetic room 4x4x2.5 m, 300-frame trajectory",
    "C3": "BASELINE.json configs[2] room with Hamming refinement every frame",
    "C4": "BASELINE.json configs[3] fine resolution room, 40 mm band",
    "C5": "BASELINE.json configs[4] 20x20 m multi-room scene",
}


class PausedGC:
    """Python's cyclic collector is run once and paused for a timed loop: a
    generation-2 pass over torch's objects takes milliseconds and lands at a
    random frame (profiles/r2_v3_raw_e2e_probe.txt: one 12 ms call)."""

    def __enter__(self):
        gc.collect()
        gc.disable()

    def __exit__(self, *exc):
        gc.enable()


def workload(args, spec, cfg):
    return {"workload": f"{args.config}: {CONFIG_TEXT.get(args.config, args.config)}, "
                        f"{spec.width}x{spec.height} depth, {cfg['cube_size'] * 1e3:.0f} mm voxels, "
                        "integrate + incremental mesh update (+refine) + GC",
            "frames": args.warmup + args.steps, "width": spec.width, "height": spec.height,
            "cube_size_m": cfg["cube_size"], "trunc_m": cfg["trunc"],
            "refine": bool(cfg.get("refine", False)), "strategy": args.strategy,
            "l2": ("not flushed: inputs larger than L2 (each step reads its own 2.46 MB depth frame, the timed "
                   "frames are > 126 MB); value_l2_flushed = the same frames each timed alone after a 256 MiB "
                   "L2 flush"),
            "python_gc": "collected, then paused during each timed loop",
            "halo": args.halo if args.gpus > 1 and args.mode == "partition" else None,
            "parallelism": (f"spatial partition x{args.gpus} (tiles of {args.tile_blocks}^3 blocks, "
                            f"halo {args.halo})"
                            if args.gpus > 1 and args.mode == "partition" else
                            f"replicas x{args.gpus}" if args.gpus > 1 else "single GPU")}


def run_gpu(args, spec, cfg, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_1803_03949_b200 import Engine, RunConfig
    from paper_1803_03949_b200.partition import PartitionedEngine
    part = world > 1 and args.mode == "partition"
    xchg = part and args.halo == "exchange"
    ekw = dict(rank=rank, nranks=world, tile_blocks=args.tile_blocks) if part else {}
    gloo = world > 1 and str(dist.get_backend()).lower() != "nccl"

    def reduce_(vals, op):
        """all-reduce of a float64 vector (gloo: on the host)"""
        t = torch.tensor(vals, dtype=torch.float64, device="cpu" if gloo else dev)
        dist.all_reduce(t, op=op)
        return t.cpu().tolist()
    local_rank %= torch.cuda.device_count()   # (several ranks may share a GPU in tests)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    nframes = args.warmup + args.steps
    poses, depths = make_frames(spec, nframes, dev)
    torch.cuda.synchronize()
    # a dedicated (non-default) stream: the engine's kernels and the timing
    # events must share it (torch's default stream has handle 0)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)

    # sizing pass: learn the arena sizes the capacity guards ask for, so no
    # frame in the timed region has to grow an arena and resume
    probe = Engine(RunConfig(strategy=args.strategy, **cfg, **ekw), spec.intrinsics())
    for i in range(nframes):
        probe.fuse_frame(depths[i], poses[i])
    pc = probe.store._counters()
    # vertex records: what the scene ends with + k_retype_place's per-frame bound
    # (2187 per scope item) + the gc CTAs' record ranges (4 chunks per CTA, <= 4096 CTAs)
    max_items = max(d["scope_blocks"] for d in probe.device_stats)
    caps = dict(block_capacity=pc["block_count"] + 64,
                vertex_capacity=pc["vertex_records"] + 2187 * max_items + 4 * 64 * 4096 + 4096)
    del probe

    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.int32, device=dev)

    def timed_pass(profiling: bool):
        """warmup + steps frames on a fresh engine, each step timed with CUDA
        events on the engine's stream, L2 flushed between steps.  Halo
        exchange: each step is PartitionedEngine.fuse_frame (begin, the
        all-gather of boundary blocks, finish, the StatsRow all-reduce)."""
        if xchg:
            pe = PartitionedEngine(RunConfig(strategy=args.strategy, **cfg, **caps), spec.intrinsics(),
                                   tile_blocks=args.tile_blocks, device=dev, halo="exchange")
            pe.engine.set_stream(stream.cuda_stream)
            for i in range(args.warmup):
                pe.fuse_frame(depths[i], poses[i])
            dist.barrier()
            torch.cuda.synchronize()
            starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
            ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
            with PausedGC():
                for k in range(args.steps):
                    i = args.warmup + k
                    flush.zero_()
                    starts[k].record(stream)
                    pe.fuse_frame(depths[i], poses[i])
                    ends[k].record(stream)
                torch.cuda.synchronize()
            return pe.engine, [s.elapsed_time(e) for s, e in zip(starts, ends)], [], 0
        eng = Engine(RunConfig(strategy=args.strategy, **cfg, **caps, **ekw), spec.intrinsics())
        eng.set_stream(stream.cuda_stream)
        eng.set_profiling(profiling)
        for i in range(args.warmup):
            eng.fuse_frame(depths[i], poses[i])
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        phases, resumes = [], 0
        with PausedGC():
            for k in range(args.steps):
                i = args.warmup + k
                flush.zero_()
                starts[k].record(stream)
                eng.fuse_frame_enqueue(depths[i], poses[i])
                ends[k].record(stream)
                eng.fuse_frame_finish()
                resumes += eng.device_stats[-1]["resumes"]
                if profiling:
                    phases.append(eng.phase_times())
            torch.cuda.synchronize()
        return eng, [s.elapsed_time(e) for s, e in zip(starts, ends)], phases, resumes

    overlapped = [0]

    def timed_stream():
        """`value`: the steps as one back-to-back stream (a live sensor's
        frames), pipelined submission of device-resident depth, one event
        before the first and one after the last step -- so frame t+1's
        k_collect runs under frame t's k_gc_normals (frame overlap).  No L2
        flush: every step reads its own 2.46 MB depth frame (the 295 timed
        frames are 725 MB of input, > the 126 MB L2); the store is the
        persistent state a stream keeps hot."""
        # (the engine's own stream: frame overlap needs the stream to itself)
        eng = Engine(RunConfig(strategy=args.strategy, **cfg, **caps, **ekw), spec.intrinsics(), pipelined=True)
        est = torch.cuda.ExternalStream(eng.stream_handle(), device=dev)
        for i in range(args.warmup):
            eng.fuse_frame(depths[i], poses[i])
        eng.stats[-1].blocks_active   # (complete the warm-up)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with PausedGC():
            t0.record(est)
            for k in range(args.steps):
                eng.fuse_frame(depths[args.warmup + k], poses[args.warmup + k])
            t1.record(est)   # (behind the last frame's kernels)
            eng.stats[-1].blocks_active
            torch.cuda.synchronize()
        resumes = sum(d["resumes"] for d in eng.device_stats[args.warmup:])
        overlapped[0] = sum(d["overlapped"] for d in eng.device_stats[args.warmup:])
        return eng, t0.elapsed_time(t1), resumes

    # timed region for `value`: no per-kernel events (an event between two
    # kernels would serialise their programmatic-dependent launch)
    # (every mode but the halo exchange, whose frames are synchronous around
    # their collectives, streams its frames: a partition rank's engine walks
    # the broadcast frames back to back like a single GPU's)
    stream_ms = None
    with ClockSampler(local_rank) as clocks:
        if not xchg:
            eng, stream_ms, resumes = timed_stream()
        eng_f, frame_ms, _, flushed_resumes = timed_pass(False)
        if xchg:
            eng, resumes = eng_f, flushed_resumes
        del eng_f
    # second pass on a fresh engine (same frames, same state evolution) with an
    # event before every kernel: per-kernel durations for the roofline
    _, prof_frame_ms, phase_ms, _ = timed_pass(True) if not xchg else (None, frame_ms, [], 0)
    flushed_s = sum(frame_ms) / 1e3   # per-frame, L2 flushed before each frame (no overlap)
    local_s = stream_ms / 1e3 if stream_ms is not None else flushed_s
    # partition: the ranks process the same frames jointly (strong scaling),
    # the job's time is the slowest rank's; replicas: N independent streams
    if part:
        # flushed per frame: a frame ends when its slowest rank ends
        flushed_dev_s = sum(reduce_(frame_ms, dist.ReduceOp.MAX)) / 1e3
        flushed_value = args.steps / flushed_dev_s
    else:
        flushed_dev_s = reduce_([flushed_s], dist.ReduceOp.MAX)[0] if world > 1 else flushed_s
        flushed_value = world * args.steps / flushed_dev_s
    if stream_ms is None:
        dev_s, value = flushed_dev_s, flushed_value
    else:
        dev_s = reduce_([local_s], dist.ReduceOp.MAX)[0] if world > 1 else local_s
        value = (1 if part else world) * args.steps / dev_s
    stats = eng.device_stats[args.warmup:]
    mc = eng.store._counters()   # HBM footprint of the final store
    memory = {"store_bytes": mc["store_bytes"], "blocks": mc["block_count"], "vertex_records": mc["vertex_records"],
              "bytes_per_cube": mc["store_bytes"] / max(1, 512 * mc["block_count"]),
              "bytes_per_block": mc["store_bytes"] / max(1, mc["block_count"]),
              "device_bytes_allocated": mc["device_bytes"], "paper_bytes_per_cube": 56}
    launches = sum(s["kernel_launches"] for s in stats)   # our kernels in the timed region

    # roofline: dominant kernel (largest share of the timed frames); the halo
    # exchange frame has no per-kernel events (its two halves are separate
    # calls around the collective): the frame as a whole
    peak, peak_kind = measured_peak_gbs()
    frame_bytes = sum(sum(phase_bytes(s, spec.height, spec.width).values()) for s in stats)
    if phase_ms:
        names = list(phase_ms[0].keys())
        tot = {n: sum(p[n] for p in phase_ms) for n in names}
        dom = max(names, key=lambda n: tot[n])
        bytes_dom = sum(phase_bytes(s, spec.height, spec.width)[dom] for s in stats)
        achieved = bytes_dom / (tot[dom] / 1e3) / 1e9
        kernel_share = tot[dom] / sum(tot.values())
    else:
        names, tot, dom = [], {}, "frame"
        bytes_dom, achieved, kernel_share = frame_bytes, frame_bytes / local_s / 1e9, 1.0
    traffic = None   # dram read+write bytes per launch of that kernel, from the committed ncu capture
    tp = ROOT / "profiles" / "ncu_traffic.json"
    if tp.exists():
        tj = json.loads(tp.read_text())
        traffic = tj.get("by_config", {}).get(args.config, tj.get("dram_bytes_per_launch", {}) if args.config == "C2"
                                              else {}).get(f"k_{dom}")

    # e2e: public API, pinned host depth, H2D + StatsRow D2H per frame, wall clock
    host = [torch.empty(d.shape, dtype=torch.float64, pin_memory=True) for d in depths]
    for hd, d in zip(host, depths):
        hd.copy_(d)
    host_np = [h.numpy() for h in host]
    if part:   # global StatsRow every frame: one NCCL all-reduce of the rank counters
        e2 = PartitionedEngine(RunConfig(strategy=args.strategy, **cfg, **caps), spec.intrinsics(),
                               tile_blocks=args.tile_blocks, device=dev, halo=args.halo)
    else:
        # pipelined submission (vm_fuse_frame_submit): the next frame's H2D copy
        # overlaps this frame's kernels; every frame's StatsRow is still read back
        e2 = Engine(RunConfig(strategy=args.strategy, **cfg, **caps), spec.intrinsics(), pipelined=True)
    for i in range(args.warmup):
        e2.fuse_frame(host_np[i], poses[i])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with PausedGC():
        t0 = time.perf_counter()
        for k in range(args.steps):
            e2.fuse_frame(host_np[args.warmup + k], poses[args.warmup + k])
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
    if world > 1:
        e2e_s = reduce_([e2e_s], dist.ReduceOp.MAX)[0]
    # parity spot check of the timed engine vs the e2e engine (same frames)
    e2_local = e2.engine if part else e2
    same = eng.stats[-1].vertices_live == e2_local.stats[-1].vertices_live
    glob = e2.stats[-1]
    # informational: the same frames as raw 16-bit depth images (read_depth's
    # format, scale 5000, i.e. quantised to 0.2 mm) through Engine.fuse_frame_raw
    # -- the device converts them, a quarter of the H2D bytes
    raw_e2e = None
    if not part:
        raws = [torch.from_numpy(np.clip(np.rint(h * 5000.0), 0, 65535).astype(np.uint16)).pin_memory().numpy()
                for h in host_np]
        e3 = Engine(RunConfig(strategy=args.strategy, **cfg, **caps), spec.intrinsics(), pipelined=True)
        for i in range(args.warmup):
            e3.fuse_frame_raw(raws[i], poses[i])
        torch.cuda.synchronize()
        with PausedGC():
            t0 = time.perf_counter()
            for k in range(args.steps):
                e3.fuse_frame_raw(raws[args.warmup + k], poses[args.warmup + k])
            torch.cuda.synchronize()
            raw_s = time.perf_counter() - t0
        e3.stats[-1].blocks_active   # (complete the last frame)
        raw_e2e = {"value": world * args.steps / raw_s, "unit": "frames/s",
                   "h2d_bytes_per_step": spec.width * spec.height * 2 + 256, "d2h_bytes_per_step": 512,
                   "input": "same frames quantised to u16 at depth_scale 5000 (read_depth format)"}
        del e3

    if rank != 0:
        return
    cpu = None
    parity = None
    if not args.no_cpu_baseline:
        hn = [d.cpu().numpy() for d in depths]
        n, t, ora = oracle_run(spec, cfg, hn, poses, budget_s=args.cpu_budget, return_engine=True)
        cpu = {"value": n / t, "unit": "frames/s", "cores": 1, "kind": "port",
               "sample": f"{args.config} frames 0..{n - 1} through the CPU oracle (serial C "
                         f"restatement of the reference, oracle/), {t:.1f} s"}
        # the published numbers' parity: the GPU engine on the same frames vs the oracle
        parity = parity_vs_oracle(spec, cfg, depths, poses, ora, n, args.strategy)
        del ora
        if args.pyref_budget > 0:
            cpu["python_reference"] = python_reference_legs(spec, cfg, hn, poses, args.pyref_budget)
    clk = clocks.summary()
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * dev_s / args.steps, "higher_is_better": True,
        "scaling": "strong" if part else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (sphere-traced analytic room, GPU-rendered f64 depth)",
        "config": workload(args, spec, cfg),
        "roofline": {"bound": "hbm", "kernel": f"k_{dom}", "achieved": achieved, "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "alg_bytes_per_launch": bytes_dom / args.steps, "kernel_share": kernel_share,
                     "frame_alg_bytes": frame_bytes / args.steps,
                     "frame_achieved_gbs": frame_bytes / local_s / 1e9,
                     "frame_frac": frame_bytes / local_s / 1e9 / peak},
        "phase_ms_mean": {n: tot[n] / args.steps for n in names},
        "value_l2_flushed": {"value": flushed_value,
                             "unit": "frames/s",
                             "how": "each frame timed alone (enqueue, events around it, L2 flushed by a 256 MiB "
                                    "write before it): no frame overlap, cold L2"},
        "profiled_pass_ms_per_step": sum(prof_frame_ms) / args.steps,
        "cpu_baseline": cpu,
        "parity": parity,
        "e2e": {"value": (1 if part else world) * args.steps / e2e_s, "unit": "frames/s",
                "h2d_bytes_per_step": spec.width * spec.height * 8 + 256,
                "d2h_bytes_per_step": 512},
        "e2e_raw_u16": raw_e2e,
        "gpu_launches": launches * world,
        "resumes_in_timed_region": resumes,
        "overlapped_frames": overlapped[0],
        "clocks": clk,
        "memory": memory,
        "final_state": {"blocks": glob.blocks_active, "vertices": glob.vertices_live,
                        "triangles": glob.triangles_live, "e2e_state_match": bool(same)},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=295)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--strategy", default="claim")
    ap.add_argument("--mode", default="partition", choices=["partition", "replicas"])
    ap.add_argument("--tile-blocks", type=int, default=8)
    ap.add_argument("--halo", default="margin", choices=["margin", "exchange"],
                    help="partition mode: margin blocks integrated locally, or received from their owners")
    ap.add_argument("--backend", default="nccl", help="gloo only to test N>1 on a single GPU")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--ref-budget", type=float, default=150.0)
    ap.add_argument("--pyref-budget", type=float, default=12.0,
                    help="seconds of the pure-Python reference per strategy (0 = skip)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    from paper_1803_03949_b200.synth import config_spec
    spec, cfg = config_spec(args.config)
    spec.frames = args.warmup + args.steps
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world > 1 and args.impl != "reference":
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank % torch.cuda.device_count())
        dist.init_process_group(args.backend)
    try:
        if args.impl == "reference":
            run_reference(args, spec, cfg, rank, world)
        else:
            run_gpu(args, spec, cfg, rank, world, local_rank)
    finally:
        if world > 1 and args.impl != "reference":
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
