"""Worker of tests/test_gpu_multiprocess.py: one rank of a partitioned
reconstruction (PartitionedEngine over torch.distributed), launched by
torch.distributed.run.  Several ranks may share one GPU (gloo backend).
Rank 0 writes the global rows and the compacted mesh to --out (npz)."""
import argparse
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scene", required=True)          # golden scene name or a config (C2)
    ap.add_argument("--frames", type=int, default=0)
    ap.add_argument("--halo", default="margin")
    ap.add_argument("--tile-blocks", type=int, default=2)
    ap.add_argument("--backend", default="gloo")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    import faulthandler
    faulthandler.dump_traceback_later(120, exit=True)   # (a hung rank reports where, then exits)
    import torch
    import torch.distributed as dist
    from paper_1803_03949_b200 import Intrinsics, Pose, RunConfig
    from paper_1803_03949_b200.partition import PartitionedEngine
    rank = int(os.environ["RANK"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
    dist.init_process_group(a.backend)
    if a.scene.startswith("C"):
        from paper_1803_03949_b200.synth import camera_pose, config_spec, render_depth_torch
        spec, cfg = config_spec(a.scene)
        intr = spec.intrinsics()
        frames = [(render_depth_torch(spec, camera_pose(spec, i)), camera_pose(spec, i))
                  for i in range(a.frames)]
    else:
        from conftest import cfg_from_golden, load_golden
        g = load_golden(a.scene)
        cfg = cfg_from_golden(g)
        i6 = g["intr6"]
        intr = Intrinsics(float(i6[0]), float(i6[1]), float(i6[2]), float(i6[3]), int(i6[4]), int(i6[5]))
        frames = [(g["depth"][i], Pose(g["rot"][i], g["trans"][i])) for i in range(len(g["depth"]))]
    halo = "exchange" if a.halo.startswith("exchange") else a.halo
    pe = PartitionedEngine(RunConfig(**cfg), intr, tile_blocks=a.tile_blocks, halo=halo,
                           shard_band=a.halo == "exchange-shard")
    rows = []
    for d, p in frames:
        r = pe.fuse_frame(d, p)
        rows.append((r.frame, r.blocks_active, r.vertices_live, r.triangles_live,
                     r.vertices_allocated_total, r.vertices_recycled_total, r.irregular_cube_count))
    mesh = pe.compact()
    sent = np.asarray(pe.exchange_log, np.int64).reshape(-1, dist.get_world_size())
    if rank == 0:
        np.savez(a.out, rows=np.asarray(rows, np.int64), positions=mesh.positions, normals=mesh.normals,
                 ages=mesh.ages, indices=mesh.indices, sent=sent)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
