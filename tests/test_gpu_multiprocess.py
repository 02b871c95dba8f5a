"""Multi-process partitioned reconstruction on the one B200 of the test box:
2 ranks launched by torch.distributed.run (gloo backend -- NCCL does not run
two ranks on one device), PartitionedEngine end to end: the per-frame
all-reduce of the StatsRow counters, the halo exchange of boundary blocks
(all-gather of the owners' records) and the distributed compaction (gathered
owned-block metadata, k-way merge by key, per-rank fills summed).  Checked
against the reference's golden fixtures and against the CPU oracle at C2.
Also runs bench.py --gpus 2 --backend gloo under torchrun."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
NORMAL_ATOL = 1e-12


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torchrun(script_args, nproc=2, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", f"--master-port={_port()}"] + script_args
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout,
                       env=dict(os.environ, OMP_NUM_THREADS="1"))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return r


@pytest.mark.parametrize("halo", ["margin", "exchange", "exchange-shard"])
@pytest.mark.parametrize("name", ["room_noise_refine", "gc_carve"])
def test_two_process_partition_matches_reference_golden(tmp_path, name, halo):
    out = tmp_path / "r.npz"
    _torchrun(["tests/mp_partition_worker.py", "--scene", name, "--halo", halo, "--tile-blocks", "1",
               "--out", str(out)])
    g = load_golden(name)
    z = np.load(out)
    assert np.array_equal(z["rows"], g["stats"][:, :7].astype(np.int64))
    assert np.array_equal(z["indices"], g["m_indices"])
    assert np.array_equal(z["positions"], g["m_positions"])
    assert np.array_equal(z["ages"], g["m_ages"])
    assert np.allclose(z["normals"], g["m_normals"], rtol=0, atol=NORMAL_ATOL)
    if halo != "margin":
        assert z["sent"].sum() > 0


@pytest.mark.slow
@pytest.mark.parametrize("halo", ["margin", "exchange", "exchange-shard"])
def test_two_process_partition_c2_matches_oracle(tmp_path, halo):
    import torch
    from oracle.oracle import OracleEngine
    from oracle.parity import stats_tuple_oracle
    from paper_1803_03949_b200.synth import camera_pose, config_spec, render_depth_torch
    n = 12
    out = tmp_path / "r.npz"
    _torchrun(["tests/mp_partition_worker.py", "--scene", "C2", "--frames", str(n), "--halo", halo,
               "--tile-blocks", "8", "--out", str(out)])
    spec, cfg = config_spec("C2")
    intr = spec.intrinsics()
    ora = OracleEngine(cfg, (intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height))
    rows = []
    for i in range(n):
        p = camera_pose(spec, i)
        d = render_depth_torch(spec, p)
        torch.cuda.synchronize()
        rows.append(stats_tuple_oracle(ora.fuse_frame(d.cpu().numpy(), p.rotation, p.translation)))
    z = np.load(out)
    assert [tuple(r) for r in z["rows"].tolist()] == rows
    pos, nrm, ages, idx = ora.compact()
    assert np.array_equal(z["indices"], idx)
    assert np.array_equal(z["positions"], pos)
    assert np.array_equal(z["ages"], ages)
    assert np.allclose(z["normals"], nrm, rtol=0, atol=NORMAL_ATOL)


@pytest.mark.parametrize("halo", ["margin", "exchange"])
def test_bench_two_ranks_gloo_runs(halo):
    """bench.py's multi-GPU arm (spatial partition, strong scaling) under
    torchrun with 2 ranks sharing the GPU: one JSON line from rank 0."""
    r = _torchrun(["bench.py", "--gpus", "2", "--backend", "gloo", "--steps", "6", "--warmup", "3",
                   "--no-cpu-baseline", "--halo", halo], timeout=900)
    line = json.loads([s for s in r.stdout.splitlines() if s.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["scaling"] == "strong"
    assert line["config"]["halo"] == halo
