"""Compact-vs-loose compare (reference cli.py:148-167, test_cli.py:117-125).

CPU: the reference's own compare.csv (tests/golden/make_compare_golden.py ran
``cmd_compare``) is reproduced byte for byte from the golden StatsRows.
GPU: the same file from the CUDA engine's own StatsRows on the same frames.
"""
import numpy as np
import pytest

from conftest import GOLDEN, cfg_from_golden, load_golden
from paper_1803_03949_b200.compare import compare, compare_rows, summary_line, write_compare_csv
from paper_1803_03949_b200.engine import StatsRow

SCENES = ("sphere_orbit", "room_noise_refine")


def _rows_from_golden(g):
    return [StatsRow(*[int(v) for v in s], 0.0, 0.0, 0.0) for s in g["stats"]]


@pytest.mark.parametrize("name", SCENES)
def test_compare_csv_matches_reference_bytes(name, tmp_path):
    rows = compare_rows(_rows_from_golden(load_golden(name)))
    write_compare_csv(tmp_path / "compare.csv", rows)
    assert (tmp_path / "compare.csv").read_bytes() == (GOLDEN / f"compare_{name}.csv").read_bytes()
    for r in rows:   # test_cli.py:117-125
        assert r[3] == 3 * r[2]


def test_compare_empty_and_zero_triangles():
    assert summary_line([]) == "final: compact=0 loose=0 ratio=1.0000"
    rows = compare_rows([StatsRow(0, 1, 0, 0, 0, 0, 0, 0.0, 0.0, 0.0)])
    assert rows == [(0, 0, 0, 0, 1.0)]


@pytest.mark.gpu
@pytest.mark.parametrize("name", SCENES)
def test_compare_through_cuda_engine_matches_reference(name, tmp_path):
    from paper_1803_03949_b200 import Engine, Intrinsics, Pose, RunConfig
    g = load_golden(name)
    i6 = g["intr6"]
    intr = Intrinsics(float(i6[0]), float(i6[1]), float(i6[2]), float(i6[3]), int(i6[4]), int(i6[5]))
    eng = Engine(RunConfig(**cfg_from_golden(g)), intr)
    for d, r, t in zip(g["depth"], g["rot"], g["trans"]):
        eng.fuse_frame(np.ascontiguousarray(d), Pose(r, t))
    compare(eng, tmp_path)
    assert (tmp_path / "compare.csv").read_bytes() == (GOLDEN / f"compare_{name}.csv").read_bytes()
