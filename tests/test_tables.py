"""The kernels compute EDGE_MASK from the type bits (csrc/vm_device.cuh
edge_mask_of) instead of reading the table: the formula, restated here, equals
the packed table generated from the reference (mc_tables.py:79-112) for all
256 cube types."""
from paper_1803_03949_b200 import _tables_data as td


def edge_mask_of(t: int) -> int:   # csrc/vm_device.cuh: edge_mask_of
    x = t ^ (((t >> 1) & 0x77) | ((t << 3) & 0x88))
    return (x & 0xFF) | (((t ^ (t >> 4)) & 0xF) << 8)


def test_edge_mask_formula_matches_table():
    assert [edge_mask_of(t) for t in range(256)] == list(td.EDGE_MASK)


def test_edge_mask_formula_in_header():
    from pathlib import Path
    src = (Path(__file__).resolve().parents[1] / "paper_1803_03949_b200/csrc/vm_device.cuh").read_text()
    assert "t ^ (((t >> 1) & 0x77u) | ((t << 3) & 0x88u))" in src
    assert "(((t ^ (t >> 4)) & 0xFu) << 8)" in src
