"""Compact-vs-loose vertex comparison.

The reference's ``voxmesh compare`` (pkg/src/voxmesh/cli.py:148-167) runs a
reconstruction and reports, per frame, the shared-vertex mesh (the paper's
"compact" representation: each cube owns its 3 edges, so a vertex is stored
once) against a no-sharing baseline of 3 vertices per triangle.  Everything it
needs is in the per-frame ``StatsRow`` the engine already returns (the device
counters of ``k_gc_normals``' commit), so this is host arithmetic over those
rows, with the reference's CSV layout and rounding.
"""
from __future__ import annotations

import csv
from pathlib import Path
from typing import Iterable, List, Sequence, Tuple

from .engine import StatsRow

CompareRow = Tuple[int, int, int, int, float]
HEADER = ("frame", "vertices_compact", "triangles", "vertices_loose", "ratio")


def compare_rows(stats: Iterable[StatsRow]) -> List[CompareRow]:
    """Per frame: (frame, compact vertices, triangles, loose = 3 * triangles,
    compact / loose, 1.0 for an empty mesh) -- cli.py:154-157."""
    rows: List[CompareRow] = []
    for r in stats:
        loose = 3 * r.triangles_live
        rows.append((r.frame, r.vertices_live, r.triangles_live, loose,
                     (r.vertices_live / loose) if loose else 1.0))
    return rows


def write_compare_csv(path: Path, rows: Sequence[CompareRow]) -> None:
    """compare.csv exactly as cli.py:158-163 writes it."""
    with open(path, "w", encoding="utf-8", newline="") as f:
        w = csv.writer(f, lineterminator="\n")
        w.writerow(list(HEADER))
        w.writerows(rows)


def summary_line(rows: Sequence[CompareRow]) -> str:
    """The reference's closing line (cli.py:164-165)."""
    final = rows[-1] if rows else (0, 0, 0, 0, 1.0)
    return f"final: compact={final[1]} loose={final[3]} ratio={final[4]:.4f}"


def compare(engine, out: Path) -> List[CompareRow]:
    """Write ``out/compare.csv`` for an engine's frames so far and return the rows."""
    out = Path(out)
    out.mkdir(parents=True, exist_ok=True)
    rows = compare_rows(engine.stats)
    write_compare_csv(out / "compare.csv", rows)
    return rows
