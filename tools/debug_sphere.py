"""Debug aid: analytic-sphere extract on the GPU vs the CPU oracle, first diffs."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from oracle.oracle import OracleStore
from paper_1803_03949_b200 import SpatialStore
from paper_1803_03949_b200.mesher import extract_frame

B = 8
r, l = 0.25, 0.025
ext = l * B
n = int(np.ceil((r + 6 * l) / ext)) + 1
grid = np.stack(np.meshgrid(*[np.arange(B)] * 3, indexing="ij"), axis=-1).reshape(-1, 3)
coords, fields = [], []
for bx in range(-n, n + 1):
    for by in range(-n, n + 1):
        for bz in range(-n, n + 1):
            ctr = (np.array([bx, by, bz]) + 0.5) * ext
            if abs(np.linalg.norm(ctr) - r) < ext * 1.4:
                pts = (np.array([bx, by, bz]) * B + grid) * l
                coords.append((bx, by, bz))
                fields.append(np.clip((np.linalg.norm(pts, axis=1) - r) / (3 * l), -1, 1))
print("blocks", len(coords))
st = SpatialStore(cube_size=l)
st.set_block_samples(coords, np.stack(fields), np.ones((len(coords), 8, 8, 8), np.int32))
o = OracleStore(l)
for c, f in zip(coords, fields):
    o.set_block(c, f, np.ones(512, np.int32))
sc = sorted(coords)
extract_frame(st, [(c, None) for c in sc], 0)
o.extract(sc, None, o.scope_halo(sc)[2], 0)
snap = o.snapshot_blocks()
blocks = list(st.blocks())
gc = np.array([b.coord for b in blocks])
print("coords equal", np.array_equal(gc, snap["coords"]))
for k in ("tsdf", "weight", "type_prev", "type_curr"):
    g = np.stack([getattr(b, k) for b in blocks])
    bad = np.argwhere(g != snap[k])
    print(k, "mismatches", len(bad), bad[:5].tolist())
ev = np.stack([b.edge_vertex for b in blocks]) >= 0
oev = snap["edge_vertex"] >= 0
bad = np.argwhere(ev != oev)
print("slot occupancy mismatches", len(bad), bad[:8].tolist())
for b in bad[:8]:
    print("  block", gc[b[0]], "local", b[1:4], "axis", b[4], "gpu", ev[tuple(b)], "oracle", oev[tuple(b)])
m = st.compact_mesh()
pos, nrm, ages, idx = o.compact()
print("V", len(m.positions), len(pos), "T", len(m.indices), len(idx))
print("indices equal", np.array_equal(m.indices, idx), "pos equal", np.array_equal(m.positions, pos))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from conftest import edge_use_counts
for trial in range(6):
    st2 = SpatialStore(cube_size=l)
    st2.set_block_samples(coords, np.stack(fields), np.ones((len(coords), 8, 8, 8), np.int32))
    extract_frame(st2, [(c, None) for c in st2.block_coords()], 0)
    m2 = st2.compact_mesh()
    cnt = edge_use_counts(m2.indices)
    print("trial", trial, "nonmanifold", sum(1 for v in cnt.values() if v != 2), "V", len(m2.positions), "T", len(m2.indices),
          "idx==oracle", np.array_equal(m2.indices, idx))
