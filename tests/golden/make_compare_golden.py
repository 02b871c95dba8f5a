"""Golden compare.csv files made by the REFERENCE's own ``cmd_compare``
(pkg/src/voxmesh/cli.py:148-167), run on the frames of existing golden scenes.

Run in the builder container only (needs the reference):

    python tests/golden/make_compare_golden.py [/root/reference/pkg/src]

``_run_reconstruction`` (cli.py:116-130) is replaced by a reference Engine fed
the golden scene's f64 frames (the dataset loader reads PGM files, whose u16
quantisation the golden frames do not have); everything after it is the
reference's code path.  Output: ``compare_<scene>.csv`` next to this script.
"""
from __future__ import annotations

import sys
import types
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SCENES = ("sphere_orbit", "room_noise_refine")


def main(src: str) -> None:
    sys.path.insert(0, src)
    import voxmesh
    from voxmesh import cli

    for name in SCENES:
        with np.load(HERE / f"{name}.npz") as z:
            g = {k: z[k] for k in z.files}
        c = g["cfg"]
        i6 = g["intr6"]
        intr = voxmesh.Intrinsics(fx=float(i6[0]), fy=float(i6[1]), cx=float(i6[2]), cy=float(i6[3]),
                                  width=int(i6[4]), height=int(i6[5]))

        def fake_run(config, dataset_dir, depth_scale, progress=True, g=g, intr=intr):
            eng = voxmesh.Engine(config, intr)
            for d, r, t in zip(g["depth"], g["rot"], g["trans"]):
                eng.fuse_frame(d, voxmesh.Pose(r, t))
            return eng

        cli._run_reconstruction = fake_run
        out = HERE / f"_cmp_{name}"
        args = types.SimpleNamespace(
            cube_size=float(c[0]), trunc=float(c[1]), epsilon=float(c[2]), refine=bool(c[3]),
            strategy="serial", baseline=False, max_range=float(c[4]), frustum_only=bool(c[5]),
            workers=1, seed=0, out=out, dataset=Path("."), depth_scale=1000.0)
        cli._write_manifest = lambda *a, **k: None
        assert cli.cmd_compare(args) == 0
        (HERE / f"compare_{name}.csv").write_bytes((out / "compare.csv").read_bytes())
        (out / "compare.csv").unlink()
        out.rmdir()
        print(name, "->", HERE / f"compare_{name}.csv")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src")
