"""Build the sm_100a shared library in-tree (used by __graft_entry__.build())."""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
SRC = PKG / "csrc" / "vm_engine.cu"
OUT = PKG / "libvoxmesh_b200.so"
DEPS = [SRC, PKG / "csrc" / "vm_kernels.cuh", PKG / "csrc" / "vm_device.cuh",
        PKG / "csrc" / "mc_tables.inc", ROOT / "include" / "voxmesh_b200.h"]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3",
              "--fmad=false",          # no implicit FMA contraction (numeric parity)
              "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-ldl"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and Path(c).exists():
            return c
    raise RuntimeError("nvcc not found")


TRACE_OUT = PKG / "libvoxmesh_b200_trace.so"


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> Path:
    """The product library; trace=True builds the diagnostics variant with the
    per-CTA phase timestamps compiled in (-DVM_TRACE, vm_set_trace)."""
    out = TRACE_OUT if trace else OUT
    if not force and out.exists() and all(out.stat().st_mtime >= d.stat().st_mtime for d in DEPS):
        return out
    tmp = out.with_suffix(".so.tmp")
    cmd = [nvcc(), *NVCC_FLAGS, *(["-DVM_TRACE"] if trace else []), "-o", str(tmp), str(SRC)]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force=True, verbose=True))
