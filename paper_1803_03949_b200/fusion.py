"""Per-frame block collection and TSDF integration (mirror of reference
pkg/src/voxmesh/fusion.py).

``collect_blocks`` and ``integrate_frame`` run the device kernels
``k_collect`` / ``k_integrate`` (csrc/vm_kernels.cuh) through the C ABI.
``Intrinsics``/``Pose``/``DepthFrame`` are plain host value types;
``truncate`` and ``block_in_frustum`` are small host helpers with the
reference's semantics (the engine evaluates the frustum test on the device
inside ``k_retype``).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .store import SpatialStore


@dataclass(frozen=True)
class Intrinsics:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def backproject(self, u, v):
        """Unit-depth camera-frame directions (x/z, y/z, 1) for pixels."""
        x = (np.asarray(u, dtype=np.float64) - self.cx) / self.fx
        y = (np.asarray(v, dtype=np.float64) - self.cy) / self.fy
        return np.stack([x, y, np.ones_like(x)], axis=-1)


@dataclass(frozen=True)
class Pose:
    """Sensor-to-world rigid transform."""

    rotation: np.ndarray
    translation: np.ndarray

    def transform(self, pts):
        return np.asarray(pts) @ self.rotation.T + self.translation

    def inverse_transform(self, pts):
        return (np.asarray(pts) - self.translation) @ self.rotation

    def inverse(self) -> "Pose":
        return Pose(self.rotation.T.copy(), -(self.rotation.T @ self.translation))

    @staticmethod
    def identity() -> "Pose":
        return Pose(np.eye(3), np.zeros(3))


@dataclass
class DepthFrame:
    pixels: np.ndarray   # (H, W) float64 metres, 0 = invalid
    frame_index: int = 0


def truncate(sdf_metric, trunc: float):
    """fusion.py:65-67: scale by the band and clamp to [-1, 1]."""
    return np.clip(np.asarray(sdf_metric, dtype=np.float64) / trunc, -1.0, 1.0)


def _depth(frame):
    d = frame.pixels if isinstance(frame, DepthFrame) else frame
    return np.ascontiguousarray(np.asarray(d, dtype=np.float64))


def collect_blocks(store: SpatialStore, frame, pose: Pose, intr: Intrinsics, trunc: float,
                   max_range: float = np.inf) -> list:
    """Allocate and return (sorted) the blocks touched by this frame's band."""
    d = _depth(frame)
    L = _lib.load()
    n = C.c_int64()
    store._touch()
    _lib.check(L.vm_collect(store._h, _lib.ptr(d), d.shape[0], d.shape[1], 0,
                            C.byref(_lib.intr_c(intr)), C.byref(_lib.pose_c(pose)),
                            float(trunc), float(max_range), C.byref(n)))
    out = np.zeros((n.value, 3), np.int32)
    if n.value:
        _lib.check(L.vm_get_collected(store._h, _lib.ptr(out), n.value))
    return sorted((int(a), int(b), int(c)) for a, b, c in out)


def integrate_frame(store: SpatialStore, blocks, frame, pose: Pose, intr: Intrinsics,
                    trunc: float, max_range: float = np.inf, weight_cap: int = 128) -> None:
    """Fold this frame's truncated distances into the given blocks (device)."""
    d = _depth(frame)
    c = _lib.coords_array(blocks)
    store._touch()
    _lib.check(_lib.load().vm_integrate(store._h, _lib.ptr(c), len(c), _lib.ptr(d), d.shape[0],
                                        d.shape[1], 0, C.byref(_lib.intr_c(intr)),
                                        C.byref(_lib.pose_c(pose)), float(trunc),
                                        float(max_range), int(weight_cap)))


def block_in_frustum(coord, pose: Pose, intr: Intrinsics, block_extent: float) -> bool:
    """fusion.py:171-190 conservative visibility test (host helper)."""
    base = np.array(coord, dtype=np.float64) * block_extent
    cam_pos = np.asarray(pose.translation, dtype=np.float64)
    if np.all(cam_pos >= base) and np.all(cam_pos <= base + block_extent):
        return True
    offs = np.array([[i, j, k] for i in (0, 1) for j in (0, 1) for k in (0, 1)], dtype=np.float64)
    cam = (base + offs * block_extent - cam_pos) @ np.asarray(pose.rotation)
    z = cam[:, 2]
    front = z > 0
    if not front.any():
        return False
    u = intr.fx * cam[front, 0] / z[front] + intr.cx
    v = intr.fy * cam[front, 1] / z[front] + intr.cy
    return bool(((u >= 0) & (u < intr.width) & (v >= 0) & (v < intr.height)).any())


def block_in_frustum_device(store: SpatialStore, coords, pose: Pose, intr: Intrinsics) -> np.ndarray:
    """The device evaluation used by the engine's frustum filter (k_retype)."""
    c = _lib.coords_array(coords)
    out = np.zeros(len(c), np.uint8)
    _lib.check(_lib.load().vm_block_in_frustum(store._h, _lib.ptr(c), len(c),
                                               C.byref(_lib.pose_c(pose)),
                                               C.byref(_lib.intr_c(intr)), _lib.ptr(out)))
    return out.astype(bool)
