"""Synthetic depth input (mirror of reference pkg/src/voxmesh/synth.py).

Analytic signed-distance scenes sphere-traced into z-depth frames along an
orbit.  This is the INPUT GENERATOR for tests and the benchmark, not part of
the meshing path.  ``render_depth`` is the numpy form (reference semantics:
128 steps, tolerance 1e-6, synth.py:147-179); ``render_depth_torch`` runs the
same march in float64 on a CUDA device so C2-size sequences (300 x 640x480)
are produced in seconds.  Extra scene kinds for the BASELINE.json configs:
``sphere_box`` (C1) and ``multiroom`` (C5).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .errors import InputError
from .fusion import Intrinsics, Pose

MARCH_TOL = 1e-6
MARCH_MAX_STEPS = 128


@dataclass
class SceneSpec:
    scene: str = "plane"           # plane | sphere | room | sphere_box | multiroom
    plane_normal: tuple = (0.0, 0.0, -1.0)
    plane_offset: float = -1.0
    sphere_center: tuple = (0.0, 0.0, 0.0)
    sphere_radius: float = 0.5
    sphere_inverted: bool = False
    room_center: tuple = (0.0, 0.0, 0.0)
    room_size: tuple = (4.0, 3.0, 2.5)
    orbit_radius: float = 1.0
    orbit_height: float = 0.0
    angular_step_deg: float = 6.0
    elevation_amp_deg: float = 0.0
    elevation_rings: int = 3
    look: str = "inward"
    target: tuple = (0.0, 0.0, 0.0)
    orbit_center: Optional[tuple] = None
    frames: int = 60
    width: int = 128
    height: int = 96
    fx: float = 100.0
    fy: float = 100.0
    cx: Optional[float] = None
    cy: Optional[float] = None
    max_depth: float = 10.0
    noise_sigma: float = 0.0
    seed: int = 0
    # multiroom: list of axis-aligned wall boxes (center, half extents)
    boxes: list = field(default_factory=list)

    def intrinsics(self) -> Intrinsics:
        cx = (self.width - 1) / 2.0 if self.cx is None else self.cx
        cy = (self.height - 1) / 2.0 if self.cy is None else self.cy
        return Intrinsics(self.fx, self.fy, cx, cy, self.width, self.height)


def _box_sdf(xp, pts, c, h):
    q = xp.abs(pts - c) - h
    if xp is np:
        return np.linalg.norm(np.maximum(q, 0.0), axis=-1) + np.minimum(q.max(axis=-1), 0.0)
    return (xp.linalg.vector_norm(xp.clamp(q, min=0.0), dim=-1)
            + xp.clamp(q.max(dim=-1).values, max=0.0))


def scene_sdf(spec: SceneSpec, pts, xp=np):
    """Exact signed distance; positive on the observable (free-space) side."""
    if spec.scene == "plane":
        n = np.asarray(spec.plane_normal, dtype=np.float64)
        n = n / np.linalg.norm(n)
        nn = xp.asarray(n) if xp is np else xp.tensor(n, dtype=pts.dtype, device=pts.device)
        return pts @ nn - spec.plane_offset
    if spec.scene == "sphere":
        c = _const(xp, spec.sphere_center, pts)
        d = _norm(xp, pts - c) - spec.sphere_radius
        return -d if spec.sphere_inverted else d
    if spec.scene in ("room", "sphere_box", "multiroom"):
        c = _const(xp, spec.room_center, pts)
        half = _const(xp, spec.room_size, pts) / 2.0
        r = half - xp.abs(pts - c)
        room = r.min(axis=-1) if xp is np else r.min(dim=-1).values
        if spec.scene == "room":
            return room
        if spec.scene == "sphere_box":
            sph = _norm(xp, pts - _const(xp, (0.9, 0.0, -0.4), pts)) - 0.4
            box = _box_sdf(xp, pts, _const(xp, (-0.8, 0.5, -0.6), pts), 0.25)
            return xp.minimum(room, xp.minimum(sph, box))
        out = room
        for bc, bh in spec.boxes:
            out = xp.minimum(out, _box_sdf(xp, pts, _const(xp, bc, pts), _const(xp, bh, pts)))
        return out
    raise InputError(f"unknown scene kind {spec.scene!r}")


def _const(xp, v, like):
    if xp is np:
        return np.asarray(v, dtype=np.float64)
    return xp.tensor(np.asarray(v, dtype=np.float64), dtype=like.dtype, device=like.device)


def _norm(xp, v):
    return np.linalg.norm(v, axis=-1) if xp is np else xp.linalg.vector_norm(v, dim=-1)


def tilted_plane_spec(tilt_deg: float, distance: float = 1.0, **kw) -> SceneSpec:
    t = math.radians(tilt_deg)
    return SceneSpec(scene="plane", plane_normal=(math.sin(t), 0.0, -math.cos(t)),
                     plane_offset=-(distance * math.cos(t)), **kw)


def _look_rotation(fwd):
    up = np.array([0.0, 0.0, -1.0])               # image v grows downwards
    if abs(fwd @ up) > 0.999:
        up = np.array([0.0, -1.0, 0.0])
    right = -np.cross(up, fwd)
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    return np.stack([right, down, fwd], axis=1)   # columns: camera x, y, z in world


def camera_pose(spec: SceneSpec, i: int) -> Pose:
    """Orbit pose of frame i (elevation cycles through rings, synth.py:94-130)."""
    theta = math.radians(spec.angular_step_deg) * i
    phi = 0.0
    if spec.elevation_amp_deg and spec.elevation_rings > 1:
        k = spec.elevation_rings
        phi = math.radians(spec.elevation_amp_deg) * (2.0 * (i % k) / (k - 1) - 1.0)
    target = np.asarray(spec.target, dtype=np.float64)
    center = target if spec.orbit_center is None else np.asarray(spec.orbit_center, np.float64)
    position = center + np.array([spec.orbit_radius * math.cos(theta) * math.cos(phi),
                                  spec.orbit_radius * math.sin(theta) * math.cos(phi),
                                  spec.orbit_height + spec.orbit_radius * math.sin(phi)])
    fwd = (target - position) if spec.look == "inward" else (position - target)
    n = np.linalg.norm(fwd)
    fwd = np.array([0.0, 0.0, 1.0]) if n < 1e-12 else fwd / n
    return Pose(_look_rotation(fwd), position)


def static_pose(position, look_at) -> Pose:
    position = np.asarray(position, dtype=np.float64)
    fwd = np.asarray(look_at, dtype=np.float64) - position
    return Pose(_look_rotation(fwd / np.linalg.norm(fwd)), position)


def _ray_dirs(intr: Intrinsics):
    u, v = np.meshgrid(np.arange(intr.width), np.arange(intr.height))
    d = intr.backproject(u, v).reshape(-1, 3)
    return d / np.linalg.norm(d, axis=1)[:, None]


def render_depth(spec: SceneSpec, pose: Pose, rng: Optional[np.random.Generator] = None):
    """Sphere-trace a z-depth image (metres; 0 where the march fails)."""
    intr = spec.intrinsics()
    dirs_cam = _ray_dirs(intr)
    dirs = dirs_cam @ pose.rotation.T
    t = np.zeros(len(dirs))
    live = np.ones(len(dirs), bool)
    hit = np.zeros(len(dirs), bool)
    for _ in range(MARCH_MAX_STEPS):
        idx = np.nonzero(live)[0]
        if idx.size == 0:
            break
        d = scene_sdf(spec, pose.translation + dirs[idx] * t[idx, None])
        close = d < MARCH_TOL
        hit[idx[close]] = True
        live[idx[close]] = False
        t[idx[~close]] += d[~close]
        live &= t <= spec.max_depth
    z = np.where(hit, t, 0.0) * dirs_cam[:, 2]
    if rng is not None and spec.noise_sigma > 0:
        z = np.where(z > 0, np.maximum(z + rng.normal(0.0, spec.noise_sigma, z.shape), 1e-4), 0.0)
    return z.reshape(intr.height, intr.width)


def render_depth_torch(spec: SceneSpec, pose: Pose, device="cuda", rng=None):
    """Same march in float64 on a torch device; returns a (H, W) float64 tensor."""
    import torch
    intr = spec.intrinsics()
    dirs_cam = torch.tensor(_ray_dirs(intr), dtype=torch.float64, device=device)
    rot = torch.tensor(pose.rotation, dtype=torch.float64, device=device)
    org = torch.tensor(pose.translation, dtype=torch.float64, device=device)
    dirs = dirs_cam @ rot.T
    t = torch.zeros(dirs.shape[0], dtype=torch.float64, device=device)
    live = torch.ones_like(t, dtype=torch.bool)
    hit = torch.zeros_like(live)
    for _ in range(MARCH_MAX_STEPS):
        d = scene_sdf(spec, org + dirs * t[:, None], xp=torch)
        close = (d < MARCH_TOL) & live
        hit |= close
        live &= ~close
        t = torch.where(live, t + d, t)
        live &= t <= spec.max_depth
    z = torch.where(hit, t, torch.zeros_like(t)) * dirs_cam[:, 2]
    if rng is not None and spec.noise_sigma > 0:
        noise = torch.tensor(rng.normal(0.0, spec.noise_sigma, z.shape[0]), dtype=torch.float64,
                             device=device)
        z = torch.where(z > 0, torch.clamp(z + noise, min=1e-4), torch.zeros_like(z))
    return z.reshape(intr.height, intr.width).contiguous()


def frame_poses(spec: SceneSpec) -> list:
    return [camera_pose(spec, i) for i in range(spec.frames)]


# ---------------------------------------------------------------- BASELINE configs
def config_spec(name: str) -> tuple:
    """(SceneSpec, RunConfig kwargs) of BASELINE.json configs C1..C5."""
    if name == "C1":
        spec = SceneSpec(scene="sphere_box", room_size=(3.0, 3.0, 2.0), orbit_radius=0.3,
                         look="outward", elevation_amp_deg=20.0, elevation_rings=3,
                         angular_step_deg=9.0, frames=20, width=320, height=240,
                         fx=262.5, fy=262.5)
        return spec, dict(cube_size=0.008, trunc=0.024)
    if name in ("C2", "C3", "C4"):
        spec = SceneSpec(scene="room", room_size=(4.0, 4.0, 2.5), orbit_radius=0.5,
                         look="outward", angular_step_deg=1.2, elevation_amp_deg=15.0,
                         elevation_rings=3, frames=300, width=640, height=480, fx=525.0, fy=525.0)
        if name == "C2":
            return spec, dict(cube_size=0.008, trunc=0.024)
        if name == "C3":
            return spec, dict(cube_size=0.008, trunc=0.024, refine=True, epsilon=0.1)
        return spec, dict(cube_size=0.004, trunc=0.04)
    if name == "C5":
        boxes = []
        for k in range(1, 4):            # interior walls on a 5 m grid with 1 m door gaps
            p = -10.0 + 5.0 * k
            for seg in ((-10.0, -6.0), (-5.0, -1.0), (0.0, 4.0), (5.0, 10.0)):
                c = (seg[0] + seg[1]) / 2.0
                h = (seg[1] - seg[0]) / 2.0
                boxes.append(((p, c, 0.0), (0.075, h, 1.5)))
                boxes.append(((c, p, 0.0), (h, 0.075, 1.5)))
        spec = SceneSpec(scene="multiroom", room_size=(20.0, 20.0, 3.0), boxes=boxes,
                         orbit_radius=0.0, frames=2000, width=640, height=480, fx=525.0, fy=525.0)
        return spec, dict(cube_size=0.008, trunc=0.024, table_size=1 << 21)
    raise KeyError(name)


def multiroom_pose(spec: SceneSpec, i: int) -> Pose:
    """C5 trajectory: the camera visits the 16 rooms of the 20x20 m floor in a
    serpentine order, 125 frames per room, circling 0.6 m around the room
    centre at 1.4 m above the floor while panning (two turns per room)."""
    room = (i // 125) % 16
    row, col = room // 4, room % 4
    if row % 2:
        col = 3 - col
    cx, cy = -7.5 + 5.0 * col, -7.5 + 5.0 * row
    ph = 2.0 * math.pi * (i % 125) / 125.0
    pos = np.array([cx + 0.6 * math.cos(ph), cy + 0.6 * math.sin(ph), -0.1])
    ang = 2.0 * ph + 0.3
    fwd = np.array([math.cos(ang), math.sin(ang), -0.2 + 0.15 * math.sin(3.0 * ph)])
    return static_pose(pos, pos + fwd)
