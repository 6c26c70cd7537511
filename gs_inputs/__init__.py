"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no projection, blending, loss or
gradient). It only draws random numbers and lays them out, so that `oracle/`
and the CUDA path can both consume the same bytes without sharing code.

Recipe (stands in for the paper's Replica / TUM frames,
PAPER.md:204 — neither dataset is available here):
  numpy default_rng(seed) (PCG64), float64 draws in this order
    1. means      U(lo, hi)          [N, 3]
    2. log-scales N(-3, 0.5)         [N, 3]
    3. quaternion N(0, 1)            [N, 4], normalised (r, i, j, k)
    4. opacity    logit ~ N(0, 1)    [N]
    5. rgb        U(0, 1)            [N, 3]   (SH degree 0, "light")
  activated in float64 (exp, sigmoid), cast to float32, SoA rows [14][N]:
    0-2 mean xyz, 3-5 scale xyz (linear), 6-9 quat r,i,j,k, 10 opacity, 11-13 rgb.

Pose rule ("random pose inside" the room): camera centre
U([0.5,3.5]x[0.5,2.5]x[0.5,3.5]) m, yaw U[0, 2pi), pitch U[-15deg, 15deg],
roll 0, world y up, OpenCV camera axes (x right, y down, z forward);
viewmat = [R_cw^T | -R_cw^T c] (world -> camera, row-major 3x4).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

N_PARAM_ROWS = 14
ROW_MEAN, ROW_SCALE, ROW_QUAT, ROW_OPACITY, ROW_RGB = 0, 3, 6, 10, 11

ROOM_LO = (0.0, 0.0, 0.0)
ROOM_HI = (4.0, 3.0, 4.0)


@dataclasses.dataclass(frozen=True)
class Camera:
    """Pinhole intrinsics + render settings (host struct; mirrors gs_camera in include/gs.h)."""
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    znear: float = 0.2
    bg: tuple = (0.0, 0.0, 0.0)
    cov2d_dilation: float = 0.3

    def half(self) -> "Camera":
        """Half-resolution camera for coarse tracking."""
        return dataclasses.replace(
            self, fx=self.fx / 2, fy=self.fy / 2,
            cx=(self.cx + 0.5) / 2 - 0.5, cy=(self.cy + 0.5) / 2 - 0.5,
            width=self.width // 2, height=self.height // 2)


CAM_TINY = Camera(60.0, 60.0, 31.5, 23.5, 64, 48)
CAM_TUM = Camera(525.0, 525.0, 319.5, 239.5, 640, 480)
CAM_REPLICA = Camera(600.0, 600.0, 599.5, 339.5, 1200, 680)


def gaussians(n: int, seed: int, lo=ROOM_LO, hi=ROOM_HI) -> np.ndarray:
    """Seeded Gaussian parameters, float32 SoA [14][n] (activated values)."""
    rng = np.random.default_rng(seed)
    means = rng.uniform(np.asarray(lo, np.float64), np.asarray(hi, np.float64), size=(n, 3))
    log_scales = rng.normal(-3.0, 0.5, size=(n, 3))
    quats = rng.normal(0.0, 1.0, size=(n, 4))
    quats /= np.linalg.norm(quats, axis=1, keepdims=True)
    logits = rng.normal(0.0, 1.0, size=n)
    rgb = rng.uniform(0.0, 1.0, size=(n, 3))
    out = np.empty((N_PARAM_ROWS, n), np.float64)
    out[0:3] = means.T
    out[3:6] = np.exp(log_scales).T
    out[6:10] = quats.T
    out[10] = 1.0 / (1.0 + np.exp(-logits))
    out[11:14] = rgb.T
    return out.astype(np.float32)


def room_surface_gaussians(n: int, seed: int, lo=ROOM_LO, hi=ROOM_HI) -> np.ndarray:
    """Seeded surface-like room (stands in for a Replica map, whose Gaussians sit on surfaces):
    n flat Gaussians on the 6 faces of the room box (face chosen by area), in-plane log-scales
    N(log 0.02, 0.3), normal scale 2 mm, axis-aligned (identity rotation), opacity sigmoid(N(2, 0.5)),
    colour a smooth seeded texture of position. float32 SoA [14][n] (activated)."""
    rng = np.random.default_rng(seed)
    lo = np.asarray(lo, np.float64)
    hi = np.asarray(hi, np.float64)
    ext = hi - lo
    faces = [(a, s) for a in range(3) for s in (0, 1)]   # normal axis, low/high side
    area = np.array([np.prod(np.delete(ext, a)) for a, _ in faces])
    f = rng.choice(len(faces), size=n, p=area / area.sum())
    pos = lo + rng.uniform(size=(n, 3)) * ext
    scale = np.exp(rng.normal(np.log(0.02), 0.3, size=(n, 3)))
    for k, (a, s) in enumerate(faces):
        sel = f == k
        pos[sel, a] = hi[a] if s else lo[a]
        scale[sel, a] = 0.002
    logits = rng.normal(2.0, 0.5, size=n)
    freq = rng.uniform(1.0, 4.0, size=(3, 3))
    phase = rng.uniform(0, 2 * math.pi, size=3)
    rgb = 0.5 + 0.45 * np.sin(pos @ freq.T + phase)
    out = np.zeros((N_PARAM_ROWS, n), np.float64)
    out[0:3] = pos.T
    out[3:6] = scale.T
    out[6] = 1.0
    out[10] = 1.0 / (1.0 + np.exp(-logits))
    out[11:14] = rgb.T
    return out.astype(np.float32)


def sh_coefficients(n: int, seed: int, lin: float = 0.3) -> np.ndarray:
    """Degree-1 SH inputs: [12][n] fp32 draws, row 3k + c = coefficient k of
    channel c; constant terms N(0, 1), linear terms N(0, lin). Appended to rows 0-10 of a scene they
    give the [23][n] layout of gs_project_sh."""
    rng = np.random.default_rng(seed)
    out = np.empty((12, n), np.float64)
    out[0:3] = rng.normal(0.0, 1.0, (3, n))
    out[3:12] = rng.normal(0.0, lin, (9, n))
    return out.astype(np.float32)


def with_sh(params: np.ndarray, seed: int, lin: float = 0.3) -> np.ndarray:
    """Rows 0-10 of `params` (geometry, opacity) + seeded degree-1 SH coefficients -> [23][n]."""
    return np.concatenate([params[:11], sh_coefficients(params.shape[1], seed, lin)]).astype(np.float32)


def identity_view() -> np.ndarray:
    v = np.zeros((3, 4), np.float32)
    v[0, 0] = v[1, 1] = v[2, 2] = 1.0
    return v


def look_view(centre, yaw: float, pitch: float) -> np.ndarray:
    """World->camera 3x4 for a camera at `centre` looking along (yaw, pitch), roll 0."""
    c = np.asarray(centre, np.float64)
    f = np.array([math.cos(pitch) * math.sin(yaw), math.sin(pitch), math.cos(pitch) * math.cos(yaw)])
    up = np.array([0.0, 1.0, 0.0])
    r = np.cross(f, up)
    r /= np.linalg.norm(r)
    d = np.cross(f, r)
    r_cw = np.stack([r, d, f], axis=1)  # columns = camera axes in world
    v = np.empty((3, 4), np.float64)
    v[:, :3] = r_cw.T
    v[:, 3] = -r_cw.T @ c
    return v.astype(np.float32)


def room_view(pose_seed: int) -> np.ndarray:
    rng = np.random.default_rng(pose_seed)
    centre = rng.uniform([0.5, 0.5, 0.5], [3.5, 2.5, 3.5])
    yaw = rng.uniform(0.0, 2.0 * math.pi)
    pitch = rng.uniform(-math.radians(15.0), math.radians(15.0))
    return look_view(centre, yaw, pitch)


def upstream(width: int, height: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """dL/dC [3][H][W] and dL/dD [H][W] ~ N(0, 1), float32 (config 0)."""
    rng = np.random.default_rng(seed)
    dc = rng.normal(0.0, 1.0, size=(3, height, width)).astype(np.float32)
    dd = rng.normal(0.0, 1.0, size=(height, width)).astype(np.float32)
    return dc, dd


def random_images(width: int, height: int, seed: int, depth_lo=0.5, depth_hi=4.0,
                  invalid_frac=0.05) -> tuple[np.ndarray, np.ndarray]:
    """Seeded RGB-D target: colour U(0,1) [3][H][W], depth U(lo,hi) [H][W] with a
    fraction of invalid (0) depths (stands in for sensor holes)."""
    rng = np.random.default_rng(seed)
    c = rng.uniform(0.0, 1.0, size=(3, height, width)).astype(np.float32)
    d = rng.uniform(depth_lo, depth_hi, size=(height, width))
    d[rng.uniform(size=(height, width)) < invalid_frac] = 0.0
    return c, d.astype(np.float32)


def twist_perturbation(seed: int, trans_m: float = 0.02, rot_deg: float = 1.0) -> np.ndarray:
    """(rho, phi) with |rho| = trans_m and |phi| = rot_deg, uniform directions (config 3)."""
    rng = np.random.default_rng(seed)
    a = rng.normal(size=3)
    b = rng.normal(size=3)
    rho = a / np.linalg.norm(a) * trans_m
    phi = b / np.linalg.norm(b) * math.radians(rot_deg)
    return np.concatenate([rho, phi])


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n: int
    scene_seed: int
    cam: Camera
    pose_seed: int | None          # None -> identity pose
    target_seed: int | None        # scene seed rendered as the target
    lo: tuple = ROOM_LO
    hi: tuple = ROOM_HI
    w_color: float = 0.9
    w_depth: float = 0.1

    def scene(self) -> np.ndarray:
        return gaussians(self.n, self.scene_seed, self.lo, self.hi)

    def view(self) -> np.ndarray:
        return identity_view() if self.pose_seed is None else room_view(self.pose_seed)


CONFIGS = {
    0: Config("tiny", 1000, 0, CAM_TINY, None, None, lo=(-1.0, -0.75, 1.0), hi=(1.0, 0.75, 5.0)),
    1: Config("tum", 100_000, 1, CAM_TUM, 101, 2),
    2: Config("replica", 500_000, 3, CAM_REPLICA, 103, 4),
    3: Config("tracking", 500_000, 3, CAM_REPLICA, 103, None),
    4: Config("mapping", 2_000_000, 5, CAM_REPLICA, 201, 6),
}
UPSTREAM_SEED_CFG0 = 1000
TRACK_PERTURB_SEED = 105
MAPPING_POSE_SEEDS = tuple(range(201, 209))
