"""ORACLE — TEST INFRASTRUCTURE ONLY.

Plain CPU reference of the GS-SLAM RGB-D splatting renderer (arXiv 2311.11700). Only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl reference` legs may
import this package. It shares no code with `paper_2311_11700_b200` (neither imports the other).

  * projection, binning, forward, backward: `oracle.cpp` (C++17 + OpenMP, ctypes), O1-O4
  * loss, Adam, pose step, densify/prune/select: numpy fp64 below, O5

Parity unpinned: none of the functions here (each is pinned by tests/test_oracle_*.py; see
DESIGN.md §4 for the pin of every function).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.cpp")

GFLAGS = ["-O2", "-std=c++17", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC"]


def build(force: bool = False) -> str:
    """Compile liboracle.so (plain g++; no CUDA)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", *GFLAGS, _SRC, "-o", _SO])
    return _SO


class OracleCam(ctypes.Structure):
    _fields_ = [("fx", ctypes.c_double), ("fy", ctypes.c_double), ("cx", ctypes.c_double),
                ("cy", ctypes.c_double), ("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("znear", ctypes.c_double), ("bg", ctypes.c_double * 3), ("dil", ctypes.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
    return _lib


def _cam(cam) -> OracleCam:
    c = OracleCam()
    c.fx, c.fy, c.cx, c.cy = cam.fx, cam.fy, cam.cx, cam.cy
    c.width, c.height = cam.width, cam.height
    c.znear = cam.znear
    for k in range(3):
        c.bg[k] = cam.bg[k]
    c.dil = cam.cov2d_dilation
    return c


def _p(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def _dtype(precision: str):
    return {"f32": np.float32, "f64": np.float64}[precision]


def set_threads(n: int) -> None:
    lib().oracle_set_threads(ctypes.c_int(n))


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def grid(cam) -> tuple[int, int]:
    return (cam.width + 15) // 16, (cam.height + 15) // 16


def sh_degree_of(params) -> int:
    """Colour model from the parameter rows: 14 = RGB (reading C17), 23 = degree-1 SH (C29)."""
    rows = np.asarray(params).shape[0]
    if rows not in (14, 23):
        raise ValueError(f"params must have 14 or 23 rows, got {rows}")
    return 1 if rows == 23 else 0


def _mode(params, opacity_radius, o3_power=False) -> int:
    """Oracle C ABI mode word: colour model | (opacity-aware radius, reading C33) << 8 | (power in
    SURVEY.md §8(c) O3's printed order instead of reading R1's fma order) << 9."""
    return sh_degree_of(params) | (256 if opacity_radius else 0) | (512 if o3_power else 0)


# ------------------------------------------------------------------------------------ O1
def project(params, view, cam, precision="f32", opacity_radius=False) -> dict:
    """O1 (Eq. 2-3): per-Gaussian projection. params [14][n] (RGB) or [23][n] (degree-1 SH, C29),
    view [3][4]. rgb: the colour the blend uses (SH evaluated at the view direction).
    opacity_radius: reading C33's radius (the alpha >= 1/255 reach) instead of 3 sigma."""
    dt = _dtype(precision)
    params = np.ascontiguousarray(params, dt)
    view = np.ascontiguousarray(view, dt)
    n = params.shape[1]
    out = dict(mean2d=np.zeros((2, n), dt), conic=np.zeros((3, n), dt), depth=np.zeros(n, dt),
               radius=np.zeros(n, np.int32), rect=np.zeros((4, n), np.int32), tiles=np.zeros(n, np.uint32),
               depth_bits=np.zeros(n, np.uint32), cov2d=np.zeros((3, n), dt), rgb=np.zeros((3, n), dt))
    c = _cam(cam)
    fn = getattr(lib(), f"oracle_project_{precision}")
    fn(_p(params), ctypes.c_int64(n), ctypes.c_int64(n), _p(view), ctypes.byref(c), _p(out["mean2d"]),
       _p(out["conic"]), _p(out["depth"]), _p(out["radius"]), _p(out["rect"]), _p(out["tiles"]),
       _p(out["depth_bits"]), _p(out["cov2d"]), ctypes.c_int32(_mode(params, opacity_radius)), _p(out["rgb"]))
    return out


# ------------------------------------------------------------------------------------ O2
def bin_sort(depth_bits, rect, tiles, cam) -> dict:
    """O2: keys (tile<<32 | depth bits) emitted in index order, stable-sorted; per-tile ranges."""
    gx, gy = grid(cam)
    depth_bits = np.ascontiguousarray(depth_bits, np.uint32)
    rect = np.ascontiguousarray(rect, np.int32)
    tiles = np.ascontiguousarray(tiles, np.uint32)
    n = depth_bits.shape[0]
    k = int(tiles.astype(np.int64).sum())
    keys = np.zeros(k, np.uint64)
    vals = np.zeros(k, np.uint32)
    ranges = np.zeros((gx * gy, 2), np.uint32)
    got = lib().oracle_bin
    got.restype = ctypes.c_int64
    kk = got(_p(depth_bits), _p(rect), _p(tiles), ctypes.c_int64(n), ctypes.c_int32(gx), ctypes.c_int32(gy),
             _p(keys), _p(vals), _p(ranges), ctypes.c_int64(k))
    assert kk == k
    return dict(keys=keys, vals=vals, ranges=ranges, n_keys=k)


# ------------------------------------------------------------------------------------ O3
def forward(params, view, cam, precision="f32", pixels=None, replay_nlast=None, accum_weight=False,
            flip_skip_ties=False, opacity_radius=False, o3_power=False) -> dict:
    """O3 (Eq. 4-5, cumulative opacity P:118). Full images unless `pixels` (linear ids) given.
    replay_nlast / flip_skip_ties: the parity tie rule's replays (reading R1).
    o3_power: evaluate the exponent in the order SURVEY.md §8(c) O3 prints,
    -0.5*((a*dx)*dx + (c*dy)*dy) - (b*dx)*dy, instead of R1's fma order (for the pin that both
    orders take the same decisions outside the tie band)."""
    dt = _dtype(precision)
    params = np.ascontiguousarray(params, dt)
    view = np.ascontiguousarray(view, dt)
    n = params.shape[1]
    if pixels is not None:
        pixels = np.ascontiguousarray(pixels, np.int64)
        npx = pixels.shape[0]
        shape = (npx,)
    else:
        npx = cam.width * cam.height
        shape = (cam.height, cam.width)
    color = np.zeros((3, npx), np.float64)
    depth = np.zeros(npx, np.float64)
    alpha = np.zeros(npx, np.float64)
    n_last = np.zeros(npx, np.uint32)
    examined = np.zeros(npx, np.uint32)
    amb = np.zeros(npx, np.uint8)
    h = np.zeros(1, np.uint64)
    aw = np.zeros(n, np.float64) if accum_weight else None
    rp = np.ascontiguousarray(replay_nlast, np.uint32).reshape(-1) if replay_nlast is not None else None
    c = _cam(cam)
    getattr(lib(), f"oracle_forward_{precision}")(
        _p(params), ctypes.c_int64(n), ctypes.c_int64(n), _p(view), ctypes.byref(c), _p(pixels),
        ctypes.c_int64(npx), _p(rp), _p(color), _p(depth), _p(alpha), _p(n_last), _p(examined), _p(amb),
        _p(h), _p(aw), ctypes.c_int32(1 if flip_skip_ties else 0),
        ctypes.c_int32(_mode(params, opacity_radius, o3_power)))
    out = dict(color=color.reshape((3,) + shape), depth=depth.reshape(shape), alpha=alpha.reshape(shape),
               n_last=n_last.reshape(shape), examined=examined.reshape(shape), ambiguous=amb.reshape(shape),
               hash=int(h[0]))
    if accum_weight:
        out["accum_weight"] = aw
    return out


# ------------------------------------------------------------------------------------ O4
def backward(params, view, cam, dL_dcolor, dL_ddepth, precision="f32", replay_nlast=None, qt_cov=True,
             pixels=None, opacity_radius=False, bound=False) -> dict:
    """O4 (Eq. 11, S1-S6): fp64 gradients for the 14 (RGB) or 23 (degree-1 SH) params, screen grads,
    and the pose.

    pose_twist: (rho, phi) left-perturbation twist, covariance path included (reading C7);
    pose_twist_paper: same without the Sigma'-through-pose term (paper mode);
    pose_qt: dL/d(q_r,q_i,q_j,q_k,t) via Eq. S1/S3 (independent path), plus the pose quaternion.
    bound=True adds grad_bound [rows][n], pose_bound[6], pose_bound_paper[6], screen_bound [10][n]
    (the screen quantities' sums of term magnitudes), chain_scale [rows][n] (the per-Gaussian chain
    evaluated on magnitudes: the rounding scale of the chain itself): the error-bound scale
    of each result, sum_j |d grad / d s_j| sum_p |c_pj| (the per-pixel terms' magnitudes carried
    through the linear per-Gaussian chain; oracle.cpp error_bound). |result| <= bound always.
    """
    dt = _dtype(precision)
    params = np.ascontiguousarray(params, dt)
    view = np.ascontiguousarray(view, dt)
    n = params.shape[1]
    dc = np.ascontiguousarray(dL_dcolor, np.float32).reshape(-1)
    dd = np.ascontiguousarray(dL_ddepth, np.float32).reshape(-1)
    gp = np.zeros((params.shape[0], n), np.float64)
    gs = np.zeros((10, n), np.float64)
    tw = np.zeros(6, np.float64)
    twp = np.zeros(6, np.float64)
    qt = np.zeros(11, np.float64)
    rp = np.ascontiguousarray(replay_nlast, np.uint32).reshape(-1) if replay_nlast is not None else None
    px = np.ascontiguousarray(pixels, np.int64) if pixels is not None else None
    gb = np.zeros((params.shape[0], n), np.float64) if bound else None
    pb = np.zeros(6, np.float64) if bound else None
    pbp = np.zeros(6, np.float64) if bound else None
    sb = np.zeros((10, n), np.float64) if bound else None
    cs = np.zeros((params.shape[0], n), np.float64) if bound else None
    c = _cam(cam)
    getattr(lib(), f"oracle_backward_{precision}")(
        _p(params), ctypes.c_int64(n), ctypes.c_int64(n), _p(view), ctypes.byref(c), _p(dc), _p(dd), _p(rp),
        _p(gp), _p(gs), _p(tw), _p(twp), _p(qt), ctypes.c_int32(1 if qt_cov else 0), _p(px),
        ctypes.c_int64(0 if px is None else px.shape[0]), ctypes.c_int32(_mode(params, opacity_radius)),
        _p(gb), _p(pb), _p(pbp), _p(sb), _p(cs))
    out = dict(grad_params=gp, grad_screen=gs, pose_twist=tw, pose_twist_paper=twp,
               pose_q=qt[0:4], pose_t=qt[4:7], pose_quat=qt[7:11])
    if bound:
        out.update(grad_bound=gb, pose_bound=pb, pose_bound_paper=pbp, screen_bound=sb, chain_scale=cs)
    return out


# ------------------------------------------------------------------------------------ O5 (numpy fp64)
def loss_l1(color, depth, tgt_color, tgt_depth, w_color=0.9, w_depth=0.1) -> dict:
    """Eq. 6 as means (reading C20): L = w_c/(3HW) sum|C-C*| + w_d/#valid sum_valid|D-D*|.
    dL/dC = w_c/(3HW) sign(C-C*), sign(0)=0; dL/dD likewise over valid pixels (D* > 0)."""
    c = np.asarray(color, np.float64)
    d = np.asarray(depth, np.float64)
    tc = np.asarray(tgt_color, np.float64)
    td = np.asarray(tgt_depth, np.float64)
    h, w = d.shape
    valid = td > 0
    nvalid = int(valid.sum())
    sc = w_color / (3.0 * h * w)
    sd = w_depth / nvalid if nvalid > 0 else 0.0
    loss = sc * np.abs(c - tc).sum() + sd * np.abs(d - td)[valid].sum()
    return dict(loss=loss, dL_dcolor=sc * np.sign(c - tc), dL_ddepth=sd * np.sign(d - td) * valid, n_valid=nvalid)


RAW_ACT = ("id",) * 3 + ("exp",) * 3 + ("id",) * 4 + ("sigmoid",) + ("id",) * 3


def activate(raw) -> np.ndarray:
    """Raw (log-scale, logit-opacity) -> activated parameters (reading C18)."""
    raw = np.asarray(raw, np.float64)
    act = raw.copy()
    act[3:6] = np.exp(raw[3:6])
    act[10] = 1.0 / (1.0 + np.exp(-raw[10]))
    return act


def adam_step(raw, grad_act, m, v, lr, step, b1=0.9, b2=0.999, eps=1e-8) -> dict:
    """Textbook Adam (betas/eps unstated -> 0.9/0.999/1e-8) in raw space with the
    activation chain rule: d/dlog s = s d/ds, d/dlogit o = o(1-o) d/do. lr: one rate per row (14
    rows, or 23 for the degree-1 SH layout, whose extra rows are identity-activated)."""
    raw = np.asarray(raw, np.float64)
    g = np.asarray(grad_act, np.float64).copy()
    act = activate(raw)
    g[3:6] *= act[3:6]
    g[10] *= act[10] * (1.0 - act[10])
    m = b1 * np.asarray(m, np.float64) + (1 - b1) * g
    v = b2 * np.asarray(v, np.float64) + (1 - b2) * g * g
    mh = m / (1 - b1 ** step)
    vh = v / (1 - b2 ** step)
    lr = np.asarray(lr, np.float64).reshape(raw.shape[0], 1)
    new_raw = raw - lr * mh / (np.sqrt(vh) + eps)
    return dict(raw=new_raw, act=activate(new_raw), m=m, v=v)


def skew(w):
    return np.array([[0.0, -w[2], w[1]], [w[2], 0.0, -w[0]], [-w[1], w[0], 0.0]])


def se3_exp(delta) -> np.ndarray:
    """exp of the twist (rho, phi) as a 3x4 [R | t] (Rodrigues; V(phi) rho)."""
    rho = np.asarray(delta[:3], np.float64)
    phi = np.asarray(delta[3:], np.float64)
    th = float(np.linalg.norm(phi))
    K = skew(phi)
    if th < 1e-12:
        R = np.eye(3) + K
        V = np.eye(3) + 0.5 * K
    else:
        R = np.eye(3) + math.sin(th) / th * K + (1 - math.cos(th)) / th ** 2 * K @ K
        V = np.eye(3) + (1 - math.cos(th)) / th ** 2 * K + (th - math.sin(th)) / th ** 3 * K @ K
    out = np.empty((3, 4))
    out[:, :3] = R
    out[:, 3] = V @ rho
    return out


def apply_twist(delta, view) -> np.ndarray:
    """Left perturbation T <- exp(delta^) T of a world->camera 3x4 (DESIGN.md pose convention)."""
    e = se3_exp(delta)
    v = np.asarray(view, np.float64)
    out = np.empty((3, 4))
    out[:, :3] = e[:, :3] @ v[:, :3]
    out[:, 3] = e[:, :3] @ v[:, 3] + e[:, 3]
    return out


def pose_adam_step(view, grad_twist, m6, v6, step, lr_rho, lr_phi, b1=0.9, b2=0.999, eps=1e-8) -> dict:
    """Adam on the twist (reading C23), then T <- exp(delta^) T ("FusedAdam" on the pose)."""
    g = np.asarray(grad_twist, np.float64)
    m6 = b1 * np.asarray(m6, np.float64) + (1 - b1) * g
    v6 = b2 * np.asarray(v6, np.float64) + (1 - b2) * g * g
    mh = m6 / (1 - b1 ** step)
    vh = v6 / (1 - b2 ** step)
    lr = np.array([lr_rho] * 3 + [lr_phi] * 3)
    delta = -lr * mh / (np.sqrt(vh) + eps)
    return dict(view=apply_twist(delta, view), m=m6, v=v6, delta=delta)


def densify_add(alpha, depth, tgt_color, tgt_depth, view, cam, tau_alpha=0.5, tau_depth=0.10, stride=2,
                init_opacity=0.5, max_add=None, sh_degree=0) -> np.ndarray:
    """Eq. 8: unreliable iff T < tau_T or |D - D_hat| > tau_D (T = alpha image);
    restricted to valid target depth and the stride-2 checkerboard ((u+v) % 2 == 0, the HW/2 of
    Eq. 7), ordered by pixel index; back-projected from the target depth through the inverse
    pose; init per reading C22. Returns activated params [14][n_add], or [23][n_add] with sh_degree=1
    (reading C34: the colour becomes the DC coefficient (c - 1/2)/C0 in fp32, linear terms 0)."""
    a = np.asarray(alpha, np.float64)
    d = np.asarray(depth, np.float64)
    td = np.asarray(tgt_depth, np.float64)
    tc = np.asarray(tgt_color, np.float64)
    h, w = a.shape
    vv, uu = np.mgrid[0:h, 0:w]
    flag = (td > 0) & ((a < tau_alpha) | (np.abs(td - d) > tau_depth)) & (((uu + vv) % stride) == 0)
    idx = np.flatnonzero(flag.reshape(-1))
    if max_add is not None:
        idx = idx[:max_add]
    u = (idx % w).astype(np.float64)
    v = (idx // w).astype(np.float64)
    z = td.reshape(-1)[idx]
    xc = np.stack([(u - cam.cx) / cam.fx * z, (v - cam.cy) / cam.fy * z, z])
    V = np.asarray(view, np.float64)
    X = V[:, :3].T @ (xc - V[:, 3:4])
    out = np.zeros((23 if sh_degree == 1 else 14, idx.size))
    out[0:3] = X
    out[3:6] = z * stride / (cam.fx + cam.fy)
    out[6] = 1.0
    out[10] = init_opacity
    out[11:14] = tc.reshape(3, -1)[:, idx]
    if sh_degree == 1:
        c = tc.reshape(3, -1)[:, idx].astype(np.float32)
        out[11:14] = (c - np.float32(0.5)) / np.float32(0.28209479177387814)
    return out


def densify_prune_mask(opacity, min_opacity=0.005) -> np.ndarray:
    """Keep mask of the opacity prune (BASELINE config 4; not in the paper): keep o >= min."""
    return np.asarray(opacity, np.float64) >= min_opacity


def _rot(q):
    q = np.asarray(q, np.float64)
    r, x, y, z = q / np.linalg.norm(q)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - r * z), 2 * (x * z + r * y)],
                     [2 * (x * y + r * z), 1 - 2 * (x * x + z * z), 2 * (y * z - r * x)],
                     [2 * (x * z - r * y), 2 * (y * z + r * x), 1 - 2 * (x * x + y * y)]])   # Eq. S1


def accum_grad(grad_screen, tiles, W, H, accum, count):
    """Reading C30 (3DGS adaptive density control): for the on-screen Gaussians,
    accum += |(dL/dm_x W/2, dL/dm_y H/2)| (NDC units), count += 1."""
    on = np.asarray(tiles) > 0
    g = np.hypot(np.asarray(grad_screen[0], np.float64) * (W / 2), np.asarray(grad_screen[1], np.float64) * (H / 2))
    a = np.asarray(accum, np.float64).copy()
    c = np.asarray(count, np.float64).copy()
    a[on] += g[on]
    c[on] += 1
    return a, c


def split_clone(params, accum, count, noise, grad_thresh=0.002, scale_thresh=0.02, capacity=None):
    """Reading C30: avg = accum / count (0 if count == 0); candidates avg >= grad_thresh; clone
    (max scale <= scale_thresh) = a copy; split = two children X + R(q) diag(s) eps_k (noise rows 3k..3k+2)
    with scale s / 1.6, the original removed. Order: kept originals, clones, children. Appends beyond
    capacity are dropped (clones first; a split only if both children fit). Returns (params, appended
    mask of the result [new columns], removed originals)."""
    p = np.asarray(params, np.float64)
    n = p.shape[1]
    cap = n if capacity is None else capacity
    cnt = np.asarray(count, np.float64)
    avg = np.where(cnt > 0, np.asarray(accum, np.float64) / np.where(cnt > 0, cnt, 1), 0.0)
    cand = avg >= grad_thresh
    smax = p[3:6].max(0)
    clone = np.flatnonzero(cand & (smax <= scale_thresh))
    split = np.flatnonzero(cand & ~(smax <= scale_thresh))
    avail = cap - n
    clone = clone[:max(avail, 0)]
    split = split[:max(avail - clone.size, 0) // 2]
    new = [p[:, i] for i in clone]
    for i in split:
        R = _rot(p[6:10, i])
        s = p[3:6, i]
        for k in range(2):
            c = p[:, i].copy()
            c[0:3] = p[0:3, i] + R @ (s * np.asarray(noise, np.float64)[3 * k:3 * k + 3, i])
            c[3:6] = s / 1.6
            new.append(c)
    keep = np.ones(n, bool)
    keep[split] = False
    out = np.concatenate([p[:, keep]] + ([np.stack(new, 1)] if new else []), axis=1)
    return out, clone, split


def pose_extrapolate(view_prev2, view_prev) -> np.ndarray:
    """Constant velocity: out = (T2 T1^-1) T2 for world->camera 3x4 poses (fp64)."""
    def h(v):
        m = np.eye(4)
        m[:3] = np.asarray(v, np.float64)
        return m
    T1, T2 = h(view_prev2), h(view_prev)
    return (T2 @ np.linalg.inv(T1) @ T2)[:3]


def image_half(color, depth):
    """PAPER.md:173 coarse image (reading C12's half camera): 2x2 mean of colour in the order
    ((c00 + c01) + (c10 + c11)) * 0.25 in fp32; depth = mean of the valid samples (00, 01, 10, 11)."""
    c = np.asarray(color, np.float32)
    d = np.asarray(depth, np.float32)
    H, W = d.shape
    Hh, Wh = H // 2, W // 2
    c = c[:, :2 * Hh, :2 * Wh]
    d = d[:2 * Hh, :2 * Wh]
    ch = ((c[:, 0::2, 0::2] + c[:, 0::2, 1::2]) + (c[:, 1::2, 0::2] + c[:, 1::2, 1::2])) * np.float32(0.25)
    s = np.zeros((Hh, Wh), np.float32)
    cnt = np.zeros((Hh, Wh), np.int32)
    for dv, du in ((0, 0), (0, 1), (1, 0), (1, 1)):
        x = d[dv::2, du::2]
        s = np.where(x > 0, s + x, s).astype(np.float32)
        cnt += x > 0
    dh = np.where(cnt > 0, s / np.maximum(cnt, 1).astype(np.float32), np.float32(0)).astype(np.float32)
    return ch.astype(np.float32), dh


def frame_stats(alpha, depth, tgt_depth, tau_alpha=0.5, tau_depth=0.10) -> tuple[int, int, int]:
    """Keyframe rule measurement: (reliable valid pixels by Eq. 8's complement, valid pixels,
    observed pixels alpha >= tau_alpha). Comparisons in fp32."""
    a = np.asarray(alpha, np.float32)
    d = np.asarray(depth, np.float32)
    t = np.asarray(tgt_depth, np.float32)
    valid = t > 0
    obs = a >= np.float32(tau_alpha)
    rel = valid & obs & (np.abs(t - d) <= np.float32(tau_depth))
    return int(rel.sum()), int(valid.sum()), int(obs.sum())


def pixel_colour_loss(color, tgt_color) -> np.ndarray:
    """Reading C32 ("the loss on the pixel"): the per-pixel colour L1, (|dC_0| + |dC_1|) + |dC_2|,
    evaluated in fp32 in that order."""
    c = np.asarray(color, np.float32)
    t = np.asarray(tgt_color, np.float32)
    e = np.abs(c - t)
    return (e[0] + e[1]) + e[2]


def loss_l1_masked(color, depth, tgt_color, tgt_depth, alpha, alpha_min=0.5, w_color=0.9, w_depth=0.1,
                   outlier_k=0.0) -> dict:
    """Reading C31 (tracking only on previously observed areas): Eq. 6 as means over the kept
    pixels: colour over 3 N_kept values, depth over the kept pixels with valid D*; zero gradient
    elsewhere. Kept = observed (alpha >= alpha_min) and, with outlier_k > 0, reading C32 (P:954,
    "more than ten times the median loss ... ignored"): l_p <= outlier_k * m in fp32, m the lower
    median of l_p over the observed pixels."""
    obs = np.asarray(alpha, np.float32) >= np.float32(alpha_min)
    if outlier_k > 0 and obs.any():
        lp = pixel_colour_loss(color, tgt_color)
        vals = np.sort(lp[obs])
        med = vals[(vals.size - 1) // 2]
        obs = obs & (lp <= np.float32(outlier_k) * med)
    elif outlier_k > 0:
        obs = np.zeros_like(obs)
    c = np.asarray(color, np.float64)
    d = np.asarray(depth, np.float64)
    tc = np.asarray(tgt_color, np.float64)
    td = np.asarray(tgt_depth, np.float64)
    valid = obs & (td > 0)
    nobs, nv = int(obs.sum()), int(valid.sum())
    sc = w_color / (3.0 * nobs) if nobs else 0.0
    sd = w_depth / nv if nv else 0.0
    loss = sc * np.abs(c - tc)[:, obs].sum() + sd * np.abs(d - td)[valid].sum()
    return dict(loss=loss, dL_dcolor=sc * np.sign(c - tc) * obs, dL_ddepth=sd * np.sign(d - td) * valid, kept=obs)


def degenerate_mask(mean2d, depth, tiles, tgt_depth, gamma=0.10) -> np.ndarray:
    """Eq. 9, reading C27: a Gaussian visible in the frame (tiles > 0) is a floater iff its
    centre pixel round(m) = floor(m + 0.5) is inside the image with valid D* > 0 and D* - d > gamma
    ("in front of the scene surfaces"). The comparison is fp32 (both sides decide in fp32)."""
    td = np.asarray(tgt_depth, np.float32)
    h, w = td.shape
    m = np.asarray(mean2d, np.float32)
    u = np.floor(m[0] + np.float32(0.5))
    v = np.floor(m[1] + np.float32(0.5))
    inside = (u >= 0) & (u < w) & (v >= 0) & (v < h) & (np.asarray(tiles) > 0)
    ui = np.where(inside, u, 0).astype(np.int64)
    vi = np.where(inside, v, 0).astype(np.int64)
    dstar = td[vi, ui]
    return inside & (dstar > 0) & ((dstar - np.asarray(depth, np.float32)) > np.float32(gamma))


def degenerate(opacity, mask, eta=0.1):
    """Eq. 9: Lambda_i <- eta Lambda_i for the flagged Gaussians (fp32 product); the raw (logit) value
    of the new opacity in fp64."""
    o = np.asarray(opacity, np.float32).copy()
    o[mask] = np.float32(eta) * o[mask]
    od = o.astype(np.float64)
    return o, np.log(od / (1.0 - od))


def select_mask(mean2d, depth, tiles, accum_weight, tgt_depth, sel_weight=0.5, sel_depth=0.05) -> np.ndarray:
    """Eq. 12, reading C24: keep iff accumulated alpha*T > sel_weight and
    |D*(round m) - d| < sel_depth at pixel round(m) = floor(m + 0.5) inside the image, D* > 0."""
    td = np.asarray(tgt_depth, np.float64)
    h, w = td.shape
    m = np.asarray(mean2d, np.float64)
    u = np.floor(m[0] + 0.5)
    v = np.floor(m[1] + 0.5)
    inside = (u >= 0) & (u < w) & (v >= 0) & (v < h) & (np.asarray(tiles) > 0)
    ui = np.where(inside, u, 0).astype(np.int64)
    vi = np.where(inside, v, 0).astype(np.int64)
    dstar = td[vi, ui]
    return inside & (dstar > 0) & (np.asarray(accum_weight) > sel_weight) & \
        (np.abs(dstar - np.asarray(depth, np.float64)) < sel_depth)
