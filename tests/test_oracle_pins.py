"""Pins of the oracle against things other than itself (task rule ③): worked examples and closed
forms from the paper, library routines (scipy rotations / expm, torch.optim.Adam, autograd),
brute force on tiny inputs, central finite differences and invariants. CPU only."""
import dataclasses
import json
import math
import os

import numpy as np
import pytest

import gs_inputs as gi
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def single(mean, scale, quat, opacity, rgb):
    p = np.zeros((14, 1), np.float64)
    p[0:3, 0] = mean
    p[3:6, 0] = scale
    p[6:10, 0] = quat
    p[10, 0] = opacity
    p[11:14, 0] = rgb
    return p


def tiny_scene(n, seed, W=32, H=32, f=30.0, opacity=(0.3, 0.8)):
    """Seeded <=20-Gaussian scene in front of a 32x32 camera (FD fixtures)."""
    rng = np.random.default_rng(seed)
    cam = gi.Camera(f, f, (W - 1) / 2, (H - 1) / 2, W, H)
    z = rng.uniform(1.5, 3.0, n)
    p = np.zeros((14, n))
    p[0] = rng.uniform(-0.4, 0.4, n) * z
    p[1] = rng.uniform(-0.4, 0.4, n) * z
    p[2] = z
    p[3:6] = np.exp(rng.normal(math.log(0.08), 0.3, (3, n)))
    q = rng.normal(size=(4, n))
    p[6:10] = q / np.linalg.norm(q, axis=0)
    p[10] = rng.uniform(*opacity, n)
    p[11:14] = rng.uniform(0, 1, (3, n))
    return p, cam


def small_pose(seed, rot_deg=8.0, trans=0.15):
    rng = np.random.default_rng(seed)
    d = np.concatenate([rng.normal(size=3) * trans, np.radians(rot_deg) * rng.normal(size=3) / math.sqrt(3)])
    return oracle.apply_twist(d, gi.identity_view().astype(np.float64))


# ------------------------------------------------------------------ O1/O3 worked example (golden)
def test_worked_example_golden():
    g = json.load(open(os.path.join(GOLDEN, "worked_example.json")))
    c, gs_, e = g["camera"], g["gaussian"], g["expect"]
    cam = gi.Camera(c["fx"], c["fy"], c["cx"], c["cy"], c["width"], c["height"])
    p = single(gs_["mean"], gs_["scale"], gs_["quat"], gs_["opacity"], gs_["rgb"])
    for prec in ("f32", "f64"):
        pr = oracle.project(p, gi.identity_view(), cam, prec)
        np.testing.assert_allclose(pr["cov2d"][:, 0], [e["cov2d_A"], e["cov2d_B"], e["cov2d_C"]], rtol=1e-6)
        np.testing.assert_allclose(pr["conic"][[0, 2], 0], [e["conic_a"], e["conic_c"]], rtol=1e-6)
        assert pr["radius"][0] == e["radius"]
        np.testing.assert_allclose(pr["mean2d"][:, 0], e["mean2d"], rtol=0, atol=1e-6)
        assert pr["rect"][:, 0].tolist() == e["rect"]
        assert pr["tiles"][0] == e["tiles"]
        assert pr["depth_bits"][0] == e["depth_bits"]
        b = oracle.bin_sort(pr["depth_bits"], pr["rect"], pr["tiles"], cam)
        assert (b["keys"] >> np.uint64(32)).tolist() == e["tile_ids"]
        f = oracle.forward(p, gi.identity_view(), cam, prec)
        u, v = e["pixel"]
        np.testing.assert_allclose(f["alpha"][v, u], e["alpha_at_pixel"], rtol=1e-6)
        np.testing.assert_allclose(f["depth"][v, u], e["depth_at_pixel"], rtol=1e-6)
    # lambda1 (largest eigenvalue + the 0.1 floor of reading C11)
    A, C = e["cov2d_A"], e["cov2d_C"]
    assert abs((A + C) / 2 + math.sqrt(max(0.1, ((A + C) / 2) ** 2 - e["det"])) - e["lambda1"]) < 1e-5


# ------------------------------------------------------------------ O1 vs library rotation + numeric Jacobian
def ewa_reference(mean_w, scale, quat, view, cam):
    """Sigma' built from scipy's quaternion->matrix and a finite-difference Jacobian of the
    pinhole map (independent of Eq. S1 as typed and of the analytic J)."""
    from scipy.spatial.transform import Rotation
    R = Rotation.from_quat([quat[1], quat[2], quat[3], quat[0]]).as_matrix()
    Sigma = R @ np.diag(np.asarray(scale) ** 2) @ R.T
    W, t = view[:, :3], view[:, 3]
    xc = W @ mean_w + t

    def pin(x):
        return np.array([cam.fx * x[0] / x[2] + cam.cx, cam.fy * x[1] / x[2] + cam.cy])
    J = np.zeros((2, 3))
    for k in range(3):
        h = 1e-6 * max(1.0, abs(xc[k]))
        e = np.zeros(3)
        e[k] = h
        J[:, k] = (pin(xc + e) - pin(xc - e)) / (2 * h)
    Sp = J @ W @ Sigma @ W.T @ J.T + cam.cov2d_dilation * np.eye(2)
    return pin(xc), Sp, xc[2]


def test_projection_matches_library_rotation_and_numeric_jacobian():
    rng = np.random.default_rng(7)
    cam = gi.CAM_TUM
    view = small_pose(3, rot_deg=20, trans=0.3)
    for _ in range(50):
        z = rng.uniform(0.5, 6)
        mean = np.array([rng.uniform(-0.5, 0.5) * z, rng.uniform(-0.4, 0.4) * z, z])
        mean_w = view[:, :3].T @ (mean - view[:, 3])
        scale = np.exp(rng.normal(-3, 0.5, 3))
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        p = single(mean_w, scale, q * rng.uniform(0.5, 2.0), 0.5, [0, 0, 0])   # unnormalised quat
        pr = oracle.project(p, view, cam, "f64")
        m_ref, Sp_ref, d_ref = ewa_reference(mean_w, scale, q, view, cam)
        np.testing.assert_allclose(pr["mean2d"][:, 0], m_ref, rtol=1e-9)
        np.testing.assert_allclose(pr["depth"][0], d_ref, rtol=1e-12)
        A, B, C = pr["cov2d"][:, 0]
        np.testing.assert_allclose([A, B, C], [Sp_ref[0, 0], Sp_ref[0, 1], Sp_ref[1, 1]], rtol=2e-6, atol=1e-9)
        Q = np.linalg.inv(Sp_ref)
        np.testing.assert_allclose(pr["conic"][:, 0], [Q[0, 0], Q[0, 1], Q[1, 1]], rtol=2e-6, atol=1e-12)


def test_spec_geometry_examples():
    # S:42-44 q->R examples via the projected footprint: q=(0,0,0,1) is 180 deg about z, which
    # maps an x-elongated Gaussian to an x-elongated one; 90 deg about z swaps the axes.
    cam = gi.CAM_TINY
    base = dict(mean=[0, 0, 2], opacity=0.5, rgb=[0, 0, 0])
    a = oracle.project(single(scale=[0.2, 0.05, 0.05], quat=[1, 0, 0, 0], **base), gi.identity_view(), cam, "f64")
    b = oracle.project(single(scale=[0.2, 0.05, 0.05], quat=[0, 0, 0, 1], **base), gi.identity_view(), cam, "f64")
    c = oracle.project(single(scale=[0.2, 0.05, 0.05], quat=[math.cos(math.pi / 4), 0, 0, math.sin(math.pi / 4)],
                              **base), gi.identity_view(), cam, "f64")
    np.testing.assert_allclose(a["cov2d"], b["cov2d"], atol=1e-12)
    np.testing.assert_allclose(c["cov2d"][[0, 2], 0], a["cov2d"][[2, 0], 0], rtol=1e-12)
    # on-axis Sigma' = (f s / z)^2 + 0.3
    np.testing.assert_allclose(a["cov2d"][0, 0], (60 * 0.2 / 2) ** 2 + 0.3, rtol=1e-12)
    # behind the near plane -> culled (radius 0, no tiles)
    d = oracle.project(single(mean=[0, 0, 0.1], scale=[0.1] * 3, quat=[1, 0, 0, 0], opacity=0.5, rgb=[0, 0, 0]),
                       gi.identity_view(), cam, "f32")
    assert d["radius"][0] == 0 and d["tiles"][0] == 0


def test_camera_roll_rotates_footprint():
    # rolling the camera 90 deg about its axis keeps d and rotates Sigma' by 90 deg
    cam = dataclasses.replace(gi.CAM_TINY, cx=32.0, cy=32.0, width=64, height=64)
    p = single([0.1, -0.05, 2.5], [0.2, 0.05, 0.08], [0.9, 0.2, -0.3, 0.1], 0.5, [0, 0, 0])
    roll = oracle.apply_twist([0, 0, 0, 0, 0, math.pi / 2], gi.identity_view().astype(np.float64))
    a = oracle.project(p, gi.identity_view(), cam, "f64")
    b = oracle.project(p, roll, cam, "f64")
    np.testing.assert_allclose(a["depth"], b["depth"], rtol=1e-12)
    np.testing.assert_allclose(b["cov2d"][:, 0], [a["cov2d"][2, 0], -a["cov2d"][1, 0], a["cov2d"][0, 0]], rtol=1e-9)


# ------------------------------------------------------------------ O2 brute force
def test_bin_sort_brute_force():
    cfg = gi.CONFIGS[0]
    p = cfg.scene()
    pr = oracle.project(p, cfg.view(), cfg.cam, "f32")
    b = oracle.bin_sort(pr["depth_bits"], pr["rect"], pr["tiles"], cfg.cam)
    gx, gy = oracle.grid(cfg.cam)
    pairs = []
    for i in range(p.shape[1]):
        for ty in range(pr["rect"][2, i], pr["rect"][3, i]):
            for tx in range(pr["rect"][0, i], pr["rect"][1, i]):
                pairs.append(((ty * gx + tx) << 32 | int(pr["depth_bits"][i]), i))
    pairs.sort()  # (key, index): stable order of index-ordered emission
    assert b["n_keys"] == len(pairs) == int(pr["tiles"].sum())
    assert b["keys"].tolist() == [k for k, _ in pairs]
    assert b["vals"].tolist() == [v for _, v in pairs]
    for t in range(gx * gy):
        js = [j for j, (k, _) in enumerate(pairs) if k >> 32 == t]
        want = (js[0], js[-1] + 1) if js else (0, 0)
        assert tuple(b["ranges"][t]) == want


def test_tile_list_equals_candidate_walk():
    """O3 walks the global depth order with the rect rule; every pixel that did not terminate
    examines exactly its tile's list."""
    cfg = gi.CONFIGS[0]
    p = cfg.scene()
    pr = oracle.project(p, cfg.view(), cfg.cam, "f32")
    b = oracle.bin_sort(pr["depth_bits"], pr["rect"], pr["tiles"], cfg.cam)
    f = oracle.forward(p, cfg.view(), cfg.cam, "f32")
    gx, _ = oracle.grid(cfg.cam)
    H, W = f["alpha"].shape
    vv, uu = np.mgrid[0:H, 0:W]
    t = (vv // 16) * gx + uu // 16
    ln = (b["ranges"][:, 1].astype(np.int64) - b["ranges"][:, 0])[t]
    # a pixel can only have terminated if T_final < 1e-4 / (1 - 0.99), i.e. alpha > 0.99
    open_px = f["alpha"] <= 0.99
    assert open_px.mean() > 0.5
    assert np.array_equal(f["examined"][open_px], ln[open_px])
    assert (f["examined"] <= ln).all() and (f["n_last"] <= f["examined"]).all()


# ------------------------------------------------------------------ O3 closed forms and invariants
def test_empty_scene():
    cam = dataclasses.replace(gi.CAM_TINY, bg=(0.1, 0.2, 0.3))
    f = oracle.forward(np.zeros((14, 0)), gi.identity_view(), cam, "f64")
    assert np.allclose(f["color"][0], 0.1) and np.allclose(f["color"][2], 0.3)
    assert (f["depth"] == 0).all() and (f["alpha"] == 0).all()


def test_clamped_single_gaussian():
    # opacity -> 1 is clamped to alpha = 0.99: C = 0.99 c, D = 0.99 d at the centre pixel
    cam = gi.CAM_TINY
    p = single([0.5 * 2 / 60, 0.5 * 2 / 60, 2.0], [0.1] * 3, [1, 0, 0, 0], 0.9999, [0.3, 0.6, 0.9])
    for prec in ("f32", "f64"):
        f = oracle.forward(p, gi.identity_view(), cam, prec)
        np.testing.assert_allclose(f["alpha"][24, 32], 0.99, rtol=1e-7)
        np.testing.assert_allclose(f["color"][:, 24, 32], 0.99 * np.array([0.3, 0.6, 0.9]), rtol=1e-6)
        np.testing.assert_allclose(f["depth"][24, 32], 1.98, rtol=1e-6)


def footprint(p, i, u, v, cam, view):
    """Closed-form alpha = o exp(-1/2 d^T Sigma'^-1 d) (north_star pin) with Sigma' from the
    library-rotation / numeric-Jacobian reference."""
    m, Sp, _ = ewa_reference(p[0:3, i], p[3:6, i], p[6:10, i] / np.linalg.norm(p[6:10, i]), view, cam)
    d = m - np.array([u, v])
    return min(0.99, p[10, i] * math.exp(-0.5 * d @ np.linalg.solve(Sp, d)))


def test_two_gaussian_expansion():
    # C = c1 a1 + c2 a2 (1 - a1) + bg (1 - a1)(1 - a2)
    cam = dataclasses.replace(gi.CAM_TINY, bg=(1.0, 1.0, 1.0))
    p = np.concatenate([single([0.02, 0.01, 2.0], [0.1, 0.12, 0.08], [0.9, 0.1, 0.2, 0.3], 0.6, [0.9, 0.1, 0.2]),
                        single([-0.03, 0.02, 3.0], [0.15, 0.1, 0.1], [0.8, -0.1, 0.3, 0.2], 0.7, [0.1, 0.8, 0.3])], 1)
    view = gi.identity_view().astype(np.float64)
    f = oracle.forward(p, view, cam, "f64")
    for (u, v) in [(31, 23), (30, 25), (33, 22)]:
        a1 = footprint(p, 0, u, v, cam, view)
        a2 = footprint(p, 1, u, v, cam, view)
        want = p[11:14, 0] * a1 + p[11:14, 1] * a2 * (1 - a1) + np.array(cam.bg) * (1 - a1) * (1 - a2)
        np.testing.assert_allclose(f["color"][:, v, u], want, rtol=1e-7)
        np.testing.assert_allclose(f["depth"][v, u], 2.0 * a1 + 3.0 * a2 * (1 - a1), rtol=1e-7)
        np.testing.assert_allclose(f["alpha"][v, u], 1 - (1 - a1) * (1 - a2), rtol=1e-7)


def test_weight_identity_convexity_and_monotone_T():
    cfg = gi.CONFIGS[0]
    p = cfg.scene().astype(np.float64)
    p1 = p.copy()
    p1[11:14] = 1.0
    for prec, tol in (("f64", 1e-12), ("f32", 1e-6)):
        f = oracle.forward(p1, cfg.view(), cfg.cam, prec)   # black bg: colour = sum of weights
        assert np.abs(f["color"][0] - f["alpha"]).max() < tol
    f = oracle.forward(p, cfg.view(), cfg.cam, "f64")
    assert (f["color"] >= -1e-12).all() and (f["color"] <= 1 + 1e-12).all()   # convex (bg black, rgb in [0,1])
    # T non-increasing: replaying with a growing contributor prefix never lowers alpha
    px = np.array([23 * 64 + 31, 10 * 64 + 5, 40 * 64 + 60])
    prev = np.zeros(3)
    for k in range(0, 40, 3):
        g = oracle.forward(p, cfg.view(), cfg.cam, "f64", pixels=px, replay_nlast=np.full(3, k))
        assert (g["alpha"] >= prev - 1e-15).all()
        prev = g["alpha"]


def test_permutation_invariance():
    cfg = gi.CONFIGS[0]
    p = cfg.scene()
    pr = oracle.project(p, cfg.view(), cfg.cam, "f32")
    vis = pr["tiles"] > 0
    assert len(np.unique(pr["depth_bits"][vis])) == vis.sum()   # distinct depths
    perm = np.random.default_rng(5).permutation(p.shape[1])
    a = oracle.forward(p, cfg.view(), cfg.cam, "f32")
    b = oracle.forward(p[:, perm], cfg.view(), cfg.cam, "f32")
    for k in ("color", "depth", "alpha"):
        assert np.array_equal(a[k], b[k])


def test_f32_and_f64_instantiations_agree():
    cfg = gi.CONFIGS[0]
    p = cfg.scene()
    a = oracle.forward(p, cfg.view(), cfg.cam, "f32")
    b = oracle.forward(p, cfg.view(), cfg.cam, "f64")
    ok = (a["ambiguous"] == 0) & (b["ambiguous"] == 0)
    assert np.abs(a["color"] - b["color"])[:, ok].max() < 1e-5
    assert np.abs(a["depth"] - b["depth"])[ok].max() < 1e-5


# ------------------------------------------------------------------ O4: finite differences
def linear_loss(p, view, cam, dc, dd):
    f = oracle.forward(p, view, cam, "f64")
    return float((dc * f["color"]).sum() + (dd * f["depth"]).sum()), f["hash"]


@pytest.mark.parametrize("seed,posed,opac", [(11, False, (0.3, 0.8)), (12, True, (0.3, 0.8)),
                                             (13, True, (0.5, 1.0))])
def test_backward_matches_central_fd(seed, posed, opac):
    p, cam = tiny_scene(12, seed, opacity=opac)
    view = small_pose(seed) if posed else gi.identity_view().astype(np.float64)
    if posed:   # keep the scene in front of the moved camera: express means in world frame
        p[0:3] = view[:, :3].T @ (p[0:3] - view[:, 3:4])
    dc, dd = gi.upstream(cam.width, cam.height, seed + 100)
    dc, dd = dc.astype(np.float64), dd.astype(np.float64)
    g = oracle.backward(p, view, cam, dc.astype(np.float32), dd.astype(np.float32), "f64")
    # the oracle takes fp32 upstream; use exactly those values in the FD loss
    dc32, dd32 = dc.astype(np.float32).astype(np.float64), dd.astype(np.float32).astype(np.float64)
    checked = rejected = 0
    for i in range(p.shape[1]):
        for k in range(14):
            h = 1e-6 * max(abs(p[k, i]), 0.05)
            pp, pm = p.copy(), p.copy()
            pp[k, i] += h
            pm[k, i] -= h
            lp, hp = linear_loss(pp, view, cam, dc32, dd32)
            lm, hm = linear_loss(pm, view, cam, dc32, dd32)
            if hp != hm:
                rejected += 1
                continue
            fd = (lp - lm) / (2 * h)
            an = g["grad_params"][k, i]
            assert abs(fd - an) <= 1e-3 * max(abs(fd), abs(an)) + 1e-8, (i, k, fd, an)
            checked += 1
    assert checked >= 0.9 * 14 * p.shape[1] and rejected < 0.1 * 14 * p.shape[1]
    # pose: FD on exp(eps e_k) T, covariance path on (reading C7)
    pose_checked = 0
    for k in range(6):
        for eps in (1e-6, 3e-7, 1e-7):   # a pose step moves every Gaussian: retry if a decision flips
            e = np.zeros(6)
            e[k] = eps
            lp, hp = linear_loss(p, oracle.apply_twist(e, view), cam, dc32, dd32)
            lm, hm = linear_loss(p, oracle.apply_twist(-e, view), cam, dc32, dd32)
            if hp == hm:
                break
        if hp != hm:
            continue
        fd = (lp - lm) / (2 * eps)
        an = g["pose_twist"][k]
        assert abs(fd - an) <= 1e-3 * max(abs(fd), abs(an)) + 1e-8, (k, fd, an)
        pose_checked += 1
    assert pose_checked >= 5


def test_pose_qt_path_equals_twist_path():
    """Eq. S1/S3 (q,t) gradient mapped to the twist equals the twist path (both with and without
    the covariance term)."""
    p, cam = tiny_scene(15, 21)
    view = small_pose(22, rot_deg=25, trans=0.2)
    p[0:3] = view[:, :3].T @ (p[0:3] - view[:, 3:4])
    dc, dd = gi.upstream(cam.width, cam.height, 23)
    for cov in (True, False):
        g = oracle.backward(p, view, cam, dc, dd, "f64", qt_cov=cov)
        q = g["pose_quat"]
        t = view[:, 3]
        tw = np.zeros(6)
        tw[:3] = g["pose_t"]
        for k in range(3):
            ek = np.zeros(3)
            ek[k] = 1.0
            # Hamilton product (0, e_k/2) (x) q
            dq = np.concatenate([[-0.5 * ek @ q[1:]], 0.5 * (q[0] * ek + np.cross(ek, q[1:]))])
            tw[3 + k] = g["pose_q"] @ dq + g["pose_t"] @ np.cross(ek, t)
        want = g["pose_twist"] if cov else g["pose_twist_paper"]
        np.testing.assert_allclose(tw, want, rtol=1e-9, atol=1e-12)


def test_eq_s6_depth_and_colour_on_stacks():
    """Eq. S6 in its printed product form on a 3-Gaussian on-axis stack (G = 1 at the
    centre pixel so alpha_i = o_i), plus its colour analogue with a white background."""
    cam = gi.Camera(40.0, 40.0, 16.0, 16.0, 33, 33, bg=(1.0, 1.0, 1.0))
    o = [0.3, 0.5, 0.4]
    z = [1.0, 2.0, 3.0]
    cols = np.array([[0.9, 0.1, 0.2], [0.2, 0.7, 0.1], [0.3, 0.3, 0.8]])
    p = np.concatenate([single([0, 0, z[i]], [0.05] * 3, [1, 0, 0, 0], o[i], cols[i]) for i in range(3)], 1)
    view = gi.identity_view().astype(np.float64)
    H = W = 33
    dd = np.zeros((H, W), np.float32)
    dd[16, 16] = 1.0
    dc = np.zeros((3, H, W), np.float32)
    g = oracle.backward(p, view, cam, dc, dd, "f64")
    a = o

    def prod(js):
        return float(np.prod([1 - a[j] for j in js]))
    for i in range(3):
        Ti = prod(range(i))
        # dD/dd_i = alpha_i prod_{j<i}(1 - alpha_j)
        np.testing.assert_allclose(g["grad_screen"][9, i], a[i] * Ti, rtol=1e-12)
        want = z[i] * Ti - sum(z[k] * a[k] * prod([j for j in range(k) if j != i]) for k in range(i + 1, 3))
        np.testing.assert_allclose(g["grad_screen"][5, i], want, rtol=1e-12)   # dL/do = G dL/dalpha, G = 1
    for ch in range(3):
        dc = np.zeros((3, H, W), np.float32)
        dc[ch, 16, 16] = 1.0
        g = oracle.backward(p, view, cam, dc, np.zeros((H, W), np.float32), "f64")
        for i in range(3):
            Ti = prod(range(i))
            want = cols[i, ch] * Ti - sum(cols[k, ch] * a[k] * prod([j for j in range(k) if j != i])
                                          for k in range(i + 1, 3)) - 1.0 * prod([j for j in range(3) if j != i])
            np.testing.assert_allclose(g["grad_screen"][5, i], want, rtol=1e-12)
            np.testing.assert_allclose(g["grad_screen"][6 + ch, i], a[i] * Ti, rtol=1e-12)


def test_zero_upstream_and_linearity():
    cfg = gi.CONFIGS[0]
    p = cfg.scene()
    H, W = cfg.cam.height, cfg.cam.width
    z = oracle.backward(p, cfg.view(), cfg.cam, np.zeros((3, H, W), np.float32), np.zeros((H, W), np.float32))
    assert not z["grad_params"].any() and not z["pose_twist"].any()
    # quantised so that the fp32 sums c1 + c2, d1 + d2 are exact
    c1, d1 = (np.round(a * 1024) / 1024 for a in gi.upstream(W, H, 1))
    c2, d2 = (np.round(a * 1024) / 1024 for a in gi.upstream(W, H, 2))
    g1 = oracle.backward(p, cfg.view(), cfg.cam, c1, d1)
    g2 = oracle.backward(p, cfg.view(), cfg.cam, c2, d2)
    g12 = oracle.backward(p, cfg.view(), cfg.cam, c1 + c2, d1 + d2)
    np.testing.assert_allclose(g12["grad_params"], g1["grad_params"] + g2["grad_params"], rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(g12["pose_twist"], g1["pose_twist"] + g2["pose_twist"], rtol=1e-9, atol=1e-9)


def test_self_target_stationarity():
    """L1 to the image rendered at the same pose has zero upstream, hence zero pose grad."""
    cfg = gi.CONFIGS[0]
    p = cfg.scene()
    f = oracle.forward(p, cfg.view(), cfg.cam)
    L = oracle.loss_l1(f["color"], f["depth"], f["color"], f["depth"])
    assert L["loss"] == 0 and not L["dL_dcolor"].any() and not L["dL_ddepth"].any()
    g = oracle.backward(p, cfg.view(), cfg.cam, L["dL_dcolor"].astype(np.float32), L["dL_ddepth"].astype(np.float32))
    assert not g["pose_twist"].any()


# ------------------------------------------------------------------ O5 (numpy) pins
def test_loss_l1_brute_force():
    rng = np.random.default_rng(3)
    H, W = 4, 5
    c = rng.uniform(size=(3, H, W))
    tc = rng.uniform(size=(3, H, W))
    tc[0, 1, 2] = c[0, 1, 2]          # sign(0) = 0
    d = rng.uniform(1, 2, (H, W))
    td = rng.uniform(1, 2, (H, W))
    td[0, 0] = 0.0                    # invalid depth
    L = oracle.loss_l1(c, d, tc, td, 0.9, 0.1)
    nvalid = sum(1 for v in range(H) for u in range(W) if td[v, u] > 0)
    want = 0.0
    for v in range(H):
        for u in range(W):
            for ch in range(3):
                want += 0.9 / (3 * H * W) * abs(c[ch, v, u] - tc[ch, v, u])
            if td[v, u] > 0:
                want += 0.1 / nvalid * abs(d[v, u] - td[v, u])
    assert abs(L["loss"] - want) < 1e-14
    assert L["dL_dcolor"][0, 1, 2] == 0 and L["dL_ddepth"][0, 0] == 0
    assert L["dL_dcolor"][1, 1, 2] == math.copysign(0.9 / (3 * H * W), c[1, 1, 2] - tc[1, 1, 2])


@pytest.mark.parametrize("rows", [14, 23])
def test_adam_matches_torch(rows):
    """O5 Adam against torch.optim.Adam with autograd through the activations; 23 rows is the
    degree-1 SH layout (rows 11-22 identity-activated)."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(4)
    n = 7
    raw = rng.normal(size=(rows, n))
    lr = [1.6e-5] * 3 + [2e-4] * 3 + [4e-5] * 4 + [1e-2] + [5e-4] * (rows - 11)
    m = np.zeros((rows, n))
    v = np.zeros((rows, n))
    traw = torch.tensor(raw, dtype=torch.float64, requires_grad=True)
    groups = [{"params": [], "lr": r} for r in lr]
    prm = [torch.nn.Parameter(traw[k].detach().clone()) for k in range(rows)]
    for k in range(rows):
        groups[k]["params"] = [prm[k]]
    opt = torch.optim.Adam(groups, betas=(0.9, 0.999), eps=1e-8)
    for step in range(1, 4):
        gact = rng.normal(size=(rows, n))
        out = oracle.adam_step(raw, gact, m, v, lr, step)
        opt.zero_grad()
        act = [prm[k] for k in range(rows)]
        act[3:6] = [torch.exp(prm[k]) for k in range(3, 6)]
        act[10] = torch.sigmoid(prm[10])
        sum((a * torch.tensor(gact[k])).sum() for k, a in enumerate(act)).backward()
        opt.step()
        raw, m, v = out["raw"], out["m"], out["v"]
        np.testing.assert_allclose(raw, np.stack([r.detach().numpy() for r in prm]), rtol=1e-12, atol=1e-15)


def test_se3_exp_matches_expm():
    from scipy.linalg import expm
    d = np.array([0.01, -0.02, 0.015, 0.2, -0.1, 0.3])
    T = np.zeros((4, 4))
    T[:3, :3] = oracle.skew(d[3:])
    T[:3, 3] = d[:3]
    np.testing.assert_allclose(oracle.se3_exp(d), expm(T)[:3], atol=1e-14)


def test_densify_add_brute_force_and_backprojection():
    rng = np.random.default_rng(9)
    H, W = 5, 6
    cam = gi.Camera(5.0, 5.0, 2.5, 2.0, W, H)
    view = small_pose(2)
    alpha = rng.uniform(size=(H, W))
    depth = rng.uniform(1, 2, (H, W))
    td = depth + rng.choice([0.0, 0.05, 0.3], size=(H, W))
    td[1, 1] = 0.0
    tc = rng.uniform(size=(3, H, W))
    out = oracle.densify_add(alpha, depth, tc, td, view, cam, 0.5, 0.10, 2)
    want = [v * W + u for v in range(H) for u in range(W)
            if td[v, u] > 0 and (alpha[v, u] < 0.5 or abs(td[v, u] - depth[v, u]) > 0.10) and (u + v) % 2 == 0]
    assert out.shape[1] == len(want)
    for j, pid in enumerate(want):
        u, v = pid % W, pid // W
        xc = view[:, :3] @ out[0:3, j] + view[:, 3]
        np.testing.assert_allclose([cam.fx * xc[0] / xc[2] + cam.cx, cam.fy * xc[1] / xc[2] + cam.cy, xc[2]],
                                   [u, v, td[v, u]], atol=1e-12)
        np.testing.assert_allclose(out[11:14, j], tc[:, v, u])
        assert out[10, j] == 0.5 and out[6, j] == 1.0
    capped = oracle.densify_add(alpha, depth, tc, td, view, cam, max_add=2)
    np.testing.assert_array_equal(capped, out[:, :2])


def test_select_mask_brute_force():
    rng = np.random.default_rng(10)
    H, W = 6, 7
    n = 40
    m = np.stack([rng.uniform(-2, W + 1, n), rng.uniform(-2, H + 1, n)])
    d = rng.uniform(1, 2, n)
    tiles = rng.integers(0, 3, n)
    aw = rng.uniform(0, 1, n)
    td = rng.uniform(1, 2, (H, W))
    td[2, 3] = 0
    for i in range(n):   # force some near-surface ones
        u, v = math.floor(m[0, i] + 0.5), math.floor(m[1, i] + 0.5)
        if 0 <= u < W and 0 <= v < H and i % 2 == 0:
            d[i] = td[v, u] + 0.01
    got = oracle.select_mask(m, d, tiles, aw, td)
    for i in range(n):
        u, v = math.floor(m[0, i] + 0.5), math.floor(m[1, i] + 0.5)
        want = (0 <= u < W and 0 <= v < H and tiles[i] > 0 and td[v, u] > 0 and aw[i] > 0.5
                and abs(td[v, u] - d[i]) < 0.05)
        assert bool(got[i]) == want


def test_prune_mask():
    o = np.array([0.001, 0.005, 0.0049999, 0.5])
    assert oracle.densify_prune_mask(o).tolist() == [False, True, False, True]


# ------------------------------------------------------------------ degree-1 SH colour (NEXT-1, reading C29)
def sh1_of(p, seed, lin=0.6):
    """Append degree-1 SH rows to a 14-row scene: constant terms Y0 ~ N(0, 1), linear terms ~ N(0, lin)
    (rows 11 + 3k + c). The RGB rows are replaced by the constant terms."""
    rng = np.random.default_rng(seed)
    n = p.shape[1]
    q = np.zeros((23, n))
    q[:11] = p[:11]
    q[11:14] = rng.normal(0.0, 1.0, (3, n))
    q[14:23] = rng.normal(0.0, lin, (9, n))
    return q


def test_sh1_basis_normalised_on_the_sphere():
    """The degree-1 real SH basis is orthonormal on the unit sphere: with one unit coefficient the
    colour minus its 1/2 offset, squared and averaged over uniformly distributed view directions,
    equals 1/(4 pi) (for l = 0 and each l = 1 term), and distinct terms are orthogonal."""
    rng = np.random.default_rng(5)
    n = 200_000
    u = rng.normal(size=(3, n))
    u /= np.linalg.norm(u, axis=0)
    cam = gi.Camera(30.0, 30.0, 15.5, 15.5, 32, 32)
    vals = []
    for k in range(4):
        p = np.zeros((23, n))
        p[0:3] = 3.0 * u            # camera centre at the origin (identity pose): direction u
        p[3:6] = 0.05
        p[6] = 1.0
        p[10] = 0.5
        p[11 + 3 * k] = 1.0        # channel r: unit coefficient of basis term k
        p[11 + 3 * k + 1] = 1.0    # channel g too (channel b stays 0: colour 1/2 exactly)
        rgb = oracle.project(p, gi.identity_view(), cam, "f64")["rgb"]
        # clamping at 0 would bias the integral: use a unit coefficient small enough to stay above 0
        assert (rgb[0] > 0).all()
        f = rgb[0] - 0.5
        vals.append(f)
        assert np.allclose(rgb[2], 0.5)
        np.testing.assert_allclose(rgb[1], rgb[0], rtol=0, atol=1e-15)
    for k in range(4):
        assert abs(4 * math.pi * np.mean(vals[k] ** 2) - 1.0) < 0.01, k
        for m in range(k):
            assert abs(4 * math.pi * np.mean(vals[k] * vals[m])) < 0.01, (k, m)


def test_sh1_odd_symmetry_and_rgb_reduction():
    """The l = 1 terms are odd in the view direction: mirroring a Gaussian through the camera centre
    flips them, so rgb(X) + rgb(2c - X) = 2 (1/2 + C0 Y0) (unclamped). With zero linear terms the SH
    scene renders exactly like the RGB scene with rgb = 1/2 + C0 Y0 at any pose."""
    p14, cam = tiny_scene(12, 41)
    view = small_pose(42, rot_deg=20, trans=0.3)
    p14[0:3] = view[:, :3].T @ (p14[0:3] - view[:, 3:4])
    p = sh1_of(p14, 43, lin=0.1)
    p[11:14] = np.abs(p[11:14]) + 0.5    # keep every channel above the clamp
    c = -view[:, :3].T @ view[:, 3]
    mirrored = p.copy()
    mirrored[0:3] = 2 * c[:, None] - p[0:3]
    a = oracle.project(p, view, cam, "f64")["rgb"]
    b = oracle.project(mirrored, view, cam, "f64")["rgb"]
    const = oracle.project(np.concatenate([p[:14], np.zeros((9, p.shape[1]))]), view, cam, "f64")["rgb"]
    np.testing.assert_allclose(a + b, 2 * const, rtol=0, atol=1e-12)
    # reduction: zero linear terms == RGB rows holding the constant-term colour
    p0 = p.copy()
    p0[14:23] = 0.0
    rgb = p14.copy()
    rgb[11:14] = oracle.project(p0, view, cam, "f64")["rgb"]
    f_sh = oracle.forward(p0, view, cam, "f64")
    f_rgb = oracle.forward(rgb, view, cam, "f64")
    np.testing.assert_allclose(f_sh["color"], f_rgb["color"], rtol=0, atol=1e-12)
    assert f_sh["hash"] == f_rgb["hash"]


@pytest.mark.parametrize("seed", [61, 62])
def test_sh1_backward_matches_central_fd(seed):
    """Central FD on the fp64 oracle over all 23 parameter rows (12 SH coefficients, and the mean
    through the view direction) and the 6 pose components (the colour reaches the pose through the
    camera centre)."""
    p14, cam = tiny_scene(10, seed)
    view = small_pose(seed, rot_deg=10, trans=0.2)
    p14[0:3] = view[:, :3].T @ (p14[0:3] - view[:, 3:4])
    p = sh1_of(p14, seed + 1)
    dc, dd = gi.upstream(cam.width, cam.height, seed + 100)
    dc32, dd32 = dc.astype(np.float32).astype(np.float64), dd.astype(np.float32).astype(np.float64)
    g = oracle.backward(p, view, cam, dc.astype(np.float32), dd.astype(np.float32), "f64")
    checked = rejected = 0
    for i in range(p.shape[1]):
        for k in range(23):
            h = 1e-6 * max(abs(p[k, i]), 0.05)
            pp, pm = p.copy(), p.copy()
            pp[k, i] += h
            pm[k, i] -= h
            lp, hp = linear_loss(pp, view, cam, dc32, dd32)
            lm, hm = linear_loss(pm, view, cam, dc32, dd32)
            rp = oracle.project(pp, view, cam, "f64")["rgb"][:, i]
            rm = oracle.project(pm, view, cam, "f64")["rgb"][:, i]
            if hp != hm or ((rp > 0) != (rm > 0)).any():   # a decision or a colour clamp flips
                rejected += 1
                continue
            fd = (lp - lm) / (2 * h)
            an = g["grad_params"][k, i]
            assert abs(fd - an) <= 1e-3 * max(abs(fd), abs(an)) + 1e-8, (i, k, fd, an)
            checked += 1
    assert checked >= 0.9 * 23 * p.shape[1] and rejected < 0.1 * 23 * p.shape[1]
    pose_checked = 0
    for k in range(6):
        for eps in (1e-6, 3e-7, 1e-7):
            e = np.zeros(6)
            e[k] = eps
            lp, hp = linear_loss(p, oracle.apply_twist(e, view), cam, dc32, dd32)
            lm, hm = linear_loss(p, oracle.apply_twist(-e, view), cam, dc32, dd32)
            if hp == hm:
                break
        if hp != hm:
            continue
        fd = (lp - lm) / (2 * eps)
        an = g["pose_twist"][k]
        assert abs(fd - an) <= 1e-3 * max(abs(fd), abs(an)) + 1e-8, (k, fd, an)
        pose_checked += 1
    assert pose_checked >= 5


def test_sh1_pose_qt_path_equals_twist_path():
    """With degree-1 SH the colour depends on the camera centre c = -W^T t: the (q, t) path (which
    sees c move with both q and t) mapped to the twist equals the twist path, whose colour term is
    rho += W sum dL/dX_dir and nothing in phi."""
    p14, cam = tiny_scene(15, 71)
    view = small_pose(72, rot_deg=25, trans=0.2)
    p14[0:3] = view[:, :3].T @ (p14[0:3] - view[:, 3:4])
    p = sh1_of(p14, 73)
    dc, dd = gi.upstream(cam.width, cam.height, 74)
    g = oracle.backward(p, view, cam, dc, dd, "f64", qt_cov=True)
    q = g["pose_quat"]
    t = view[:, 3]
    tw = np.zeros(6)
    tw[:3] = g["pose_t"]
    for k in range(3):
        ek = np.zeros(3)
        ek[k] = 1.0
        dq = np.concatenate([[-0.5 * ek @ q[1:]], 0.5 * (q[0] * ek + np.cross(ek, q[1:]))])
        tw[3 + k] = g["pose_q"] @ dq + g["pose_t"] @ np.cross(ek, t)
    np.testing.assert_allclose(tw, g["pose_twist"], rtol=1e-9, atol=1e-12)


# ------------------------------------------------------------------ Eq. 9 opacity degeneration (NEXT-2)
def test_degenerate_hand_built_fixture():
    """Eq. 9 with a flat wall at D* = 3 m seen head-on (reading C27: D* - d > gamma): a Gaussian
    0.5 m in front of the wall is a floater; one 0.05 m in front (within gamma = 0.1), one behind the
    wall, one whose centre pixel has no valid depth and one off-screen are not. Degeneration scales
    the flagged opacity by eta and nothing else."""
    W, H = 32, 24
    cam = gi.Camera(30.0, 30.0, (W - 1) / 2, (H - 1) / 2, W, H)
    zs = [2.5, 2.95, 3.4, 2.0, 2.0]
    xs = [0.0, 0.3, -0.3, 0.0, 40.0]   # the last one projects far outside the image
    ys = [0.0, 0.2, -0.2, 0.5, 0.0]
    n = len(zs)
    p = np.zeros((14, n))
    p[0] = np.array(xs) * np.array(zs) / 10
    p[1] = np.array(ys) * np.array(zs) / 10
    p[2] = zs
    p[3:6] = 0.02
    p[6] = 1.0
    p[10] = 0.8
    p[11:14] = 0.5
    td = np.full((H, W), 3.0, np.float32)
    pr = oracle.project(p, gi.identity_view(), cam, "f32")
    # invalidate the depth at Gaussian 3's centre pixel
    u3 = int(np.floor(pr["mean2d"][0, 3] + 0.5))
    v3 = int(np.floor(pr["mean2d"][1, 3] + 0.5))
    td[v3, u3] = 0.0
    mask = oracle.degenerate_mask(pr["mean2d"], pr["depth"], pr["tiles"], td, gamma=0.10)
    assert mask.tolist() == [True, False, False, False, False]
    o, raw = oracle.degenerate(p[10], mask, eta=0.1)
    np.testing.assert_allclose(o, [0.08, 0.8, 0.8, 0.8, 0.8], rtol=1e-7)
    np.testing.assert_allclose(raw[0], math.log(0.08 / 0.92), rtol=1e-6)


# ------------------------------------------------------------------ split / clone (NEXT-2, reading C30)
def test_split_clone_hand_built():
    """Three Gaussians with hand-set statistics: below the gradient threshold (untouched), small and
    above it (cloned: an exact copy appended), large and above it (split: removed, two children at
    X + R diag(s) eps with scale s/1.6). With the identity rotation the children sit at X + s * eps
    exactly; with a 90-degree rotation about z, (ex, ey) map to (-ey, ex)."""
    p = np.zeros((14, 4))
    p[0:3] = [[0, 1, 2, 3], [0, 0, 0, 0], [2, 2, 2, 2]]
    p[3:6] = np.array([0.01, 0.01, 0.05, 0.04])[None, :] * np.array([[1.0], [0.5], [0.5]])
    p[6] = 1.0
    p[6:10, 3] = [math.cos(math.pi / 4), 0, 0, math.sin(math.pi / 4)]   # 90 deg about z
    p[10] = [0.3, 0.4, 0.5, 0.6]
    p[11:14] = 0.5
    accum = np.array([0.001, 0.009, 0.012, 0.02])
    count = np.array([1.0, 3.0, 4.0, 4.0])    # averages 0.001, 0.003, 0.003, 0.005
    noise = np.zeros((6, 4))
    noise[:, 2] = [1, 2, 3, -1, -2, -3]
    noise[:, 3] = [1, 0, 0, 0, 1, 0]
    out, clone, split = oracle.split_clone(p, accum, count, noise, 0.002, 0.02, capacity=10)
    assert clone.tolist() == [1] and split.tolist() == [2, 3]
    assert out.shape[1] == 4 - 2 + 1 + 4
    np.testing.assert_array_equal(out[:, 0], p[:, 0])
    np.testing.assert_array_equal(out[:, 1], p[:, 1])
    np.testing.assert_array_equal(out[:, 2], p[:, 1])   # the clone
    s2 = p[3:6, 2]
    np.testing.assert_allclose(out[0:3, 3], p[0:3, 2] + s2 * [1, 2, 3])
    np.testing.assert_allclose(out[0:3, 4], p[0:3, 2] - s2 * [1, 2, 3])
    np.testing.assert_allclose(out[3:6, 3], s2 / 1.6)
    s3 = p[3:6, 3]
    np.testing.assert_allclose(out[0:3, 5], p[0:3, 3] + [0, s3[0], 0], atol=1e-12)    # e_x -> e_y
    np.testing.assert_allclose(out[0:3, 6], p[0:3, 3] + [-s3[1], 0, 0], atol=1e-12)   # e_y -> -e_x
    # capacity: one free column takes the clone only; no split fits
    out2, c2, s2_ = oracle.split_clone(p, accum, count, noise, 0.002, 0.02, capacity=5)
    assert c2.tolist() == [1] and s2_.size == 0 and out2.shape[1] == 5


# ------------------------------------------------------------------ tracking front end (NEXT-4)
def test_pose_extrapolate_constant_twist():
    """Constant velocity: on a trajectory T_k = exp(k delta) T_0 the extrapolation of T_1, T_2
    is exactly T_3 (SE(3) exponential from scipy's expm)."""
    from scipy.linalg import expm
    delta = np.array([0.03, -0.01, 0.02, 0.01, 0.04, -0.02])
    X = np.zeros((4, 4))
    X[:3, :3] = oracle.skew(delta[3:])
    X[:3, 3] = delta[:3]
    E = expm(X)
    T0 = np.eye(4)
    T0[:3] = oracle.apply_twist(np.array([0.1, 0.2, -0.3, 0.2, -0.1, 0.3]), gi.identity_view().astype(np.float64))
    T = [np.linalg.matrix_power(E, k) @ T0 for k in range(4)]
    np.testing.assert_allclose(oracle.pose_extrapolate(T[1][:3], T[2][:3]), T[3][:3], atol=1e-12)


def test_masked_loss_and_frame_stats_brute_force():
    """Masked L1 (reading C31): all pixels observed reduces to Eq. 6's colour mean over 3HW and depth
    mean over valid pixels (the unmasked oracle loss); a brute-force loop checks a partial mask.
    Frame statistics: brute-force counts."""
    W, H = 12, 9
    c, d = gi.random_images(W, H, 3)
    tc, td = gi.random_images(W, H, 4)
    full = oracle.loss_l1_masked(c, d, tc, td, np.ones((H, W)), 0.5)
    ref = oracle.loss_l1(c, d, tc, td)
    assert abs(full["loss"] - ref["loss"]) <= 1e-12 * abs(ref["loss"])
    a = np.random.default_rng(5).uniform(0, 1, (H, W)).astype(np.float32)
    m = oracle.loss_l1_masked(c, d, tc, td, a, 0.5)
    obs = [(v, u) for v in range(H) for u in range(W) if a[v, u] >= 0.5]
    val = [(v, u) for v, u in obs if td[v, u] > 0]
    lc = sum(abs(float(c[ch, v, u]) - float(tc[ch, v, u])) for v, u in obs for ch in range(3)) * 0.9 / (3 * len(obs))
    ld = sum(abs(float(d[v, u]) - float(td[v, u])) for v, u in val) * 0.1 / len(val)
    assert abs(m["loss"] - (lc + ld)) <= 1e-12
    assert (m["dL_dcolor"][:, a < 0.5] == 0).all()
    rel = sum(1 for v in range(H) for u in range(W)
              if td[v, u] > 0 and a[v, u] >= 0.5 and abs(float(td[v, u]) - float(d[v, u])) <= np.float32(0.1))
    assert oracle.frame_stats(a, d, td, 0.5, 0.10) == (rel, int((td > 0).sum()), int((a >= 0.5).sum()))


def test_outlier_rejection_brute_force():
    """Reading C32: the lower median by Python's statistics.median_low over the observed
    pixels' colour losses; a planted set of 5 gross outliers (colour off by 1.0 in every channel) is
    dropped at k = 10 and nothing else is; the kept-pixel loss equals the masked loss with the
    outliers made unobserved; k large enough keeps everything (reduces to reading C31)."""
    import statistics
    W, H = 16, 11
    c, d = gi.random_images(W, H, 31)
    tc = np.clip(c + np.random.default_rng(32).normal(0, 0.01, c.shape), 0, 1).astype(np.float32)
    td = d.copy()
    a = np.ones((H, W), np.float32)
    a[0, :3] = 0.2
    bad = [(2, 3), (5, 7), (9, 1), (10, 15), (4, 4)]
    for v, u in bad:
        tc[:, v, u] = np.where(c[:, v, u] > 0.5, c[:, v, u] - 1.0, c[:, v, u] + 1.0)
    o = oracle.loss_l1_masked(c, d, tc, td, a, 0.5, outlier_k=10.0)
    lp = [[sum(abs(float(c[ch, v, u]) - float(tc[ch, v, u])) for ch in range(3)) for u in range(W)] for v in range(H)]
    med = statistics.median_low([lp[v][u] for v in range(H) for u in range(W) if a[v, u] >= 0.5])
    drop = {(v, u) for v in range(H) for u in range(W) if a[v, u] >= 0.5 and lp[v][u] > 10 * med}
    assert drop == set(bad)
    assert set(zip(*np.nonzero(~o["kept"] & (a >= 0.5)))) == set(bad)
    a2 = a.copy()
    for v, u in bad:
        a2[v, u] = 0.0
    ref = oracle.loss_l1_masked(c, d, tc, td, a2, 0.5)
    assert abs(o["loss"] - ref["loss"]) <= 1e-12 * ref["loss"]
    np.testing.assert_array_equal(o["dL_dcolor"], ref["dL_dcolor"])
    everything = oracle.loss_l1_masked(c, d, tc, td, a, 0.5, outlier_k=1e9)
    assert everything["loss"] == oracle.loss_l1_masked(c, d, tc, td, a, 0.5)["loss"]


def test_opacity_radius_box_holds_every_contributing_pixel():
    """Reading C33: with the opacity-aware radius every pixel where the closed-form footprint
    (library rotation, numeric Jacobian) reaches alpha >= 1/255 lies in a tile of the rect; the
    rect holds no tile without such a pixel beyond the box's own rounding (each edge tile meets the
    ellipse's bounding box); o <= 1/255 is culled; on an isotropic footprint the radius is
    ceil(sqrt((2 ln(255 o) + 2e-3) lambda))."""
    rng = np.random.default_rng(11)
    cam = gi.CAM_TUM
    view = small_pose(5, rot_deg=10, trans=0.2)
    uu, vv = np.meshgrid(np.arange(cam.width), np.arange(cam.height))
    for k in range(40):
        z = rng.uniform(1.0, 5)
        mean = np.array([rng.uniform(-0.4, 0.4) * z, rng.uniform(-0.3, 0.3) * z, z])
        mean_w = view[:, :3].T @ (mean - view[:, 3])
        scale = np.exp(rng.normal(-3.5, 0.6, 3))
        q = rng.normal(size=4)
        o = [0.003, 0.0039, 0.004, 0.05, 0.3, 0.7, 0.99][k % 7]
        p = single(mean_w, scale, q, o, [0, 0, 0])
        pr = oracle.project(p, view, cam, "f32", opacity_radius=True)
        if o <= 1 / 255:
            assert pr["tiles"][0] == 0 and pr["radius"][0] == 0
            continue
        m, Sp, _ = ewa_reference(mean_w, scale, q / np.linalg.norm(q), view, cam)
        d = np.stack([m[0] - uu, m[1] - vv], -1)
        Q = np.linalg.inv(Sp)
        qq = np.einsum("...i,ij,...j->...", d, Q, d)
        hit = o * np.exp(-0.5 * qq) >= 1 / 255
        xlo, xhi, ylo, yhi = pr["rect"][:, 0]
        tx, ty = uu // 16, vv // 16
        inside = (tx >= xlo) & (tx < xhi) & (ty >= ylo) & (ty < yhi)
        assert not (hit & ~inside).any(), k
        if hit.any():   # edge tiles meet the bounding box of the 1/255 ellipse (plus the margin)
            qm = 2 * math.log(255 * o) + 2e-3
            rx, ry = math.sqrt(qm * Sp[0, 0]), math.sqrt(qm * Sp[1, 1])
            assert xlo * 16 <= m[0] + rx + 1e-3 and (xhi - 1) * 16 + 15 >= m[0] - rx - 1e-3
            assert xlo * 16 + 16 > m[0] - rx - 1 and (xhi - 1) * 16 <= m[0] + rx + 1e-3
            assert ylo * 16 + 16 > m[1] - ry - 1 and (yhi - 1) * 16 <= m[1] + ry + 1e-3
    # isotropic: Sigma' = (f s / z)^2 I + 0.3 I at the image centre; lambda_max carries the
    # rasterizer's floor sqrt(max(0.1, mid^2 - det)) = sqrt(0.1) (reading C11)
    cam0 = gi.CAM_TINY
    p = single([0.0, 0.0, 2.0], [0.05, 0.05, 0.05], [1, 0, 0, 0], 0.5, [0, 0, 0])
    lam = (60.0 * 0.05 / 2.0) ** 2 + 0.3 + math.sqrt(0.1)
    pr = oracle.project(p, gi.identity_view().astype(np.float64), cam0, "f64", opacity_radius=True)
    assert pr["radius"][0] == math.ceil(math.sqrt((2 * math.log(255 * 0.5) + 2e-3) * lam))


def test_opacity_radius_render_equals_untiled_brute_force():
    """Reading C33: with exact tiling the tiled render equals a brute-force blend that visits every
    Gaussian at every pixel in depth order (no tiles, no rect): the image no longer depends on the
    tile grid. A scene of large, opaque Gaussians placed so that the 3-sigma tile boxes cut some
    of them short shows that the 3-sigma render does depend on it."""
    cam = dataclasses.replace(gi.CAM_TINY, bg=(0.2, 0.3, 0.4))
    rng = np.random.default_rng(3)
    ps = []
    for k in range(10):
        z = 1.5 + 0.3 * k
        ps.append(single([rng.uniform(-0.4, 0.4) * z, rng.uniform(-0.3, 0.3) * z, z],
                         np.exp(rng.normal(-2.8, 0.3, 3)) * z / 2, rng.normal(size=4), rng.uniform(0.6, 0.99),
                         rng.uniform(0, 1, 3)))
    p = np.concatenate(ps, 1)
    view = gi.identity_view().astype(np.float64)
    f = oracle.forward(p, view, cam, "f64", opacity_radius=True)
    f3 = oracle.forward(p, view, cam, "f64")
    pr = oracle.project(p, view, cam, "f64")
    order = np.argsort(pr["depth"], kind="stable")
    H, W = cam.height, cam.width
    col = np.zeros((3, H, W))
    dep = np.zeros((H, W))
    alp = np.zeros((H, W))
    for v in range(H):
        for u in range(W):
            T, c, dd = 1.0, np.zeros(3), 0.0
            for i in order:
                if pr["depth"][i] <= cam.znear:
                    continue
                a = footprint(p, i, u, v, cam, view)
                if a < 1 / 255:
                    continue
                if T * (1 - a) < 1e-4:
                    break
                c += p[11:14, i] * a * T
                dd += pr["depth"][i] * a * T
                T *= 1 - a
            col[:, v, u] = c + np.array(cam.bg) * T
            dep[v, u] = dd
            alp[v, u] = 1 - T
    np.testing.assert_allclose(f["color"], col, atol=2e-6)
    np.testing.assert_allclose(f["depth"], dep, atol=2e-5)
    np.testing.assert_allclose(f["alpha"], alp, atol=2e-6)
    assert np.abs(f3["alpha"] - alp).max() > 1e-3   # the 3-sigma box cuts contributions


def test_opacity_radius_leaves_low_opacity_renders_unchanged():
    """Reading C33: for o <= 0.3 < e^4.5/255 the 1/255 reach lies inside 3 sigma, so the opacity
    radius drops only Gaussians and tiles that never pass the skip test: the image is identical to
    the 3-sigma render (n_last, a position in the shorter list, differs), with fewer keys."""
    cfg = gi.CONFIGS[1]
    p = cfg.scene().copy()
    p[10] = np.minimum(p[10], 0.3)
    v = cfg.view()
    a = oracle.forward(p, v, cfg.cam, "f32")
    b = oracle.forward(p, v, cfg.cam, "f32", opacity_radius=True)
    for k in ("color", "depth", "alpha"):
        assert np.array_equal(a[k], b[k]), k
    ka = oracle.project(p, v, cfg.cam, "f32")["tiles"].astype(np.int64).sum()
    kb = oracle.project(p, v, cfg.cam, "f32", opacity_radius=True)["tiles"].astype(np.int64).sum()
    assert kb < 0.8 * ka, (kb, ka)


def test_image_half_brute_force():
    """PAPER.md:173 coarse image, reading C12: pure-Python 2x2 loops in fp32, odd sizes drop the last
    row / column, invalid (zero) depths excluded from the mean; a constant image stays constant."""
    W, H = 9, 7
    c, d = gi.random_images(W, H, 41)
    d[1, 2] = 0.0
    d[0, 0] = d[0, 1] = d[1, 0] = d[1, 1] = 0.0
    ch, dh = oracle.image_half(c, d)
    assert ch.shape == (3, 3, 4) and dh.shape == (3, 4)
    f = np.float32
    for v in range(3):
        for u in range(4):
            for k in range(3):
                want = f(f(f(c[k, 2 * v, 2 * u]) + f(c[k, 2 * v, 2 * u + 1])) +
                         f(f(c[k, 2 * v + 1, 2 * u]) + f(c[k, 2 * v + 1, 2 * u + 1]))) * f(0.25)
                assert ch[k, v, u] == want
            vals = [d[2 * v + a, 2 * u + b] for a in (0, 1) for b in (0, 1) if d[2 * v + a, 2 * u + b] > 0]
            want = f(0)
            if vals:
                s = f(0)
                for x in vals:
                    s = f(s + f(x))
                want = f(s / f(len(vals)))
            assert dh[v, u] == want
    assert dh[0, 0] == 0
    ch, dh = oracle.image_half(np.full((3, 4, 6), 0.3, np.float32), np.full((4, 6), 2.5, np.float32))
    assert (ch == np.float32(0.3)).all() and (dh == np.float32(2.5)).all()


def test_sh_densify_init_reproduces_the_target_colour():
    """Reading C34: a Gaussian added with the degree-1 SH layout renders, through the SH evaluation
    of reading C29 (oracle.project's colour at the view direction), the target colour at ANY view:
    DC = (c - 1/2)/C0 and zero linear terms."""
    cam = gi.CAM_TINY
    W, H = cam.width, cam.height
    tc, td = gi.random_images(W, H, 61)
    alpha = np.zeros((H, W))
    depth = np.zeros((H, W))
    view = small_pose(9)
    add = oracle.densify_add(alpha, depth, tc, td, view, cam, sh_degree=1)
    rgb = oracle.densify_add(alpha, depth, tc, td, view, cam)
    assert add.shape[0] == 23 and add.shape[1] == rgb.shape[1] > 0
    assert (add[14:] == 0).all()
    for seed in (1, 2):
        v2 = small_pose(seed, rot_deg=30, trans=0.5)
        pr = oracle.project(add, v2, cam, "f64")
        np.testing.assert_allclose(pr["rgb"], rgb[11:14], rtol=0, atol=2e-6)
