"""Debug build (libgs_debug.so, GS_DEBUG=1): every stage's output invariants are
checked after the call (compute-sanitizer is not available on this pool). -m gpu:
- configs 0-2 run project -> bin_sort -> fwd -> L1 -> bwd and the pose-only passes clean;
- a NaN colour makes gs_project's record check fail with GS_ERR_CUDA naming the check."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import gs_inputs as gi
import paper_2311_11700_b200 as g
assert g.DEBUG and g.LIB_PATH.endswith("libgs_debug.so")
c = int(sys.argv[1]); poison = sys.argv[2] == "nan"
cfg = gi.CONFIGS[c]; p = cfg.scene(); v = cfg.view(); cam = cfg.cam; n = p.shape[1]
if poison:
    p[11, 7] = np.nan
P = torch.as_tensor(p, device="cuda"); V = torch.as_tensor(v, device="cuda")
pipe = g.RenderPipeline(n, 1 << 26 if c == 2 else 1 << 23, cam.width, cam.height)
try:
    pipe.forward(P, n, V, cam)
except g.GSError as e:
    print("GSError", e); sys.exit(3)
tc, td = gi.random_images(cam.width, cam.height, 5)
tc, td = torch.as_tensor(tc, device="cuda"), torch.as_tensor(td, device="cuda")
grad = torch.zeros_like(P); gp = torch.zeros(6, dtype=torch.float64, device="cuda")
pipe.iteration(P, n, V, cam, tc, td, grad, gp)
pipe.iteration(P, n, V, cam, tc, td, grad, gp, fused_loss=True, assign_grads=True)
for flags in (0, g.GS_FLAG_POSE_COV_PATH):
    pipe.forward(P, n, V, cam)
    pipe.pose_grad_l1(P, n, V, cam, tc, td, gp, flags=flags)
torch.cuda.synchronize()
print("debug ok", c)
'''


def _run(c, mode):
    env = dict(os.environ, GS_DEBUG="1")
    return subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT), str(c), mode], env=env,
                          capture_output=True, text=True, timeout=600)


@pytest.mark.parametrize("c", [0, 1, 2])
def test_debug_build_clean_on_configs(c):
    r = _run(c, "clean")
    assert r.returncode == 0, r.stdout + r.stderr
    assert "debug ok" in r.stdout


def test_debug_build_catches_nan_record():
    r = _run(0, "nan")
    assert r.returncode == 3, r.stdout + r.stderr
    assert "debug check failed" in r.stdout and "record finite" in (r.stdout + r.stderr)


def test_second_device_after_first():
    """Per-device kernel attributes and SM counts (PerDeviceOnce): the pipeline on cuda:1 after cuda:0
    in one process gives the same lists and images (skipped on 1-GPU boxes)."""
    import numpy as np
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    import gs_inputs as gi
    import paper_2311_11700_b200 as g
    cfg = gi.CONFIGS[1]
    p, v, cam = cfg.scene(), cfg.view(), cfg.cam
    out = []
    for d in (0, 1):
        dev = torch.device("cuda", d)
        with torch.cuda.device(dev):
            P, V = torch.as_tensor(p, device=dev), torch.as_tensor(v, device=dev)
            pipe = g.RenderPipeline(p.shape[1], 1 << 23, cam.width, cam.height, dev)
            fr = pipe.forward(P, p.shape[1], V, cam)
            grad = torch.zeros_like(P)
            tc, td = gi.random_images(cam.width, cam.height, 5)
            pipe.iteration(P, p.shape[1], V, cam, torch.as_tensor(tc, device=dev), torch.as_tensor(td, device=dev),
                           grad, None, fused_loss=True)
            torch.cuda.synchronize(dev)
            out.append((pipe.arrays()["vals"].cpu().numpy(), fr.color.cpu().numpy(), grad.cpu().numpy()))
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])   # the forward is deterministic: same bits on both devices
    assert np.isfinite(out[1][2]).all() and np.abs(out[1][2]).max() > 0
