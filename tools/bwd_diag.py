"""Backward parity diagnostics (GPU): per-row fraction of gradient elements outside tolerance.
usage: python tools/bwd_diag.py [config]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import gs_inputs as gi  # noqa: E402
import oracle  # noqa: E402
from gpu_helpers import grad_close, run_forward, to_dev  # noqa: E402


def main():
    c = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    cfg = gi.CONFIGS[c]
    p, v = cfg.scene(), cfg.view()
    pipe, P, V, fr = run_forward(p, v, cfg.cam)
    W, H = cfg.cam.width, cfg.cam.height
    dc, dd = gi.upstream(W, H, gi.UPSTREAM_SEED_CFG0)
    nl = pipe.arrays(p.shape[1])["n_last"].cpu().numpy()
    grad = torch.zeros_like(P)
    gpose = torch.zeros(6, dtype=torch.float64, device="cuda")
    pipe.backward(P, p.shape[1], V, cfg.cam, to_dev(dc), to_dev(dd), grad, gpose, flags=1)
    torch.cuda.synchronize()
    gg = grad.cpu().numpy()
    o = oracle.backward(p, v, cfg.cam, dc, dd, "f32", replay_nlast=nl)
    og = o["grad_params"]
    bad = grad_close(gg, og)
    print("bad frac per row", np.round(bad.mean(1), 4))
    idx = np.argwhere(bad)[:12]
    for r, i in idx:
        print(r, i, gg[r, i], og[r, i])
    sg = o.get("grad_screen")
    if sg is not None:
        print("oracle screen grads shape", np.shape(sg))


if __name__ == "__main__":
    main()
