"""Diagnostics of the render work at config 2 (GPU): how many live-list evaluations the backward
issues per tile (walk to max n_last) vs per pixel, and how many of those actually blend.
usage: python tools/live_diag.py [config]"""
import sys

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import gs_inputs as gi  # noqa: E402
import paper_2311_11700_b200 as g  # noqa: E402


def main():
    c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    cfg = gi.CONFIGS[c]
    cam = cfg.cam
    P = torch.as_tensor(cfg.scene(), device="cuda")
    V = torch.as_tensor(cfg.view(), device="cuda")
    pipe = g.RenderPipeline(cfg.n, 1 << 26, cam.width, cam.height)
    pipe.forward(P, cfg.n, V, cam, fwd_flags=g.GS_FLAG_EXAMINED)
    a = pipe.arrays(cfg.n)
    GX, GY = (cam.width + 15) // 16, (cam.height + 15) // 16
    rg = a["ranges"].cpu().numpy().view(np.uint32).astype(np.int64)
    cnt = a["live_cnt"].cpu().numpy().astype(np.int64)
    lj = a["live_j"].cpu().numpy().view(np.uint32).astype(np.int64)
    lg = a["live_g"].cpu().numpy().view(np.uint32).astype(np.int64)
    nl = a["n_last"].cpu().numpy().astype(np.int64)
    rec = a["records"].cpu().numpy().astype(np.float64)
    rng = np.random.default_rng(0)
    tiles = rng.choice(GX * GY, 200, replace=False)
    ly, lx = np.meshgrid(np.arange(16.0), np.arange(16.0), indexing="ij")
    tot_tile = tot_px = tot_blend = tot_full = 0
    warp_live = 0
    for t in tiles:
        s = rg[t, 0]
        k = cnt[t]
        ty, tx = divmod(int(t), GX)
        nlt = np.zeros((16, 16), np.int64)
        blk = nl[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16]
        nlt[:blk.shape[0], :blk.shape[1]] = blk
        mx = nlt.max()
        j = lj[s:s + k]
        L = int((j <= mx).sum())
        if L == 0:
            continue
        tot_tile += L * 256
        r = rec[lg[s:s + L]]
        dx = r[:, 0, None, None] - (tx * 16 + lx)[None]
        dy = r[:, 1, None, None] - (ty * 16 + ly)[None]
        power = r[:, 2, None, None] * dx * dx + r[:, 3, None, None] * dx * dy + r[:, 4, None, None] * dy * dy
        alpha = np.minimum(0.99, r[:, 5, None, None] * np.exp(np.minimum(power, 0.0)))
        within = j[:L, None, None] <= nlt[None]
        tot_px += int(within.sum())
        hit = within & (alpha >= 1 / 255)
        tot_blend += int(hit.sum())
        tot_full += int((j[:L] <= mx).sum()) * 256
        # warp = 2 rows: does any pixel of the warp blend entry e?
        hw = hit.reshape(L, 8, 32).any(2)
        warp_live += int(hw.sum()) * 32
    print(f"config {c}: tiles sampled {len(tiles)}")
    print(f"  tile-walk evals (len(max_nl) x 256): {tot_tile}")
    print(f"  per-pixel live evals (pos <= n_last): {tot_px}  ({tot_px / tot_tile:.3f} of tile-walk)")
    print(f"  blended (alpha >= 1/255, pos <= n_last): {tot_blend}  ({tot_blend / tot_px:.3f} of per-pixel)")
    print(f"  warp-granular live (warp has a blending pixel): {warp_live}  ({warp_live / tot_tile:.3f} of tile-walk)")


if __name__ == "__main__":
    main()
