"""Backward work accounting at config 2: per-pixel live evaluations (up to each pixel's n_last, the
E_b,live of bench.py) against the slots the tile kernel evaluates (256 pixels x the live entries up to
the tile's max n_last, rounded up to batches of 16), and the share of slots whose warp has no pixel
with n_last >= the entry's position (a warp-uniform skip would save those)."""
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import gs_inputs as gi
import paper_2311_11700_b200 as g

cfg = gi.CONFIGS[2]
p, v, cam = cfg.scene(), cfg.view(), cfg.cam
n = p.shape[1]
pipe = g.RenderPipeline(n, 60_000_000, cam.width, cam.height)
pipe.forward(torch.as_tensor(p, device="cuda"), n, torch.as_tensor(v, device="cuda"), cam, fwd_flags=0)
torch.cuda.synchronize()
a = pipe.arrays(n)
GX = (cam.width + 15) // 16
GY = (cam.height + 15) // 16
nl = a["n_last"].cpu().numpy().astype(np.int64)
cnt = a["live_cnt"].cpu().numpy().astype(np.int64)
start = a["ranges"].cpu().numpy()[:, 0].astype(np.int64)
lj = a["live_j"].cpu().numpy().astype(np.int64) & 0xffffffff
H, W = nl.shape
per_px = slots = warp_skip = 0
for t in range(GX * GY):
    tx, ty = t % GX, t // GX
    tile = np.zeros((16, 16), np.int64)
    blk = nl[ty * 16:ty * 16 + 16, tx * 16:tx * 16 + 16]
    tile[:blk.shape[0], :blk.shape[1]] = blk
    pos = lj[start[t]:start[t] + cnt[t]]
    mx = tile.max()
    L = int((pos <= mx).sum())
    if L == 0:
        continue
    pos = pos[:L]
    per_px += int((pos[None, :] <= tile.reshape(-1, 1)).sum())
    nb = (L + 15) // 16
    slots += 256 * nb * 16
    # warps: threads 0..127 own rows (ly, ly + 8): warp w = rows 2w, 2w+1 and 2w+8, 2w+9
    for w in range(4):
        rows = [2 * w, 2 * w + 1, 2 * w + 8, 2 * w + 9]
        wmax = tile[rows].max()
        warp_skip += 64 * int((pos > wmax).sum())
print(f"per-pixel live evals {per_px:.4g}, kernel slots {slots:.4g} (x{slots / per_px:.3f}), "
      f"warp-skippable slots {warp_skip:.4g} ({warp_skip / slots:.1%})")
