"""Tracking diagnostics (GPU box): loss / pose error per iteration, selection statistics."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gs_inputs as gi  # noqa: E402
import oracle  # noqa: E402
import paper_2311_11700_b200 as g  # noqa: E402
from paper_2311_11700_b200.tracking import TrackConfig, Tracker, pose_error  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 1
lr = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-3
cfg = gi.CONFIGS[c]
p, v_gt, cam = cfg.scene(), cfg.view(), cfg.cam
n = p.shape[1]
pr = oracle.project(p, v_gt, cam)
K = int(pr["tiles"].astype(np.int64).sum())
tr = Tracker(n, int(K * 1.6) + 65536, int(K * 0.6) + 65536, cam)
P = torch.as_tensor(p, device="cuda")
Vgt = torch.as_tensor(v_gt, device="cuda")
fh = tr.half.forward(P, n, Vgt, cam.half())
tc_h, td_h = fh.color.clone(), fh.depth.clone()
ff = tr.full.forward(P, n, Vgt, cam)
tc_f, td_f = ff.color.clone(), ff.depth.clone()
print("target depth: mean %.3f  p10 %.3f  p90 %.3f  alpha mean %.4f" % (
    td_f.mean().item(), td_f.flatten().quantile(0.1).item(), td_f.flatten().quantile(0.9).item(),
    ff.alpha.mean().item()))
v0 = oracle.apply_twist(gi.twist_perturbation(gi.TRACK_PERTURB_SEED), v_gt.astype(np.float64))
V = torch.as_tensor(v0, dtype=torch.float32, device="cuda")
tcfg = TrackConfig(lr_rho=lr, lr_phi=lr)
tr.reset()
for it in range(50):
    tr.coarse_iter(P, n, V, tc_h, td_h, tcfg)
    if it % 5 == 0 or it == 49:
        torch.cuda.synchronize()
        print("coarse", it, "loss %.5f" % tr.half.loss.item(), "err", pose_error(V.cpu().numpy(), v_gt),
              "grad", tr.grad_pose.cpu().numpy().round(4))
m = tr.select(P, n, V, td_f, tcfg)
aw = tr.accum[:n].cpu().numpy()
a = tr.full.arrays(n)
rec = a["records"].cpu().numpy()
tiles = a["tiles"].cpu().numpy()
print("selected", int(m.sum().item()), "on-screen", int((tiles > 0).sum()), "accum>0.5", int((aw > 0.5).sum()),
      "accum max %.3f" % aw.max())
for it in range(50):
    tr.fine_iter(P, n, V, tc_f, td_f, tcfg)
    if it % 5 == 0 or it == 49:
        torch.cuda.synchronize()
        print("fine", it, "loss %.5f" % tr.full.loss.item(), "err", pose_error(V.cpu().numpy(), v_gt))
