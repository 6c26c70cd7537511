"""Where a config-4 mapping iteration's time goes on one GPU (events between the phases of
ShardedMapper.step, host timestamps around them): render + backward of the keyframes (with the
Eq. 8 candidate flags), Adam, densify (append + prune), the host sync.
usage (GPU box): python tools/mapping_breakdown.py [--steps 5]"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gs_inputs as gi  # noqa: E402
import paper_2311_11700_b200 as g  # noqa: E402
from paper_2311_11700_b200 import mapping as M  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--keyframes", type=int, default=8)
    args = ap.parse_args()
    cfg = gi.CONFIGS[4]
    cam, n = cfg.cam, cfg.n
    cap = int(n * 1.05) + 65536
    P = torch.zeros(14, cap, device="cuda")
    P[:, :n] = torch.as_tensor(cfg.scene(), device="cuda")
    tgt = torch.as_tensor(gi.gaussians(n, cfg.target_seed, cfg.lo, cfg.hi), device="cuda")
    probe = g.RenderPipeline(n, 1 << 28, cam.width, cam.height)
    kfs, kmax = [], 0
    for s in gi.MAPPING_POSE_SEEDS[:args.keyframes]:
        V = torch.as_tensor(gi.room_view(s), device="cuda")
        kmax = max(kmax, probe.forward(P, n, V, cam).n_keys)
        fr = probe.forward(tgt, n, V, cam)
        kmax = max(kmax, fr.n_keys)
        kfs.append(M.Keyframe(V, fr.color.clone(), fr.depth.clone()))
    del probe
    torch.cuda.empty_cache()
    mp = M.ShardedMapper(P, n, kfs, cam, int(kmax * 1.3) + (1 << 20), max_add_per_kf=8192)
    for _ in range(3):
        mp.step()
    torch.cuda.synchronize()
    # phase timing: the same calls as ShardedMapper.step, with events between them
    names = ["render_backward", "adam", "densify", "sync"]
    acc = {k: 0.0 for k in names}
    host = {k: 0.0 for k in names}
    total = 0.0
    for _ in range(args.steps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
        t_host = [time.perf_counter()]
        ev[0].record()
        mp.render_backward()
        ev[1].record()
        t_host.append(time.perf_counter())
        mp.it += 1
        mp.adam_t += 1
        lr = M.learning_rates(mp.it - 1, mp.iters, rows=mp.rows, sh_linear=False)
        g.gs_adam_step(mp.raw, mp.P, mp.grad, mp.m, mp.v, mp.n, mp.cap, lr, mp.adam_t)
        ev[2].record()
        t_host.append(time.perf_counter())
        cand, counts = M.gather_candidates(mp.cand, mp.counts, None)
        g.gs_densify_append(mp.P, mp.raw, mp.m, mp.v, mp.n_dev, mp.cap, mp.cap, cand, counts, cand.shape[0],
                            mp.max_add, rows=mp.rows)
        g.gs_densify_prune(mp.P, mp.raw, mp.n_dev, mp.cap, mp.cap, mp.m, mp.v, None, None, None, None, None, None,
                           None, g.densify_cfg(g.GS_DENSIFY_PRUNE, rows=mp.rows), None, None, mp.pipe.ws)
        ev[3].record()
        t_host.append(time.perf_counter())
        mp.sync()
        ev[4].record()
        t_host.append(time.perf_counter())
        torch.cuda.synchronize()
        for k, nm in enumerate(names):
            acc[nm] += ev[k].elapsed_time(ev[k + 1]) / args.steps
            host[nm] += (t_host[k + 1] - t_host[k]) * 1e3 / args.steps
        total += ev[0].elapsed_time(ev[-1]) / args.steps
    print({"keyframes": args.keyframes, "gpu_ms": {k: round(v, 3) for k, v in acc.items()},
           "host_enqueue_ms": {k: round(v, 3) for k, v in host.items()}, "total_ms": round(total, 3)})
    # one keyframe's render alone (stream launches, as inside render_backward)
    kf = kfs[0]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        mp.pipe.forward(mp.P, mp.n, kf.view, cam, bin_flags=g.GS_FLAG_NO_HOST_SYNC, fwd_flags=0)
        dc, dd = mp.pipe.loss_l1(cam, kf.color, kf.depth)
        mp.pipe.backward(mp.P, mp.n, kf.view, cam, dc, dd, mp.grad)
    e1.record()
    torch.cuda.synchronize()
    print({"one_keyframe_render_ms": round(e0.elapsed_time(e1) / 5, 3)})


if __name__ == "__main__":
    main()
