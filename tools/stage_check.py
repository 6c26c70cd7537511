"""Stage-by-stage GPU vs oracle check (debug tool; run on the GPU box).
usage: python tools/stage_check.py [configs...]   e.g. 0 1 2"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gs_inputs as gi  # noqa: E402
import oracle  # noqa: E402
import paper_2311_11700_b200 as g  # noqa: E402


def emission(dk, rect, tiles, GX):
    n = dk.shape[0]
    cnt = tiles.astype(np.int64)
    off = np.concatenate([[0], np.cumsum(cnt)[:-1]])
    K = int(cnt.sum())
    idx = np.repeat(np.arange(n), cnt)
    local = np.arange(K) - np.repeat(off, cnt)
    w = (rect[1] - rect[0]).astype(np.int64)[idx]
    tx = rect[0].astype(np.int64)[idx] + local % np.maximum(w, 1)
    ty = rect[2].astype(np.int64)[idx] + local // np.maximum(w, 1)
    keys = ((ty * GX + tx).astype(np.uint64) << np.uint64(32)) | dk.astype(np.uint64)[idx]
    return off.astype(np.uint32), keys, idx.astype(np.uint32)


def first_diff(a, b, label):
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        print(f"  {label}: SHAPE {a.shape} vs {b.shape}")
        return False
    d = np.flatnonzero(a.reshape(-1) != b.reshape(-1))
    if d.size:
        i = d[0]
        print(f"  {label}: {d.size} diffs; first at {i}: gpu {a.reshape(-1)[i]} oracle {b.reshape(-1)[i]}")
        return False
    print(f"  {label}: OK ({a.size})")
    return True


def check(c):
    cfg = gi.CONFIGS[c]
    p, v, cam = cfg.scene(), cfg.view(), cfg.cam
    n = p.shape[1]
    print(f"config {c}: n={n} {cam.width}x{cam.height}", flush=True)
    pr = oracle.project(p, v, cam, "f32")
    K = int(pr["tiles"].astype(np.int64).sum())
    pipe = g.RenderPipeline(n, int(K * 1.05) + 4096, cam.width, cam.height)
    P = torch.as_tensor(p, device="cuda")
    V = torch.as_tensor(v, device="cuda")
    cm = g.make_camera(cam)
    g.gs_project(P, n, n, None, V, cm, pipe.ws)
    torch.cuda.synchronize()
    a = pipe.arrays(n)
    first_diff(a["depth_key"].cpu().numpy().view(np.uint32), pr["depth_bits"], "depth_key")
    first_diff(a["tiles"].cpu().numpy().view(np.uint32), pr["tiles"], "tiles")
    k = g.gs_bin_sort(pipe.ws, g.GS_FLAG_BINSORT_KEYS | g.GS_FLAG_BINSORT_EMIT_ONLY)
    torch.cuda.synchronize()
    print(f"  K gpu {k} oracle {K}", flush=True)
    gx, _ = oracle.grid(cam)
    off, ekeys, evals = emission(pr["depth_bits"], pr["rect"], pr["tiles"], gx)
    a = pipe.arrays(n, k)
    first_diff(a["offsets"].cpu().numpy().view(np.uint32), off, "offsets")
    first_diff(a["keys"].cpu().numpy().view(np.uint64), ekeys, "emitted keys")
    first_diff(a["vals"].cpu().numpy().view(np.uint32), evals, "emitted vals")
    k = g.gs_bin_sort(pipe.ws, g.GS_FLAG_BINSORT_KEYS)
    torch.cuda.synchronize()
    a = pipe.arrays(n, k)
    order = np.argsort(ekeys, kind="stable")
    ok = first_diff(a["keys"].cpu().numpy().view(np.uint64), ekeys[order], "sorted keys")
    first_diff(a["vals"].cpu().numpy().view(np.uint32), evals[order], "sorted vals")
    if not ok:
        gk = a["keys"].cpu().numpy().view(np.uint64)
        print("  sorted? ", bool((gk[1:] >= gk[:-1]).all()), " multiset equal:",
              bool(np.array_equal(np.sort(gk), np.sort(ekeys))))
    o2 = oracle.bin_sort(pr["depth_bits"], pr["rect"], pr["tiles"], cam)
    first_diff(a["ranges"].cpu().numpy().view(np.uint32), o2["ranges"], "ranges")
    col = torch.zeros(3, cam.height, cam.width, device="cuda")
    dep = torch.zeros(cam.height, cam.width, device="cuda")
    alp = torch.zeros(cam.height, cam.width, device="cuda")
    g.gs_render_fwd(pipe.ws, cm, col, dep, alp, None, g.GS_FLAG_EXAMINED)
    torch.cuda.synchronize()
    of = oracle.forward(p, v, cam, "f32")
    e = np.abs(col.cpu().numpy() - of["color"]).max()
    print(f"  forward colour max err {e:.3g}; depth {np.abs(dep.cpu().numpy() - of['depth']).max():.3g}")
    a = pipe.arrays(n, k)
    first_diff(a["examined"].cpu().numpy().view(np.uint32), of["examined"], "examined")
    first_diff(a["n_last"].cpu().numpy().view(np.uint32), of["n_last"], "n_last")


if __name__ == "__main__":
    for c in (sys.argv[1:] or ["0"]):
        check(int(c))
