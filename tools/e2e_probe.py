"""Which transfer bounds bench.py's e2e? The same double-buffered pipeline as bench.py with parts
switched off: full, no read-back, no upload, no compute. usage (GPU box): python tools/e2e_probe.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gs_inputs as gi  # noqa: E402
import paper_2311_11700_b200 as g  # noqa: E402


def main():
    cfg = gi.CONFIGS[2]
    cam, n = cfg.cam, cfg.n
    P = torch.as_tensor(cfg.scene(), device="cuda")
    V = torch.as_tensor(cfg.view(), device="cuda")
    probe = g.RenderPipeline(n, 1 << 26, cam.width, cam.height)
    fr = probe.forward(torch.as_tensor(gi.gaussians(n, cfg.target_seed, cfg.lo, cfg.hi), device="cuda"), n, V, cam)
    tc, td = fr.color.clone(), fr.depth.clone()
    K = probe.forward(P, n, V, cam).n_keys
    del probe
    pipe = g.RenderPipeline(n, int(K * 1.2), cam.width, cam.height)
    grad = torch.zeros_like(P)
    gpose = torch.zeros(6, dtype=torch.float64, device="cuda")
    flags = g.GS_FLAG_NO_HOST_SYNC
    hp = P.cpu().pin_memory()
    hv, htc, htd = V.cpu().pin_memory(), tc.cpu().pin_memory(), td.cpu().pin_memory()
    NB = int(os.environ.get("E2E_NB", "2"))   # buffer sets in rotation
    hgrad = [torch.empty_like(grad, device="cpu").pin_memory() for _ in range(NB)]
    bufs = [(torch.empty_like(P), torch.empty_like(V), torch.empty_like(tc), torch.empty_like(td),
             torch.empty_like(grad), torch.empty_like(gpose)) for _ in range(NB)]
    for b in bufs:
        b[0].copy_(P), b[1].copy_(V), b[2].copy_(tc), b[3].copy_(td)
    s_up, s_down = torch.cuda.Stream(), torch.cuda.Stream()
    CH = int(os.environ.get("E2E_CHUNK_MB", "0")) * (1 << 18)   # floats per chunk (0: one copy per tensor)

    def chunked(dst, src):
        if not CH or dst.numel() <= CH:
            dst.copy_(src, non_blocking=True)
            return
        d, s_ = dst.view(-1), src.view(-1)
        for o in range(0, d.numel(), CH):
            d[o:o + CH].copy_(s_[o:o + CH], non_blocking=True)
    ev_c = [torch.cuda.Event() for _ in range(NB)]
    ev_d = [torch.cuda.Event() for _ in range(NB)]
    ev_r = [torch.cuda.Event() for _ in range(NB)]

    def graph_of(b):
        Pd, Vd, tcd, tdd, gd, gpd = b
        f = lambda: pipe.iteration(Pd, n, Vd, cam, tcd, tdd, gd, gpd, bin_flags=flags, fwd_flags=0,  # noqa: E731
                                   assign_grads=True, fused_loss=True)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            f()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            f()
        return gr.replay
    its = [graph_of(b) for b in bufs]

    def run(steps, up=True, down=True, comp=True):
        cur = torch.cuda.current_stream()
        s_up.wait_stream(cur)
        s_down.wait_stream(cur)
        for e in ev_r + ev_d:
            e.record(cur)

        def upload(i):
            b = bufs[i % NB]
            with torch.cuda.stream(s_up):
                s_up.wait_event(ev_d[i % NB])
                if up:
                    for dst, src in zip(b[:4], (hp, hv, htc, htd)):
                        chunked(dst, src)
                ev_c[i % NB].record(s_up)
        upload(0)
        for i in range(steps):
            if i + 1 < steps:
                upload(i + 1)
            cur.wait_event(ev_c[i % NB])
            cur.wait_event(ev_r[i % NB])
            if comp:
                its[i % NB]()
            ev_d[i % NB].record(cur)
            with torch.cuda.stream(s_down):
                s_down.wait_event(ev_d[i % NB])
                if down:
                    chunked(hgrad[i % NB], bufs[i % NB][4])
                ev_r[i % NB].record(s_down)
        cur.wait_stream(s_down)

    for name, kw in (("full", {}), ("no read-back", {"down": False}), ("no upload", {"up": False}),
                     ("no compute", {"comp": False}), ("compute only", {"up": False, "down": False}))[
            :int(os.environ.get("E2E_CASES", "5"))]:
        run(3, **kw)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run(50, **kw)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 50
        print(f"{name:14s} {ms:.3f} ms/step ({1000 / ms:.0f} steps/s)", flush=True)


if __name__ == "__main__":
    main()
