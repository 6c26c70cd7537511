"""Per-kernel times of one coarse and one fine tracking iteration (config 3, surface room and the
config-2 fog), from the library's CUDA-event log. usage (GPU box): python tools/track_kernels.py"""
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gs_inputs as gi  # noqa: E402
import paper_2311_11700_b200 as g  # noqa: E402
from paper_2311_11700_b200.tracking import TrackConfig, Tracker  # noqa: E402


def main():
    for name, scene, view in (("config2_fog", gi.CONFIGS[2].scene(), gi.CONFIGS[2].view()),
                              ("surface_room", gi.room_surface_gaussians(500_000, 31), gi.room_view(131))):
        cam = gi.CAM_REPLICA
        n = scene.shape[1]
        P = torch.as_tensor(scene, device="cuda")
        V = torch.as_tensor(view, device="cuda")
        probe = g.RenderPipeline(n, 1 << 26, cam.width, cam.height)
        K = probe.forward(P, n, V, cam).n_keys
        del probe
        tr = Tracker(n, int(K * 1.5) + 65536, int(K * 0.6) + 65536, cam)
        fh = tr.half.forward(P, n, V, cam.half())
        tch, tdh = fh.color.clone(), fh.depth.clone()
        ff = tr.full.forward(P, n, V, cam)
        tcf, tdf = ff.color.clone(), ff.depth.clone()
        cfg = TrackConfig()
        tr.select(P, n, V, tdf, cfg)
        out = {}
        for stage, pipe, fn in (("coarse", tr.half, lambda: tr.coarse_iter(P, n, V, tch, tdh, cfg)),
                                ("fine", tr.full, lambda: tr.fine_iter(P, n, V, tcf, tdf, cfg))):
            for _ in range(5):
                fn()
            torch.cuda.synchronize()
            log = g.EventLog(pipe.ws, 256)
            reps = 20
            with log:
                for _ in range(reps):
                    fn()
            torch.cuda.synchronize()
            acc = collections.defaultdict(float)
            for k, ms in log.read():
                acc[k] += ms * 1000.0 / reps
            log.close()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            out[stage] = {"us_per_iter": round(e0.elapsed_time(e1) * 1000.0 / reps, 1),
                          "kernels_us": {k: round(v, 1) for k, v in sorted(acc.items(), key=lambda x: -x[1])}}
        print(name, int(tr.mask[:n].sum().item()), out, flush=True)


if __name__ == "__main__":
    main()
