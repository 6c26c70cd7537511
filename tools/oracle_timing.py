"""CPU-oracle timings for BASELINE.md §3/§4 (run on the GPU box's host cores; the oracle is the
reported CPU baseline, never tuned). Per config: wall-clock of each stage of one iteration
(project, bin + sort, forward, L1 loss, backward), at all host cores and, for configs 0-1, at one
thread; config 3 times one coarse (600x340) and one fine (1200x680) iteration; config 4 one
keyframe of the mapping iteration (and the 8-keyframe extrapolation).
usage: python tools/oracle_timing.py [out.json]"""
from __future__ import annotations

import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import gs_inputs as gi  # noqa: E402
import oracle  # noqa: E402


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def target_of(cfg, v):
    if cfg.target_seed is None:
        return gi.random_images(cfg.cam.width, cfg.cam.height, 77)
    t = oracle.forward(gi.gaussians(cfg.n, cfg.target_seed, cfg.lo, cfg.hi), v, cfg.cam, "f32")
    return t["color"].astype(np.float32), t["depth"].astype(np.float32)


def stages(p, v, cam, tc, td, wc=0.9, wd=0.1, with_bin=True):
    out = {}
    t = time.perf_counter()
    pr = oracle.project(p, v, cam, "f32")
    out["project"] = time.perf_counter() - t
    out["keys"] = int(pr["tiles"].astype(np.int64).sum())
    if with_bin:
        t = time.perf_counter()
        oracle.bin_sort(pr["depth_bits"], pr["rect"], pr["tiles"], cam)
        out["bin_sort"] = time.perf_counter() - t
    t = time.perf_counter()
    f = oracle.forward(p, v, cam, "f32")
    out["forward"] = time.perf_counter() - t
    t = time.perf_counter()
    L = oracle.loss_l1(f["color"], f["depth"], tc, td, wc, wd)
    out["loss_l1"] = time.perf_counter() - t
    t = time.perf_counter()
    oracle.backward(p, v, cam, L["dL_dcolor"], L["dL_ddepth"], "f32")
    out["backward"] = time.perf_counter() - t
    out["iteration"] = out["forward"] + out["loss_l1"] + out["backward"]
    out["E_f"] = int(f["examined"].astype(np.int64).sum())
    out["E_b"] = int(f["n_last"].astype(np.int64).sum())
    out["evals_per_s"] = (out["E_f"] + out["E_b"]) / out["iteration"]
    return out


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "oracle_timing.json")
    cores = len(os.sched_getaffinity(0))
    res = {"cpu_model": cpu_model(), "cores": cores,
           "note": "oracle = plain C++17/OpenMP CPU renderer (oracle/oracle.cpp); iteration = forward + loss + "
                   "backward (the oracle's forward/backward project and depth-sort internally; bin_sort is "
                   "timed separately, the oracle's blend does not need the tile lists)", "configs": {}}
    for c in (0, 1, 2):
        cfg = gi.CONFIGS[c]
        p, v = cfg.scene(), cfg.view()
        tc, td = target_of(cfg, v)
        oracle.set_threads(cores)
        r = {"all_cores": stages(p, v, cfg.cam, tc, td)}
        if c <= 1:
            oracle.set_threads(1)
            r["one_thread"] = stages(p, v, cfg.cam, tc, td)
            oracle.set_threads(cores)
        res["configs"][str(c)] = r
        print(c, json.dumps(r), flush=True)
    # config 3: one coarse (600x340, every Gaussian) and one fine (1200x680) iteration, all cores;
    # the oracle's backward computes the full gradient (it has no pose-only mode)
    cfg = gi.CONFIGS[3]
    p, v = cfg.scene(), cfg.view()
    half = cfg.cam.half()
    th = oracle.forward(p, v, half, "f32")
    tf = oracle.forward(p, v, cfg.cam, "f32")
    res["configs"]["3"] = {
        "coarse": stages(p, v, half, th["color"].astype(np.float32), th["depth"].astype(np.float32), with_bin=False),
        "fine": stages(p, v, cfg.cam, tf["color"].astype(np.float32), tf["depth"].astype(np.float32),
                       with_bin=False)}
    print(3, json.dumps(res["configs"]["3"]), flush=True)
    # config 4: one keyframe of the 8-keyframe mapping iteration (2M Gaussians), all cores
    cfg = gi.CONFIGS[4]
    p, v = cfg.scene(), cfg.view()
    tc, td = target_of(cfg, v)
    k = stages(p, v, cfg.cam, tc, td, with_bin=False)
    res["configs"]["4"] = {"one_keyframe": k, "mapping_iteration_extrapolated_s": 8 * k["iteration"],
                           "note": "8 x one keyframe's fwd + loss + bwd; the oracle's Adam/densify (numpy) excluded"}
    print(4, json.dumps(res["configs"]["4"]), flush=True)
    with open(out_path, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
