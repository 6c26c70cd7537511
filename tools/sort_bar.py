"""Path A's onesweep sort against the test-only cub::DeviceRadixSort bar on the same
emitted (tile << 32 | depth-bits, index) pairs of config 2 (or --config c): time per sort (CUDA events,
median of reps), algorithmic bytes (24 B per key per 8-bit pass), and bit-equality of the outputs.
usage (GPU box): python tools/sort_bar.py [--config 2] [--reps 10]"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def build_bar() -> str:
    src = os.path.join(ROOT, "tools", "cub_bar", "cub_bar.cu")
    out = os.path.join(ROOT, "tools", "cub_bar", "libcub_bar.so")
    if not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                               "-fPIC", src, "-o", out])
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import gs_inputs as gi
    import paper_2311_11700_b200 as g
    cfg = gi.CONFIGS[args.config]
    p, v, cam = cfg.scene(), cfg.view(), cfg.cam
    n = p.shape[1]
    P, V = torch.as_tensor(p, device="cuda"), torch.as_tensor(v, device="cuda")
    pipe = g.RenderPipeline(n, 1 << 28 if n > 1_000_000 else 1 << 26, cam.width, cam.height)
    # emitted (unsorted, index-order) pairs from path A
    fr = pipe.forward(P, n, V, cam, bin_flags=g.GS_FLAG_BINSORT_KEYS | g.GS_FLAG_BINSORT_EMIT_ONLY)
    K = fr.n_keys
    a = pipe.arrays(n, K)
    k_in = a["keys"].clone()
    v_in = a["vals"].clone()
    tiles = ((cam.width + 15) // 16) * ((cam.height + 15) // 16)
    end_bit = 32 + max(1, int(np.ceil(np.log2(tiles))))
    # path A's own sort, timed by the library's per-kernel event log (sort passes only)
    def ours():
        pipe.forward(P, n, V, cam, bin_flags=g.GS_FLAG_BINSORT_KEYS | g.GS_FLAG_NO_HOST_SYNC)
    for _ in range(3):
        ours()
    log = g.EventLog(pipe.ws, args.reps * 64)
    with log:
        for _ in range(args.reps):
            ours()
        torch.cuda.synchronize()
    per = {}
    for name, t in log.read():
        per.setdefault(name, []).append(t)
    log.close()
    sort_ms = sum(per.get("sort_pass", [])) / args.reps
    hist_ms = sum(per.get("sort_hist", [])) / args.reps
    a2 = pipe.arrays(n, K)
    ours_k, ours_v = a2["keys"].clone(), a2["vals"].clone()
    # the cub bar on the same pairs
    lib = ctypes.CDLL(build_bar())
    k_out = torch.empty_like(k_in)
    v_out = torch.empty_like(v_in)
    tb = ctypes.c_size_t(0)
    st = torch.cuda.current_stream().cuda_stream
    lib.cub_bar_sort_pairs(ctypes.c_void_p(k_in.data_ptr()), ctypes.c_void_p(v_in.data_ptr()),
                           ctypes.c_void_p(k_out.data_ptr()), ctypes.c_void_p(v_out.data_ptr()), ctypes.c_int64(K),
                           ctypes.c_int(end_bit), None, ctypes.byref(tb), ctypes.c_void_p(st))
    temp = torch.empty(tb.value, dtype=torch.uint8, device="cuda")

    def cub():
        lib.cub_bar_sort_pairs(ctypes.c_void_p(k_in.data_ptr()), ctypes.c_void_p(v_in.data_ptr()),
                               ctypes.c_void_p(k_out.data_ptr()), ctypes.c_void_p(v_out.data_ptr()),
                               ctypes.c_int64(K), ctypes.c_int(end_bit), ctypes.c_void_p(temp.data_ptr()),
                               ctypes.byref(tb), ctypes.c_void_p(st))
    for _ in range(3):
        cub()
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cub()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    cub_ms = float(np.median(ts))
    same = bool(torch.equal(k_out, ours_k) and torch.equal(v_out, ours_v))
    passes = (end_bit + 7) // 8
    algo_gb = K * (8 + 4) * 2 * passes / 1e9
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = peaks.get("hbm_gbs", 6454.3)
    out = {"config": args.config, "keys": K, "end_bit": end_bit, "passes": passes, "identical_output": same,
           "onesweep_ms": sort_ms, "onesweep_hist_ms": hist_ms, "cub_ms": cub_ms,
           "onesweep_hbm_frac": algo_gb / (sort_ms / 1e3) / hbm, "cub_hbm_frac": algo_gb / (cub_ms / 1e3) / hbm,
           "algorithmic_gb": algo_gb}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
