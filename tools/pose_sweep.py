"""SURVEY.md §8(d) timing protocol: the bench iteration at 8 pose seeds per config (1 and 2), one
bench.py process per pose (fresh allocation, same launch configuration), median over poses.
usage (GPU box): python tools/pose_sweep.py <out.json>"""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SEEDS = {1: range(101, 109), 2: range(103, 111)}


def main():
    out = {}
    for c, seeds in SEEDS.items():
        rows = []
        for s in seeds:
            r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", str(c), "--pose-seed", str(s),
                                "--steps", "50", "--warmup", "10", "--no-e2e", "--no-cpu-baseline"],
                               capture_output=True, text=True, timeout=600)
            line = json.loads(r.stdout.strip().splitlines()[-1])
            cf = line["config"]
            rows.append({"pose_seed": s, "ms_per_step": line["ms_per_step"], "step_ms": line.get("step_ms"),
                         "keys": cf["keys"], "on_screen": cf["on_screen"], "E_f": cf["E_f"], "E_b": cf["E_b"],
                         "E_f_live": cf["E_f_live"], "sm_mhz": line["clocks"]["sm_mhz"],
                         "bwd_frac": line["roofline"]["frac"]})
            print(c, rows[-1], flush=True)
        ms = [r["ms_per_step"] for r in rows]
        out[f"config{c}"] = {"poses": rows, "median_ms": float(np.median(ms)), "min_ms": float(min(ms)),
                             "max_ms": float(max(ms)), "median_iters_per_s": 1000.0 / float(np.median(ms))}
    json.dump(out, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
