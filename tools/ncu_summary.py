"""Summarise ncu outputs into profiles/ (run here, on the CPU box).
usage: python tools/ncu_summary.py <launches.csv> <prof.ncu-rep> <out_prefix>
Writes <out_prefix>_launches.md (per-kernel share of the step from the launch list),
<out_prefix>_kernels.md (key --set full metrics per kernel) and profiles/ncu_traffic.json
(DRAM bytes per launch per kernel name, read by bench.py for roofline.traffic)."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

NAMES = {"render_bwd_kernel": "render_bwd_tiles", "render_fwd2_kernel": "render_fwd", "render_fwd_kernel": "render_fwd",
         "bucket_emit_kernel": "bucket_emit", "gaussian_bwd_kernel": "gaussian_bwd", "onesweep_pass_kernel": "sort_pass",
         "project_kernel": "project", "chunk_count_kernel": "chunk_hist", "emit_keys_kernel": "emit_keys",
         "bin_coop_kernel": "bin_coop", "zero_sgrad_kernel": "sgrad_clear", "valid_count_kernel": "loss_count",
         "tile_order_fwd_kernel": "tile_order"}
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def short(name):
    base = name.split("(")[0].split("<")[0].replace("void ", "").replace("gs::", "").strip()
    return base


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            k = short(d["Kernel Name"])
            agg[k][0] += 1
            agg[k][1] += float(d["Metric Value"])
    tot = sum(v[1] for v in agg.values())
    lines = ["| kernel | launches | total us | us per launch | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| {k} | {v[0]} | {v[1] / 1e3:.1f} | {v[1] / 1e3 / max(v[0], 1):.1f} | {v[1] / tot:.3f} |")
    # the library's kernels per launch (the bench's setup runs extra forwards, so shares by total
    # time over-weight the forward-side kernels): one iteration = one launch of each
    own = {k: v[1] / 1e3 / max(v[0], 1) for k, v in agg.items() if k in NAMES}
    step = sum(own.values())
    if step:
        lines += ["", "Per iteration (one launch of each library kernel):", "",
                  "| kernel | us | share of the iteration |", "|---|---|---|"]
        for k, v in sorted(own.items(), key=lambda x: -x[1]):
            lines.append(f"| {k} | {v:.1f} | {v / step:.3f} |")
    return "\n".join(lines)


def kernels(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    out, traffic, pipes = [], {}, {}
    seen = collections.Counter()
    for r in data:
        name = short(r[idx["Kernel Name"]])
        seen[name] += 1
        out.append(f"### {name} (capture {seen[name]})")
        for m in METRICS:
            if m in idx:
                out.append(f"- `{m}`: {r[idx[m]]} {units[idx[m]]}")
        try:
            rd = float(r[idx["dram__bytes_read.sum"]])
            wr = float(r[idx["dram__bytes_write.sum"]])
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            b = rd * scale.get(units[idx["dram__bytes_read.sum"]], 1) + wr * scale.get(units[idx["dram__bytes_write.sum"]], 1)
            key = NAMES.get(name, name)
            traffic[key] = b / 1e9   # GB per launch (same unit scale as roofline amounts)
            pipes[key] = {"fma_pipe_active_pct": float(r[idx["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"]]),
                          "issue_active_pct": float(r[idx["smsp__issue_active.avg.pct_of_peak_sustained_active"]]),
                          "warps_active_pct": float(r[idx["sm__warps_active.avg.pct_of_peak_sustained_active"]]),
                          # L1 / shared-memory side: the co-limit of the render kernels
                          "memory_pipes_pct": float(r[idx["gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]]),
                          "lsu_issue_pct": float(r[idx["sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]]),
                          "dram_gb_per_launch": b / 1e9,
                          "source": os.path.basename(rep)}
        except (KeyError, ValueError):
            pass
        out.append("")
    return "\n".join(out), traffic, pipes


if __name__ == "__main__":
    ll, rep, prefix = sys.argv[1:4]
    os.makedirs(os.path.dirname(prefix) or ".", exist_ok=True)
    with open(prefix + "_launches.md", "w") as f:
        f.write(f"# ncu launch list ({os.path.basename(ll)}): `ncu --metrics gpu__time_duration.sum --clock-control "
                "none` over `bench.py --quick` (cold-cache, serialised; compare shares)\n\n" + launches(ll) + "\n")
    txt, traffic, pipes = kernels(rep)
    with open(prefix + "_kernels.md", "w") as f:
        f.write(f"# ncu --set full ({os.path.basename(rep)}), bench.py config 2\n\n" + txt)
    with open(os.path.join(os.path.dirname(prefix), "ncu_traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    with open(os.path.join(os.path.dirname(prefix), "ncu_metrics.json"), "w") as f:
        json.dump(pipes, f, indent=1)   # bench.py roofline: the measured pipe activity next to the nominal count
    print(open(prefix + "_launches.md").read())
