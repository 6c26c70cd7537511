"""Per-CUDA-source-line executed instructions and stall samples from an ncu report (needs -lineinfo).
usage: python tools/ncu_lines.py <rep> <kernel-regex> [top]"""
import csv
import subprocess
import sys


def main():
    rep, kname = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--kernel-name", kname], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    ie = hdr.index("Instructions Executed")
    ss = hdr.index("Warp Stall Sampling (All Samples)")
    lines = [r for r in rows if len(r) == len(hdr) and r[0] not in ("", "Line No")]
    ti = sum(int(r[ie] or 0) for r in lines) or 1
    ts = sum(int(r[ss] or 0) for r in lines) or 1
    print(f"warp instructions {ti}, stall samples {ts}")
    for r in sorted(lines, key=lambda r: -int(r[ie] or 0))[:top]:
        print(f"{r[0]:>5} inst {int(r[ie]) / ti:6.3f} stall {int(r[ss]) / ts:6.3f}  {r[1].strip()[:100]}")


if __name__ == "__main__":
    main()
