"""Per-instruction execution counts from an ncu report's source page (SASS), for one kernel.
usage: python tools/ncu_sass_hist.py <rep> <kernel-substring> [top]"""
import csv
import subprocess
import sys


def main():
    rep, kname = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name", kname],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = None
    body = []
    for r in rows:
        if r and r[0] == "Kernel Name":
            if body:
                break
            continue
        if r and r[0] == "Address":
            h = r
            continue
        if h and len(r) == len(h):
            body.append(r)
    ie = h.index("Instructions Executed")
    smp = h.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[ie]) for r in body)
    ts = sum(int(r[smp]) for r in body)
    print(f"warp instructions {tot}, samples {ts}")
    # opcode histogram
    hist = {}
    for r in body:
        op = r[1].split()[0] if not r[1].strip().startswith("@") else r[1].split()[1]
        op = op.split(".")[0]
        hist[op] = hist.get(op, 0) + int(r[ie])
    for op, n in sorted(hist.items(), key=lambda x: -x[1])[:top]:
        print(f"{op:12s} {n:12d} {n / tot:6.3f}")


if __name__ == "__main__":
    main()
