"""Per-instruction execution counts and stall samples from an ncu report's source page (SASS), for
one kernel: opcode histogram, then the hottest instructions in address order.
usage: python tools/ncu_sass_hist.py <rep> <kernel-substring> [top] [--dump]"""
import csv
import subprocess
import sys


def rows_of(rep, kname):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                          f"regex:{kname}", "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, body = None, []
    for r in rows:
        if r and r[0] == "Kernel Name":
            if body:
                break
            continue
        if r and r[0] == "Address":
            h = [c for c in r if c != ""]
            continue
        if h and len(r) >= len(h):
            body.append(r[:len(h)])
    return h, body


def main():
    rep, kname = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 40
    h, body = rows_of(rep, kname)
    ie = h.index("Instructions Executed")
    smp = h.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[ie]) for r in body)
    ts = sum(int(r[smp]) for r in body)
    print(f"warp instructions {tot}, samples {ts}")
    hist = {}
    for r in body:
        toks = r[1].split()
        op = toks[1] if toks[0].startswith("@") else toks[0]
        op = op.split(".")[0]
        hist[op] = hist.get(op, 0) + int(r[ie])
    for op, n in sorted(hist.items(), key=lambda x: -x[1])[:top]:
        print(f"{op:12s} {n:12d} {n / tot:6.3f}")
    if "--dump" in sys.argv:
        for r in body:
            if int(r[ie]) > tot / 2000:
                print(f"{int(r[ie]):10d} {int(r[smp]):6d}  {r[1].strip()}")


if __name__ == "__main__":
    main()
