"""Dynamic SASS instruction mix of one kernel from an ncu report (source page, SASS view):
warp-level instructions executed per opcode, per energy point when --points is given.

usage: python tools/sass_mix.py report.ncu-rep [--points N] [--top 30]
"""
import argparse
import csv
import io
import subprocess
from collections import Counter


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--points", type=float, default=0.0, help="energy points of the launch")
    ap.add_argument("--top", type=int, default=30)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(i for i, r in enumerate(rows) if "Source" in r)
    h = rows[hdr]
    si = h.index("Source")
    ei = next(i for i, c in enumerate(h) if c.startswith("Warp Instructions Executed")
              or c == "Instructions Executed")
    tci = next((i for i, c in enumerate(h) if c.startswith("Thread Instructions Executed")), None)
    warp, thr = Counter(), Counter()
    for r in rows[hdr + 1:]:
        if len(r) <= ei or not r[si].strip():
            continue
        toks = r[si].split()
        if toks[0].startswith("@"):
            toks = toks[1:]
        op = toks[0].split(".")[0]
        try:
            warp[op] += float(r[ei] or 0)
            if tci is not None:
                thr[op] += float(r[tci] or 0)
        except ValueError:
            pass
    tot = sum(warp.values())
    print("total warp instructions %.4g" % tot)
    for op, n in warp.most_common(a.top):
        per = " %.3f thread-instr/point" % (thr[op] / a.points) if a.points and tci is not None else ""
        print("%-8s %12.4g  %5.1f %%%s" % (op, n, 100 * n / tot, per))
    if a.points and tci is not None:
        print("all      %.3f thread-instr/point" % (sum(thr.values()) / a.points))


if __name__ == "__main__":
    main()
