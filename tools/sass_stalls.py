#!/usr/bin/env python
"""Top stall instructions of one kernel in an ncu report (source page, SASS).

usage: python tools/sass_stalls.py <report.ncu-rep> [n] [kernel-regex]
Prints total stall samples per reason and the n hottest instructions with
their dominant reasons and a few instructions of context."""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
    if len(sys.argv) > 3:
        args += ["-k", "regex:" + sys.argv[3]]
    out = subprocess.run(args, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    # one block per kernel: a "Kernel Name" row, the header row, the SASS rows
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
    for a, b in zip(starts, starts[1:]):
        report(rows[a:b], n)


def report(rows, n):
    hdr = rows[1]
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    ri = [hdr.index(h) for h in reasons]
    val = lambda r, i: int(r[i]) if r[i].isdigit() else 0
    tot = sum(val(r, si) for r in data)
    print(f"{rows[0][1]}: {tot} samples")
    agg = {h: sum(val(r, i) for r in data) for h, i in zip(reasons, ri)}
    print("  " + ", ".join(f"{k[6:]} {100 * v / max(tot, 1):.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1]) if v))
    order = sorted(range(len(data)), key=lambda k: -val(data[k], si))[:n]
    for k in order:
        r = data[k]
        rs = sorted(((val(r, i), h[6:]) for h, i in zip(reasons, ri)), reverse=True)[:3]
        print(f"{val(r, si):7d} {100 * val(r, si) / max(tot, 1):5.1f}%  [{k:5d}] {r[1].strip()[:70]:70s} " +
              " ".join(f"{h}:{v}" for v, h in rs if v))


if __name__ == "__main__":
    main()
