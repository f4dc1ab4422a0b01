#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into profiles/.

usage: python tools/launch_summary.py <launches.csv> <out.txt> "<header line>"
Per kernel: launches, mean us, total us, share of our step kernels (ncu times
are cold-cache and serialised: compare SHARES with bench.py's phases, not
absolute times). Kernels outside the step (init, torch fills) get no share.
"""
import csv
import re
import sys
from collections import OrderedDict

NOT_STEP = ("init_table_kernel", "at::", "gather_rows_kernel", "row_count_hist", "probe_gather")


def main():
    src, out, header = sys.argv[1], sys.argv[2], sys.argv[3]
    rows = [r for r in csv.reader(open(src)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = OrderedDict()
    for r in rows[1:]:
        name = re.sub(r"\(.*", "", r[ki]).strip()
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        us = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0) * v
        n, tot = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, tot + us)
    step_total = sum(t for k, (n, t) in agg.items() if not any(s in k for s in NOT_STEP))
    with open(out, "w") as f:
        f.write(f"# {header}\n# kernel: launches, mean us, total us, share of step kernels (cold-cache, serialised)\n")
        for k, (n, t) in agg.items():
            share = "" if any(s in k for s in NOT_STEP) else f"{100 * t / step_total:6.1f}%"
            f.write(f"{k[:90]:90s} {n:5d} {t / n:10.1f} {t:10.1f} {share}\n")
    print(open(out).read())


if __name__ == "__main__":
    main()
