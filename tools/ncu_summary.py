#!/usr/bin/env python
"""Summarise an `ncu --set full` report into profiles/ (text + ncu_traffic.json).

usage: python tools/ncu_summary.py <report.ncu-rep> <out.txt> [workload]
Maps kernel names to bench.py phases so bench.py can report `roofline.traffic`.
Each workload's entry is stamped with bench.sources_sha() of the sources the
capture ran on; bench.py ignores an entry whose stamp does not match.
"""
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 thru %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 thru %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM thru %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__occupancy_limit_registers", "occ limit regs (blocks)"),
    ("smsp__inst_executed.sum", "warp instr"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
]
# kernel-name prefix -> bench.py phase (several kernels of one phase in one
# step, e.g. the sort's upsweep/scan/downsweep of every pass, are summed)
PHASE = [("seg_reduce_kernel<1", "fwd_segreduce"), ("seg_reduce_kernel<0", "bwd_segreduce_adagrad"),
         ("seg_fixup_lane_kernel<1", "fwd_fixup"), ("seg_fixup_kernel<1", "fwd_fixup"),
         ("seg_fixup_long_kernel<1", "fwd_fixup"), ("seg_fixup_lane_kernel<0", "bwd_fixup"),
         ("seg_fixup_kernel<0", "bwd_fixup"), ("seg_fixup_long_kernel<0", "bwd_fixup"),
         ("bag_expand_kernel", "bag_expand"), ("sort_", "radix_sort")]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    workload = sys.argv[3] if len(sys.argv) > 3 else "cfg2"
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines, traffic = [f"# ncu --set full summary of {os.path.basename(rep)} ({workload})"], {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"]
        lines.append(f"\n## {name}  grid={d.get('Grid Size')} block={d.get('Block Size')}")
        vals = {}
        for m, label in METRICS:
            if m in hdr:
                u = units[hdr.index(m)]
                lines.append(f"  {label:26s} {d[m]:>20s} {u}")
                vals[m] = (d[m], u)

        def tobytes(v):
            x, u = float(v[0].replace(",", "")), v[1]
            return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)

        if "dram__bytes_read.sum" in vals:
            tot = tobytes(vals["dram__bytes_read.sum"]) + tobytes(vals["dram__bytes_write.sum"])
            lines.append(f"  {'dram bytes (r+w)':26s} {tot:20.0f} byte")
            for k, ph in PHASE:
                if name.startswith(k) or (" " + k) in name:
                    # the capture holds exactly one step (tools/measure_round.sh): sum per phase
                    e = traffic.setdefault(ph, {"dram_bytes_per_launch": 0.0, "kernels": 0,
                                                "summary": os.path.basename(out)})
                    e["dram_bytes_per_launch"] += tot
                    e["kernels"] += 1
                    break
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    tj = os.path.join(os.path.dirname(out), "ncu_traffic.json")
    from bench import sources_sha

    d = json.load(open(tj)) if os.path.exists(tj) else {}
    d[workload] = {"sources_sha": sources_sha(), "report": os.path.basename(rep), "kernels": traffic}
    json.dump(d, open(tj, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
