#!/usr/bin/env python
"""Summarise an ncu --set full report (.ncu-rep) for profiles/:

    python tools/ncu_summary.py report.ncu-rep [algorithmic_bytes_per_launch ...]

Per captured kernel: duration, DRAM bytes read + written (the roofline
`traffic`), DRAM / SM throughput, issue activity, occupancy, registers, the
pipe utilisations that matter for integer Montgomery work (ALU, FMA, IMAD
issue via the FMA-heavy pipe) and the top warp stall reasons.  When
algorithmic bytes per launch are given (one per kernel, in capture order),
the achieved algorithmic GB/s and traffic / algorithmic ratio are printed.
"""
import csv
import subprocess
import sys

KEEP = [
    ("Duration", "duration"),
    ("DRAM Throughput", "dram_pct"),
    ("Memory Throughput", "mem"),
    ("Compute (SM) Throughput", "sm_pct"),
    ("Issue Slots Busy", "issue_pct"),
    ("Executed Ipc Active", "ipc"),
    ("Achieved Occupancy", "occ_pct"),
    ("Theoretical Occupancy", "occ_theory_pct"),
    ("Registers Per Thread", "regs"),
    ("Block Size", "block"),
    ("Grid Size", "grid"),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def details(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ik, iname, iu, iv = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"),
                         h.index("Metric Value"))
    iid = h.index("ID")
    per = {}
    for r in rows[1:]:
        d = per.setdefault(r[iid], {"kernel": r[ik]})
        for name, key in KEEP:
            if r[iname] == name and key not in d:
                d[key] = (r[iv], r[iu])
    return [per[k] for k in sorted(per, key=int)]


def main():
    path = sys.argv[1]
    algo = [float(x) for x in sys.argv[2:]]
    hdr, units, rows = raw(path)

    def col(r, name):
        return float(r[hdr.index(name)]) if name in hdr and r[hdr.index(name)] else 0.0

    unit_scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    dets = details(path)
    for i, (r, d) in enumerate(zip(rows, dets)):
        rb = col(r, "dram__bytes_read.sum") * unit_scale.get(units[hdr.index("dram__bytes_read.sum")], 1)
        wb = col(r, "dram__bytes_write.sum") * unit_scale.get(units[hdr.index("dram__bytes_write.sum")], 1)
        dur_ns = col(r, "gpu__time_duration.sum")
        du = units[hdr.index("gpu__time_duration.sum")]
        dur_s = dur_ns * {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9,
                          "us": 1e-6, "ms": 1e-3, "s": 1.0}.get(du, 1e-9)
        print("kernel %d: %s" % (i, d["kernel"][:150]))
        print("  duration %.2f us   grid %s block %s   regs %s" % (
            dur_s * 1e6, d.get("grid", ("?",))[0], d.get("block", ("?",))[0],
            d.get("regs", ("?",))[0]))
        print("  DRAM read %.1f MB + write %.1f MB = traffic %.1f MB  (%.0f GB/s)" % (
            rb / 1e6, wb / 1e6, (rb + wb) / 1e6, (rb + wb) / dur_s / 1e9 if dur_s else 0))
        for key in ("dram_pct", "sm_pct", "issue_pct", "ipc", "occ_pct", "occ_theory_pct"):
            if key in d:
                print("  %-15s %s %s" % (key, d[key][0], d[key][1]))
        seen, pipes = set(), []
        for n in hdr:
            if n.startswith("sm__inst_executed_pipe_") and n.endswith("pct_of_peak_sustained_active"):
                short = n.replace("sm__inst_executed_pipe_", "").split(".")[0]
                if short not in seen:
                    seen.add(short)
                    pipes.append((n, col(r, n)))
        pipes = sorted(pipes, key=lambda x: -x[1])[:5]
        if pipes:
            print("  pipes (% of peak): " + ", ".join(
                "%s %.1f" % (n.replace("sm__inst_executed_pipe_", "").split(".")[0], v)
                for n, v in pipes))
        pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
        stalls = [(n, col(r, n)) for n in hdr if n.startswith(pre) and n.endswith(suf)]
        stalls = sorted(stalls, key=lambda x: -x[1])[:4]
        if stalls:
            print("  top stalls (warps per issue): " + ", ".join(
                "%s %.2f" % (n[len(pre):-len(suf)], v) for n, v in stalls))
        if i < len(algo) and dur_s:
            print("  algorithmic %.1f MB -> %.0f GB/s; traffic / algorithmic = %.2f" % (
                algo[i] / 1e6, algo[i] / dur_s / 1e9, (rb + wb) / algo[i]))


if __name__ == "__main__":
    main()
