#!/usr/bin/env python3
"""Summarise a tools/ncu_capture.sh export: headline metrics, stall reasons,
instruction mix and the source lines with most executed instructions.
python tools/ncu_summary.py gpurun_out/NAME [--lines 30]"""
import collections
import csv
import gzip
import re
import sys


def rows(path):
    op = gzip.open if path.endswith(".gz") else open
    with op(path, "rt") as f:
        return list(csv.reader(f))


def main():
    base = sys.argv[1]
    nlines = int(sys.argv[sys.argv.index("--lines") + 1]) if "--lines" in sys.argv else 30
    raw = rows(base + "_raw.csv")
    h = raw[0]
    units = dict(zip(h, raw[1]))
    for r in raw[2:]:
        d = dict(zip(h, r))
        print(d["Kernel Name"][:80])
        for k, lab in [("gpu__time_duration.sum", "duration"),
                       ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue busy %"),
                       ("sm__warps_active.avg.per_cycle_active", "warps/SM"),
                       ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
                       ("smsp__inst_executed.sum", "warp inst"),
                       ("dram__bytes_read.sum", "DRAM read"), ("dram__bytes_write.sum", "DRAM write"),
                       ("launch__registers_per_thread", "regs")]:
            if k in d:
                print(f"  {lab:14s} {d[k]} {units.get(k, '')}".rstrip())
        st = sorted(((k, float(v or 0)) for k, v in d.items()
                     if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")),
                    key=lambda kv: -kv[1])
        print("  stalls/issue: " + ", ".join(f"{k[34:-23]} {v:.2f}" for k, v in st[:8]))
    sass = [r for r in rows(base + "_sass.csv.gz") if len(r) > 6 and r[0].startswith("0x")]
    tot = sum(int(r[5] or 0) for r in sass)
    op = collections.Counter()
    for r in sass:
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[1])
        op[m.group(2) if m else r[1]] += int(r[5] or 0)
    print("instruction mix: " + ", ".join(f"{o} {100 * n / tot:.1f}%" for o, n in op.most_common(16)))
    agg = {}
    for r in rows(base + "_src.csv.gz"):
        if len(r) > 8 and r[0] not in ("", "Line No", "File Path", "Function Name"):
            try:
                agg[int(r[0])] = (int(r[7]), int(r[4]), r[1].strip()[:90])
            except ValueError:
                pass
    t = sum(v[0] for v in agg.values())
    s = sum(v[1] for v in agg.values())
    print(f"top source lines by executed warp instructions (of {t}), with stall-sample share:")
    for ln, (n, smp, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:nlines]:
        print(f"  {ln:5d} {100 * n / t:5.2f}%  st {100 * smp / s:5.2f}%  {src}")


if __name__ == "__main__":
    main()
