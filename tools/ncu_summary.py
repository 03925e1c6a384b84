#!/usr/bin/env python
"""Summarise ncu captures for profiles/.

    python tools/ncu_summary.py gpurun_out/prof_gemm.ncu-rep [more.ncu-rep ...] > profiles/rNN_ncu_summary.txt
    python tools/ncu_summary.py --launches gpurun_out/launches.csv

For --set full captures: per kernel, duration, DRAM bytes, DMMA pipe %,
occupancy, top stall reasons.  With --traffic FILE also writes the per-launch
DRAM bytes keyed by bench.py's kernel names (gemm_stage<i> in launch order of
one step, fbuild) so bench.py can report roofline.traffic.
"""

from __future__ import annotations

import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "dmma_pipe_pct"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_pct"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem_ld_conflicts"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def to_bytes(val, unit):
    v = float(val.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return v * scale


def summarise(rep):
    hdr, units, rows = raw(rep)
    col = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_")
                  and h.endswith("_per_issue_active.ratio")]
    out = []
    for r in rows:
        rec = {"kernel": r[col["Kernel Name"]]}
        for k, name in KEYS:
            if k in col and r[col[k]] != "":
                rec[name] = r[col[k]] + " " + units[col[k]]
        if "dram__bytes_read.sum" in col:
            rec["dram_bytes"] = (to_bytes(r[col["dram__bytes_read.sum"]], units[col["dram__bytes_read.sum"]])
                                 + to_bytes(r[col["dram__bytes_write.sum"]], units[col["dram__bytes_write.sum"]]))
        stalls = sorted(((float(r[col[h]] or 0), h.replace("smsp__average_warps_issue_stalled_", "")
                          .replace("_per_issue_active.ratio", "")) for h in stall_cols), reverse=True)
        rec["top_stalls"] = [f"{n}={v:.2f}" for v, n in stalls[:5] if v > 0.05]
        out.append(rec)
    return out


def launches(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        name = re.sub(r"\(CUtensorMap_st.*|\(cg::.*", "", r[ki])
        v = float(r[vi].replace(",", ""))
        v = v / 1e3 if r[ui] in ("ns", "nsecond") else v * 1e3 if r[ui] in ("ms", "msecond") else v
        tot[name] += v
        cnt[name] += 1
    grand = sum(tot.values())
    lines = [f"{'kernel':90s} {'launches':>8s} {'total_us':>10s} {'avg_us':>9s} {'share':>6s}"]
    for name, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"{name[:90]:90s} {cnt[name]:8d} {v:10.1f} {v / cnt[name]:9.2f} {v / grand:6.1%}")
    return "\n".join(lines)


def main(argv):
    if argv and argv[0] == "--launches":
        print(launches(argv[1]))
        return
    traffic_out = None
    if "--traffic" in argv:
        i = argv.index("--traffic")
        traffic_out = argv[i + 1]
        argv = argv[:i] + argv[i + 2:]
    traffic = {}
    for rep in argv:
        print(f"# {rep}")
        for rec in summarise(rep):
            print(json.dumps(rec))
            k = rec["kernel"]
            key = "fbuild" if "fbuild" in k else None
            if key is None and "gemm_f64_kernel" in k:
                key = k
            if key and "dram_bytes" in rec:
                traffic.setdefault(key, rec["dram_bytes"])
    if traffic_out:
        with open(traffic_out, "w") as f:
            json.dump(traffic, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])
