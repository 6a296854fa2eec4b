#!/usr/bin/env python
"""Summarise ncu outputs brought back in gpurun_out/ into profiles/ (committed).

  python tools/ncu_summary.py launches <launches.csv> <out.txt>
      per-kernel launch counts, summed / average device time and share of the
      captured launches (gpu__time_duration.sum pass: cold-cache, serialised).
  python tools/ncu_summary.py report <file.ncu-rep> <out.txt> [--filter name-substring]
                                     [--traffic profiles/traffic.json --key prec:class]
      key metrics of a `ncu --set full` capture (time, DRAM bytes, L2/L1 hit
      rates, throughput %, tensor-pipe activity, occupancy) per captured launch;
      optionally records the mean DRAM read+write bytes per launch as `traffic`.
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "smsp__average_warp_latency_issue_stalled_long_scoreboard",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    unit = ""
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        unit = r[ui]
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    lines = [f"# ncu gpu__time_duration.sum launch list ({path}); cold-cache, serialised: compare SHARES",
             f"# {sum(v[0] for v in agg.values())} launches, total {tot:.0f} {unit}",
             f"{'kernel':64s} {'launches':>8s} {'sum_'+unit:>14s} {'avg_'+unit:>12s} {'share':>6s}"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{k:64s} {v[0]:8d} {v[1]:14.0f} {v[1] / v[0]:12.1f} {v[1] / tot:6.3f}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def report(path, out, traffic=None, key=None, flt=None):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u = rows[0], rows[1]
    lines = [f"# ncu --set full summary of {os.path.basename(path)}"]
    dram = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        if flt and flt not in name:
            continue
        lines.append(f"== {name}  grid={r[h.index('Grid Size')] if 'Grid Size' in h else '?'} "
                     f"block={r[h.index('Block Size')] if 'Block Size' in h else '?'}")
        b = 0.0
        for m in METRICS:
            if m in h:
                i = h.index(m)
                lines.append(f"   {m:90s} {r[i]:>14s} {u[i]}")
                if m.startswith("dram__bytes"):
                    try:
                        b += float(r[i].replace(",", "")) * SCALE.get(u[i], 1)
                    except ValueError:
                        pass
        lines.append(f"   dram read+write bytes per launch: {b:.0f}")
        dram.append(b)
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic and key and dram:
        d = json.load(open(traffic)) if os.path.exists(traffic) else {}
        d[key] = sum(dram) / len(dram)
        json.dump(d, open(traffic, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        kw = {}
        if "--filter" in sys.argv:
            kw["flt"] = sys.argv[sys.argv.index("--filter") + 1]
        if "--traffic" in sys.argv:
            kw["traffic"] = sys.argv[sys.argv.index("--traffic") + 1]
            kw["key"] = sys.argv[sys.argv.index("--key") + 1]
        report(sys.argv[2], sys.argv[3], **kw)
