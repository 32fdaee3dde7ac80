"""Summarise ncu outputs into profiles/: launch-list shares and key --set full metrics.
usage: python tools/ncu_summary.py <launches.csv> <prof.ncu-rep|-> <out.md> [title]"""
import collections, csv, io, subprocess, sys

launches, rep, out = sys.argv[1], sys.argv[2], sys.argv[3]
title = sys.argv[4] if len(sys.argv) > 4 else "profile"
lines = [f"# {title}", ""]
rows = list(csv.reader(open(launches)))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr, data = rows[h], rows[h + 1:]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in data:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        name = r[ki].split("(")[0][:70]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", ""))
tot = sum(v[1] for v in agg.values())
lines += ["## Launch list (ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised)", "",
          "| kernel | launches | total us | avg us | share |", "|---|---|---|---|---|"]
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append(f"| `{k}` | {v[0]} | {v[1]/1e3:.1f} | {v[1]/1e3/v[0]:.1f} | {100*v[1]/tot:.1f}% |")
if rep != "-":
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hdr, units = rr[0], rr[1]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]
    idx = [hdr.index(w) if w in hdr else -1 for w in want]
    lines += ["", "## ncu --set full (per captured launch)", "",
              "| " + " | ".join(w.replace("avg.pct_of_peak_sustained_", "% ") for w in want) + " |",
              "|" + "---|" * len(want)]
    for r in rr[2:]:
        cells = []
        for i in idx:
            if i < 0:
                cells.append("NA")
            else:
                v = r[i]
                cells.append((v.split("(")[0][:48]) if hdr[i] == "Kernel Name" else f"{v} {units[i]}")
        lines.append("| " + " | ".join(cells) + " |")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:40]))
