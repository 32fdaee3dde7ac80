"""Per-kernel DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum) and
issue-slot utilisation from `ncu --set full` reports -> profiles/ncu_traffic.json, which
bench.py reports as roofline.traffic.  Launches shorter than --min-us (empty depth
chunks that return at entry) are ignored.
usage: python tools/ncu_traffic.py out.json rep1.ncu-rep [rep2.ncu-rep ...]"""
import csv
import io
import json
import subprocess
import sys

out = sys.argv[1]
agg = {}
for rep in sys.argv[2:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hdr, units = rr[0], rr[1]
    col = {h: i for i, h in enumerate(hdr)}

    def val(r, name):
        v = float(r[col[name]].replace(",", ""))
        u = units[col[name]]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "us": 1, "nsecond": 1e-3,
                    "ns": 1e-3, "msecond": 1e3, "ms": 1e3}.get(u, 1)

    for r in rr[2:]:
        name = r[col["Kernel Name"]].split("(")[0].split("<")[0].replace("void ", "").strip()
        t = val(r, "gpu__time_duration.sum")
        if t < 10:
            continue
        a = agg.setdefault(name, {"launches": 0, "bytes": 0.0, "us": 0.0, "issue": 0.0})
        a["launches"] += 1
        a["bytes"] += val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
        a["us"] += t
        a["issue"] += float(r[col["smsp__issue_active.avg.pct_of_peak_sustained_active"]]) / 100
res = {k: {"dram_bytes_per_launch": int(v["bytes"] / v["launches"]), "launches": v["launches"],
           "ncu_us_per_launch": round(v["us"] / v["launches"], 2),
           "issue_active": round(v["issue"] / v["launches"], 3)} for k, v in agg.items()}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
