"""Top stall-sampled SASS lines of one kernel from `ncu --page source --csv` output."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
hi = next(i for i, r in enumerate(rows) if 'Source' in r and 'Address' in r)
hdr = rows[hi]
i_src, i_s = hdr.index('Source'), hdr.index('Warp Stall Sampling (All Samples)')
data = [r for r in rows[hi + 1:] if len(r) > i_s and r[i_s].replace('.', '').isdigit()]
tot = sum(float(r[i_s]) for r in data) or 1
print(f"total samples {tot:.0f}")
for r in sorted(data, key=lambda r: -float(r[i_s]))[:n]:
    print(f"{100 * float(r[i_s]) / tot:5.1f}%  {r[0][-5:]} {r[i_src][:100]}")
