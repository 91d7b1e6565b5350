"""Summarise an ncu SASS source page (csv): top instructions by stall samples
with their share of executed instructions.  Usage: ncu -i rep --page source --csv
--print-source sass > x.csv; python tools/sass_hot.py x.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ia, isrc = hdr.index("Address"), hdr.index("Source")
iexe = hdr.index("Instructions Executed")
istall = hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    if len(r) <= max(iexe, istall):
        continue
    try:
        data.append((r[ia], r[isrc], float(r[iexe] or 0), float(r[istall] or 0)))
    except ValueError:
        pass
tot_e = sum(d[2] for d in data)
tot_s = sum(d[3] for d in data)
print(f"total executed {tot_e:.3e}, stall samples {tot_s:.0f}")
for a, s, e, st in sorted(data, key=lambda d: -d[3])[:n]:
    print(f"{a:>6} {st/tot_s*100:5.1f}% exe {e/tot_e*100:5.2f}%  {s}")
