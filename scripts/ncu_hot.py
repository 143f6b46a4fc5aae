"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
ia, isrc, iss = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[iss] or 0) for r in data if len(r) > iss)
top = sorted((r for r in data if len(r) > iss), key=lambda r: -float(r[iss] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
print("total samples", tot)
for r in top:
    print(f"{float(r[iss])/tot*100:5.1f}%  {r[ia]}  {r[isrc][:90]}")
