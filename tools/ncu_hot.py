"""Summarise an `ncu --page source --csv --print-source sass` dump: top SASS
lines by stall samples and the stall-reason totals (development tool)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) == len(hdr)]
tot = {}
for r in body:
    for h in hdr:
        if h.startswith("stall_") and "(Not Issued)" not in h:
            tot[h] = tot.get(h, 0) + int(r[ci[h]] or 0)
S = sum(int(r[ci["Warp Stall Sampling (All Samples)"]] or 0) for r in body)
print("total samples", S)
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:8]:
    print(f"  {k:28s} {v:8d} {100.0 * v / max(S, 1):5.1f}%")
top = sorted(body, key=lambda r: -int(r[ci["Warp Stall Sampling (All Samples)"]] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for r in top:
    print(f"{r[ci['Warp Stall Sampling (All Samples)']]:>7} {r[ci['Address']][-5:]} {r[ci['Source']].strip()[:80]}")
