"""Development tool: top sampled SASS instructions of an ncu source-page CSV
(ncu -i rep --page source --csv --print-source sass), with stall reasons."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
idx = {x: i for i, x in enumerate(h)}
stalls = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
body = rows[2:]
tot = sum(int(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in body)
print("total samples", tot)
lim = int(sys.argv[2]) if len(sys.argv) > 2 else 40
order = sorted(range(len(body)), key=lambda i: -int(body[i][idx["Warp Stall Sampling (All Samples)"]] or 0))
for i in sorted(order[:lim]):
    r = body[i]
    smp = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    st = ", ".join(f"{s[6:]}={r[idx[s]]}" for s in stalls if r[idx[s]] not in ("0", ""))
    print(f"{i:5d} {smp:6d} ex={r[idx['Instructions Executed']]:>8s}  {r[idx['Source']].strip()[:60]:60s} {st}")
