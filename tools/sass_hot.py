"""Top SASS instructions of one kernel by warp-stall samples, with their
dominant stall reasons (dev tool).

  ncu -i rep --page source --csv --print-source cuda,sass --kernel-name regex:K \
      --launch-skip S --launch-count 1 > mix.csv
  python tools/sass_hot.py mix.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr_i = [i for i, r in enumerate(rows) if r and r[0] == "Line No"]
h = rows[hdr_i[0]]
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
seen = {}
for r in rows[hdr_i[0] + 1:]:
    if len(r) < len(h) or not r[2].startswith("0x"):
        continue
    if r[2] in seen:
        continue
    seen[r[2]] = r
tot = {}
allsamp = 0
for r in seen.values():
    for i in stall_cols:
        v = float(r[i] or 0)
        tot[h[i]] = tot.get(h[i], 0) + v
        allsamp += v
print("stall mix:", ", ".join(f"{k[6:]} {100 * v / allsamp:.0f}%" for k, v in sorted(tot.items(), key=lambda a: -a[1])
                              if v / allsamp > 0.01))
items = sorted(seen.values(), key=lambda r: -float(r[4] or 0))
for r in items[:top]:
    st = sorted(((float(r[i] or 0), h[i][6:]) for i in stall_cols), reverse=True)[:2]
    print(f"{100 * float(r[4] or 0) / allsamp:5.1f}% {r[2][-5:]} {r[3][:60]:60s} " +
          " ".join(f"{n}:{100 * v / allsamp:.1f}" for v, n in st if v))
