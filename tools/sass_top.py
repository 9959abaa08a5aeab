"""Top SASS instructions of an `ncu --page source --csv --print-source sass` dump by stall samples (dev tool)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 32
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
ci = {c: i for i, c in enumerate(h)}
body = [r for r in rows[hi + 1:] if len(r) >= len(h) - 2]
tot = sum(float(r[ci["# Samples"]] or 0) for r in body)
stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
agg = {}
for r in body:
    for c in stalls:
        agg[c] = agg.get(c, 0) + float(r[ci[c]] or 0)
print("stall mix:", ", ".join(f"{k[6:]} {100 * v / tot:.0f}%" for k, v in sorted(agg.items(), key=lambda a: -a[1]) if v / tot > 0.01))
print("instructions", sum(float(r[ci["Instructions Executed"]] or 0) for r in body),
      "smem wavefronts", sum(float(r[ci["L1 Wavefronts Shared"]] or 0) for r in body),
      "ideal", sum(float(r[ci["L1 Wavefronts Shared Ideal"]] or 0) for r in body))
idx = sorted(range(len(body)), key=lambda i: -float(body[i][ci["# Samples"]] or 0))[:top]
for i in sorted(idx):
    r = body[i]
    st = sorted(((float(r[ci[c]] or 0), c[6:]) for c in stalls), reverse=True)[:2]
    print(f"{i:5d} {100 * float(r[ci['# Samples']]) / tot:5.1f}% {r[1][:64]:64s} wf={r[ci['L1 Wavefronts Shared']]}/{r[ci['L1 Wavefronts Shared Ideal']]} ",
          " ".join(f"{n}:{100 * v / tot:.1f}" for v, n in st if v))
