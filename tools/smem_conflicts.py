"""Shared-memory wavefronts vs ideal per SASS instruction kind (dev tool).

  python tools/smem_conflicts.py mix.csv  (ncu --page source --csv --print-source cuda,sass)"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
h = rows[hi]
ci = {c: i for i, c in enumerate(h)}
seen = {}
for r in rows[hi + 1:]:
    if len(r) < len(h) or not r[2].startswith("0x"):
        continue
    seen.setdefault(r[2], r)
f = lambda r, k: float(r[ci[k]] or 0)  # noqa: E731
tot = sum(f(r, "L1 Wavefronts Shared") for r in seen.values())
print(f"shared wavefronts {tot:.3e} (ideal {sum(f(r, 'L1 Wavefronts Shared Ideal') for r in seen.values()):.3e})")
top = sorted(seen.values(), key=lambda r: -f(r, "L1 Wavefronts Shared"))[:15]
for r in top:
    n = f(r, "Instructions Executed") or 1
    print(f"{f(r, 'L1 Wavefronts Shared') / tot * 100:5.1f}%  wf/instr {f(r, 'L1 Wavefronts Shared') / n:5.2f} "
          f"ideal {f(r, 'L1 Wavefronts Shared Ideal') / n:5.2f}  L{r[0]:>5} {r[3][:70]}")
