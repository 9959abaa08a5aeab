"""Aggregate an ncu --page source --print-source cuda,sass CSV by CUDA source
line (dev tool): warp-stall samples and executed warp instructions per line.

  python tools/src_hot.py <mix.csv> [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname = None
hdr = None
agg = []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or not r[0]:
        continue
    try:
        samp = int(r[4]); ins = int(r[7])
    except ValueError:
        continue
    agg.append((samp, ins, f"{fname}:{r[0]}", r[1].strip()[:90]))
ts = sum(a[0] for a in agg) or 1
ti = sum(a[1] for a in agg) or 1
print(f"total samples {ts}, warp instructions {ti:.3e}")
for s, i, loc, src in sorted(agg, reverse=True)[:top]:
    print(f"{100*s/ts:5.1f}% smp {100*i/ti:5.1f}% ins  {loc:26s} {src}")
