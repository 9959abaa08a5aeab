"""Summarise ncu outputs into profiles/ (dev tool).

  python tools/ncu_summary.py <launches.csv> <full.ncu-rep> <tag>

Writes profiles/<tag>_launches.md (per-kernel device time share of one apply,
cold-cache serialised ncu times), profiles/<tag>_kernels.md (key --set full
metrics of the hot kernels) and profiles/ncu_traffic.json (DRAM bytes per
launch by apply stage, read by bench.py for roofline.traffic)."""
import csv
import json
import os
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
launches, rep, tag = sys.argv[1], sys.argv[2], sys.argv[3]

rows = list(csv.reader(open(launches)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
data = [dict(zip(h, r)) for r in rows[hdr + 1:] if len(r) == len(h)]
by_id = OrderedDict()
for d in data:
    e = by_id.setdefault(d["ID"], {"name": d["Kernel Name"]})
    try:
        e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    except ValueError:
        pass
launch = list(by_id.values())
# one apply = the launches between two consecutive k_gather_mul
starts = [i for i, e in enumerate(launch) if "k_gather_mul" in e["name"]]
one = launch[starts[-2]:starts[-1]] if len(starts) >= 2 else launch
stage_names = ["spread_src", "interp_xi", "spmv", "spread_xi", "interp_tgt"]
total = sum(e.get("gpu__time_duration.sum", 0) for e in one)
lines = [f"# ncu launch list, one apply ({tag})", "",
         "`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
         "--clock-control none` on `tools/prof_apply.py` (config 4, N=1e7). Cold-cache, "
         "serialised per launch: compare shares, not absolute times.", "",
         "| # | kernel | time (us) | share | DRAM read (MB) | DRAM write (MB) |", "|---|---|---|---|---|---|"]
traffic = {}
stage_iter = iter(stage_names)
for i, e in enumerate(one):
    t = e.get("gpu__time_duration.sum", 0)
    unit_scale = 1e-3  # ns -> us
    rd = e.get("dram__bytes_read.sum", 0)
    wr = e.get("dram__bytes_write.sum", 0)
    nm = e["name"].split("(")[0][:70]
    lines.append(f"| {i} | `{nm}` | {t * unit_scale:.1f} | {100 * t / total:.1f}% | {rd / 1e6:.1f} | {wr / 1e6:.1f} |")
    if any(k in e["name"] for k in ("k_spread_mma", "k_spread_cta", "k_interp", "k_spmv_vec")):
        try:
            traffic[next(stage_iter)] = rd + wr
        except StopIteration:
            pass
lines.append(f"| | **total** | {total * 1e-3:.1f} | 100% | | |")
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
open(os.path.join(ROOT, "profiles", f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")
json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h = r[0]
want = [("gpu__time_duration.sum", "duration (ms)"),
        ("dram__bytes_read.sum", "DRAM read (GB)"), ("dram__bytes_write.sum", "DRAM write (GB)"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
        ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 % peak"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
        ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
        ("launch__registers_per_thread", "regs/thread"),
        ("smsp__inst_executed.sum", "warp instr")]
out = [f"# ncu --set full, hot kernels of one apply ({tag})", "",
       "`ncu --set full --clock-control none -k regex:\"k_interp|k_spread_cta|k_spmv_vec\"` "
       "on `tools/prof_apply.py` (config 4), second apply.", "",
       "| kernel | " + " | ".join(w[1] for w in want) + " |", "|---" * (len(want) + 1) + "|"]
for row in r[2:]:
    d = dict(zip(h, row))
    vals = []
    for k, _ in want:
        v = d.get(k, "")
        try:
            f = float(v.replace(",", ""))
            if k == "gpu__time_duration.sum":
                f *= 1e-6  # ns -> ms
            elif k.startswith("dram__bytes"):
                f *= 1e-9  # B -> GB
            vals.append(f"{f:.3g}")
        except ValueError:
            vals.append(v)
    out.append(f"| `{d.get('Kernel Name', '')[:48]}` | " + " | ".join(vals) + " |")
open(os.path.join(ROOT, "profiles", f"{tag}_kernels.md"), "w").write("\n".join(out) + "\n")
# per-stage pipe utilisation of the --set full capture (in apply order: the
# capture's launches are spread_src, interp_xi, spmv, spread_xi, interp_tgt),
# read by bench.py beside the HBM fraction
pipes = {}
for st_name, row in zip(stage_names, r[2:]):
    d = dict(zip(h, row))

    def num(k):
        try:
            return round(float(d.get(k, "").replace(",", "")), 1)
        except ValueError:
            return None
    pipes[st_name] = {"dmma_pct": num("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
                      "fp64_pct": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                      "issue_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                      "l1_pct": num("l1tex__throughput.avg.pct_of_peak_sustained_active"),
                      "dram_pct": num("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")}
json.dump({"source": f"profiles/{tag}_kernels.md (ncu --set full, config 4)", "pipes": pipes},
          open(os.path.join(ROOT, "profiles", "ncu_pipes.json"), "w"), indent=1)
print("\n".join(lines[-12:]))
print("\n".join(out))
