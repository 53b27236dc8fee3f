"""Summarise the committed ncu captures into profiles/<round>/*.md / *.json.

    python scripts/summarize_profiles.py gpurun_out/launches_r01.csv gpurun_out/prof_r01.ncu-rep profiles/r01
"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict

launches, rep, outdir = sys.argv[1:4]

# ---- launch list: per-kernel device time of one learner step (cold cache, serialised)
rows = list(csv.reader(open(launches)))
hdr_i = next(i for i, r in enumerate(rows) if r and "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
times = []
for r in rows[hdr_i + 1:]:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        times.append((r[ki], float(r[vi].replace(",", ""))))
def short(n):
    m = re.search(r"seed::(\w+)<.*?seed::(\w+)>", n)
    if m:
        return f"{m.group(1)}<{m.group(2)}>"
    m = re.search(r"(\w+)<([^>]*)>\(", n)
    if m:
        return f"{m.group(1)}<{m.group(2).replace('seed::', '').strip()}>"
    m = re.search(r"(\w+)\(", n)
    return m.group(1) if m else n[:60]
agg = defaultdict(lambda: [0, 0.0])
for n, t in times:
    a = agg[short(n)]
    a[0] += 1
    a[1] += t
tot = sum(v[1] for v in agg.values())
lines = ["| kernel | launches | total (ns units as ncu) | share |", "|---|---|---|---|"]
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    lines.append(f"| {k} | {c} | {t:.0f} | {t / tot:.3f} |")
open(f"{outdir}/ncu_launch_list.md", "w").write(
    "# ncu launch list (gpu__time_duration.sum, --clock-control none)\n\n"
    f"Source: `{launches}` from `ncu --metrics gpu__time_duration.sum --clock-control none -c 400 "
    "python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extra` (cold-cache, serialised "
    "launches: compare shares, not absolutes; includes the bench's warm-up and e2e steps).\n\n"
    + "\n".join(lines) + "\n")

# ---- full-set capture: per-kernel DRAM traffic and headline metrics
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--kernel-name-base", "demangled"],
                     capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h, units = rr[0], rr[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3}
out = {}
md = ["| kernel | duration (us) | DRAM read+write (MB) | SM % | mem % | tensor pipe % | grid | regs |",
      "|---|---|---|---|---|---|---|---|"]
for r in rr[2:]:
    name = short(r[h.index("Kernel Name")])
    def get(k):
        if k not in h:
            return None
        i = h.index(k)
        try:
            return float(r[i].replace(",", "")) * scale.get(units[i], 1)
        except ValueError:
            return None
    d = get("gpu__time_duration.sum")
    br, bw = get("dram__bytes_read.sum") or 0, get("dram__bytes_write.sum") or 0
    tp = get("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed")
    if tp is None:
        tp = get("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed")
    ent = dict(us=d, dram_bytes=br + bw, sm_pct=get("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
               mem_pct=get("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"),
               tensor_pct=tp, grid=get("launch__grid_size"), regs=get("launch__registers_per_thread"))
    out.setdefault(name, []).append(ent)
    md.append(f"| {name} | {d:.1f} | {(br + bw) / 1e6:.2f} | {ent['sm_pct']:.1f} | {ent['mem_pct']:.1f} | "
              f"{tp if tp is not None else '-'} | {ent['grid']:.0f} | {ent['regs']:.0f} |")
json.dump(out, open(f"{outdir}/ncu_full.json", "w"), indent=1)
open(f"{outdir}/ncu_full.md", "w").write(
    "# ncu --set full captures (round 1)\n\n"
    f"Source: `{rep}` (`ncu --set full --import-source on --clock-control none --launch-skip 24 "
    "-c 24 python scripts/step_c2.py 2`: every kernel of the second eager c2 learner step, B=32 "
    "T=20; cold cache per replay).  The DRAM column is the "
    "`traffic` figure bench.py reports for the dominant kernel.\n\n" + "\n".join(md) + "\n")
print(open(f"{outdir}/ncu_full.md").read())
print(open(f"{outdir}/ncu_launch_list.md").read()[:3000])
