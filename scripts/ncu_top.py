"""Summarise an ncu report: per-kernel key metrics + top SASS stall lines."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
filt = sys.argv[2] if len(sys.argv) > 2 else None
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 12
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
        "--kernel-name-base", "demangled"]
if filt:
    args += ["-k", "regex:" + filt]
out = subprocess.run(args, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
sections, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        sections.append(cur)
    elif r and r[0] == "Address":
        cur["hdr"] = r
    elif cur is not None and "hdr" in cur:
        cur["rows"].append(r)
for s in sections:
    h = s["hdr"]
    si = h.index("Warp Stall Sampling (All Samples)")
    tot = sum(float(r[si] or 0) for r in s["rows"]) or 1
    print("==", s["name"][:150])
    for r in sorted(s["rows"], key=lambda r: -float(r[si] or 0))[:ntop]:
        print(f"  {float(r[si]) / tot * 100:5.1f}%  {r[1].strip()[:100]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--kernel-name-base", "demangled"]
                     + (["-k", "regex:" + filt] if filt else []), capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if rr:
    hdr = rr[0]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
            "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "lts__t_bytes.sum", "l1tex__t_bytes.sum",
            "smsp__average_warp_latency_issue_stalled_long_scoreboard",
            "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"]
    idx = [(k, hdr.index(k)) for k in keys if k in hdr]
    units = rr[1]
    for r in rr[2:]:
        print(r[hdr.index("Kernel Name")][:80])
        print("   " + "; ".join(f"{k.split('.')[0].split('__')[-1]}={r[i]} {units[i]}" for k, i in idx))
