"""Map an ncu launch list of one eager traced c4 learner step (one CSV row per
kernel, in launch order) onto the traced phase labels (phase#k) and write
profiles/r02/ncu_traffic.json: {cfg: {label: dram bytes (read + write) of the
phase's main kernel}} plus the per-launch durations.

usage (on the GPU box):
  CFG=c4 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
      --clock-control none --csv --log-file gpurun_out/c4_launches.csv \\
      python scripts/traced_step.py
  python scripts/ncu_traffic.py gpurun_out/c4_launches.csv gpurun_out/c4_phase_names.json out.json
"""
import csv
import json
import sys

launches_csv, names_json, out = sys.argv[1], sys.argv[2], sys.argv[3]
rows = [r for r in csv.reader(open(launches_csv)) if r]
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, ui, vi = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"),
                  h.index("Metric Value"))
idi = h.index("ID")
kern = {}
order = []
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "usecond": 1.0, "us": 1.0,
         "msecond": 1e3}
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    k = int(r[idi])
    if k not in kern:
        kern[k] = {"name": r[ki]}
        order.append(k)
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    kern[k][r[mi]] = v
names = json.load(open(names_json))            # [(label, n_launches)] in phase order
total = sum(n for _, n in names)
order = order[-total:]                          # the last (profiled) step's kernels
out_d, seq, i = {}, [], 0
for label, n in names:
    ks = order[i:i + n]
    i += n
    main = max(ks, key=lambda k: kern[k].get("gpu__time_duration.sum", 0)) if ks else None
    if main is None:
        continue
    e = kern[main]
    out_d[label] = int(e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0))
    seq.append({"label": label, "kernels": [kern[k]["name"][:90] for k in ks],
                "us": round(sum(kern[k].get("gpu__time_duration.sum", 0) for k in ks), 2),
                "dram_bytes_main": out_d[label]})
json.dump({"c4": out_d, "launches": seq, "unmatched_kernels": len(order) - i}, open(out, "w"), indent=1)
print(f"{len(seq)} phases, {i} of {len(order)} kernels matched")
