"""Stall-reason breakdown of an ncu source-page CSV (gzip): totals per reason and
per SASS region (blocks of N instructions), from the per-instruction sampling.
usage: python scripts/ncu_stalls.py <source.csv.gz> [region_size]"""
import collections
import csv
import gzip
import io
import sys

rows = list(csv.reader(io.TextIOWrapper(gzip.open(sys.argv[1]))))
reg = int(sys.argv[2]) if len(sys.argv) > 2 else 100
h, data = rows[1], rows[2:]
reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
idx = {r: h.index(r) for r in reasons}
ie = h.index("Instructions Executed")
tot = collections.Counter()
byreg = collections.defaultdict(collections.Counter)
for i, r in enumerate(data):
    for k, j in idx.items():
        v = float(r[j] or 0)
        tot[k] += v
        byreg[i // reg][k] += v
T = sum(tot.values()) or 1
print("total samples", T)
for k, v in tot.most_common():
    if v / T > 0.005:
        print(f"  {k:24s} {v / T * 100:5.1f}%")
print("regions (start: top reasons)")
for g in sorted(byreg, key=lambda g: -sum(byreg[g].values()))[:10]:
    s = sum(byreg[g].values())
    top = ", ".join(f"{k[6:]} {v / T * 100:.1f}" for k, v in byreg[g].most_common(3))
    first = data[g * reg][1].strip()[:40]
    print(f"  {g * reg:5d} {s / T * 100:5.1f}%  {top}   [{first}]")
