"""Summarise an ncu --csv metrics log: per kernel, per launch, metric values."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Name" in r)
h = rows[hdr]
ki, mi, ui, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
out = {}
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    out.setdefault((r[ii], r[ki][:50]), []).append((r[mi], r[vi], r[ui]))
for (i, k), ms in out.items():
    print(f"[{i}] {k}")
    for m, v, u in ms:
        print(f"      {m:75s} {v:>22s} {u}")
