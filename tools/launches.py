"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list:
python tools/launches.py FILE [first_id]"""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("ID")
first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tot = 0.0
for r in rows[1:]:
    i = int(r[ii])
    if i < first:
        continue
    v = float(r[vi].replace(",", "")) / 1e3
    tot += v
    print(f"{i:5d} {r[ki][:60]:60s} {v:10.1f} us")
print(f"total {tot:.1f} us")
