"""Top CUDA source lines of an ncu report by warp-stall samples
(`--print-source cuda,sass` CSV): python tools/ncu_src_hot.py REPORT [N]"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r)
hdr = rows[hi]
ws = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
f = lambda x: float(x) if x not in ("", "-") else 0.0
data = [r for r in rows[hi + 1:] if len(r) == len(hdr) and r[2] == "-"]  # cuda-line rows
tot = sum(f(r[ws]) for r in data)
print(f"stall samples {tot:.0f}")
for r in sorted(data, key=lambda r: -f(r[ws]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{r[0]:>5s} {100 * f(r[ws]) / tot:5.1f}%  inst={f(r[ie]):11.0f}  {r[1].strip()[:90]}")
