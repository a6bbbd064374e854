"""Top SASS instructions of an ncu report by executed count and stall samples."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
ie = hdr.index("Instructions Executed")
ws = hdr.index("Warp Stall Sampling (All Samples)")
pt = hdr.index("Avg. Predicated-On Threads Executed")
f = lambda x: float(x) if x not in ("", "-") else 0.0
tot = sum(f(r[ie]) for r in data)
stot = sum(f(r[ws]) for r in data)
print(f"total warp-instr {tot:.0f}, stall samples {stot:.0f}")
key = sys.argv[2] if len(sys.argv) > 2 else "inst"
col = ie if key == "inst" else ws
for i, r in enumerate(data):
    r.append(i)
for r in sorted(data, key=lambda r: -f(r[col]))[:int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
    print(f"{r[-1]:5d} inst={f(r[ie]):10.0f} stall={f(r[ws]):7.0f} thr={f(r[pt]):5.1f}  {r[1].strip()[:70]}")
