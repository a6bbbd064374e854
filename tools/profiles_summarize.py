"""Turn a tools/gpu_profiles.sh run (gpurun_out/prof_rNN/) into the committed
evidence under profiles/rNN/: the bench launch list (raw CSV + per-kernel share
of the step), one text summary per `ncu --set full` capture (key metrics, stall
reasons, hottest source lines) next to the .ncu-rep, the cooperative-kernel
level logs, and profiles/pagerank_ncu.json (DRAM bytes of one k_pr_rows launch,
read by bench.py for roofline.traffic).

    python tools/profiles_summarize.py r01
"""
import csv
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from ncu_summary import summarize  # noqa: E402


def launch_table(src, dst_txt, header):
    rows = [r for r in csv.reader(open(src)) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        k = r[ki].split("(")[0]
        agg[k][0] += 1
        agg[k][1] += float(r[vi].replace(",", "")) / 1e3
    tot = sum(t for _, t in agg.values())
    with open(dst_txt, "w") as f:
        f.write(header)
        f.write(f"{'kernel':70s} {'launches':>8s} {'total_us':>12s} {'avg_us':>10s} {'share':>7s}\n")
        for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"{k[:70]:70s} {c:8d} {t:12.1f} {t / c:10.1f} {100 * t / tot:6.2f}%\n")


def full_summary(rep, dst_txt):
    out = []
    for name, m, stalls in summarize(rep):
        out.append(f"== {name[:110]}")
        for k, (v, u) in m.items():
            out.append(f"  {k:60s} {v} {u}")
        out.append("  stalls: " + ", ".join(f"{n}={v:.2f}" for v, n in stalls))
    hot = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_src_hot.py"), rep,
                          "15"], capture_output=True, text=True).stdout
    out.append("\n-- hottest CUDA source lines (warp-stall samples)")
    out.append(hot)
    with open(dst_txt, "w") as f:
        f.write("\n".join(out) + "\n")
    return summarize(rep)


def main():
    r = sys.argv[1] if len(sys.argv) > 1 else "r01"
    src = os.path.join(ROOT, "gpurun_out", f"prof_{r}")
    dst = os.path.join(ROOT, "profiles", r)
    os.makedirs(dst, exist_ok=True)
    common = ("# Cold, serialised launches: the SHARE of each kernel is what compares with\n"
              "# the bench, not the absolute.  The whole process is listed (graph\n"
              "# generation, plan builds, the e2e leg and the CPU-baseline setup included).\n")
    heads = {
        "bench_pagerank_launches": "# ncu --metrics gpu__time_duration.sum --clock-control none launch list of\n"
                                   "# `python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-secondary`\n"
                                   "# (PageRank runs as ONE persistent\n"
                                   "# cooperative kernel per step, k_pr_persist: row phase + long-row finish\n"
                                   "# + L1 reduction per iteration).\n" + common,
        "bench_pagerank_launches_split": "# the same with --option pagerank.host_loop=1: the same row / finish code launched as\n"
                                         "# one k_pr_rows + k_pr_finish pair per iteration, splitting the shares.\n"
                                         + common,
    }
    for base, head in heads.items():
        lc = os.path.join(src, base + ".csv")
        if os.path.exists(lc):
            shutil.copy(lc, dst)
            launch_table(lc, os.path.join(dst, base + ".txt"), head)
    for fn in sorted(os.listdir(src)):
        p = os.path.join(src, fn)
        if fn.endswith(".ncu-rep"):
            base = fn[:-len(".ncu-rep")]
            shutil.copy(p, dst)
            res = full_summary(p, os.path.join(dst, base + "_ncu_full.txt"))
            if base == "pagerank_k_pr_rows" and res:
                m = res[0][1]
                rd = float(m["dram__bytes_read.sum"][0])
                wr = float(m["dram__bytes_write.sum"][0])
                unit = m["dram__bytes_read.sum"][1]
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
                wunit = m["dram__bytes_write.sum"][1]
                wscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[wunit]
                dur, du = m["gpu__time_duration.sum"]
                dscale = {"usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3, "ns": 1e-3}[du]
                json.dump({
                    "kernel": res[0][0][:60],
                    "graph": "R-MAT scale 22 directed (seed 1), relabeled AT",
                    "dram_read_bytes": rd * scale,
                    "dram_write_bytes": wr * wscale,
                    "dram_bytes_per_launch": rd * scale + wr * wscale,
                    "duration_us_cold": float(dur) * dscale,
                    "source": f"profiles/{r}/pagerank_k_pr_rows.ncu-rep "
                              "(ncu --set full --clock-control none)",
                }, open(os.path.join(ROOT, "profiles", "pagerank_ncu.json"), "w"), indent=1)
        elif fn.endswith("_levels.txt"):
            shutil.copy(p, dst)
    print("wrote", dst)


if __name__ == "__main__":
    main()
