"""Summarise an ncu report: key metrics + top stall reasons (CSV raw page)."""
import csv
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__grid_size', 'launch__block_size', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'lts__t_sector_hit_rate.pct', 'l1tex__t_sector_hit_rate.pct',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'lts__t_bytes.sum', 'l1tex__t_bytes.sum', 'sm__cycles_elapsed.avg.per_second']


def summarize(path, kernel_filter=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        name = d.get("Kernel Name", "")
        if kernel_filter and kernel_filter not in name:
            continue
        m = {k: (d.get(k), units[hdr.index(k)] if k in hdr else "") for k in KEYS}
        stalls = []
        for h, v in zip(hdr, vals):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith(
                    "_per_issue_active.ratio"):
                try:
                    stalls.append((float(v), h[len("smsp__average_warps_issue_stalled_"):-len(
                        "_per_issue_active.ratio")]))
                except ValueError:
                    pass
        res.append((name, m, sorted(stalls, reverse=True)[:8]))
    return res


if __name__ == "__main__":
    for name, m, stalls in summarize(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None):
        print("==", name[:100])
        for k, (v, u) in m.items():
            print(f"  {k:60s} {v} {u}")
        print("  stalls:", ", ".join(f"{n}={v:.2f}" for v, n in stalls))
