"""Summarise ncu outputs for profiles/: a `--set full` report (key counters per
kernel) or a `gpu__time_duration` launch-list CSV (per-kernel totals and shares).

    python tools/ncu_summary.py report.ncu-rep > profiles/rNN/<name>.txt
    python tools/ncu_summary.py launches.csv   > profiles/rNN/<name>_launches.txt
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__waves_per_multiprocessor", "launch__occupancy_limit_registers",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
    "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct", "l1tex__t_bytes.sum", "lts__t_bytes.sum",
]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        print("no data")
        return
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"== {name[:160]}")
        for k in KEYS:
            for i, h in enumerate(hdr):
                if h == k or (k.endswith("hmma_cycles_active.avg.pct_of_peak_sustained_active") and h.startswith(
                        "sm__pipe_tensor") and h.endswith("pct_of_peak_sustained_active") and k not in hdr):
                    print(f"  {h:70s} {r[i]:>16s} {units[i]}")
                    break
        rd = wr = None
        for i, h in enumerate(hdr):
            if h == "dram__bytes_read.sum":
                rd = (float(r[i].replace(",", "")), units[i])
            if h == "dram__bytes_write.sum":
                wr = (float(r[i].replace(",", "")), units[i])
        if rd and wr:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tot = rd[0] * scale.get(rd[1], 1) + wr[0] * scale.get(wr[1], 1)
            print(f"  {'traffic_bytes (dram read + write)':70s} {tot:16.0f} byte")


def launches(path):
    txt = open(path).read()
    lines = [l for l in txt.splitlines() if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        k = r[ki].split("(")[0][:90]
        tot[k] += v
        cnt[k] += 1
    s = sum(tot.values())
    print(f"{'kernel':92s} {'launches':>8s} {'total':>12s} {'avg':>10s} {'share':>7s}")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k:92s} {cnt[k]:8d} {tot[k]:12.0f} {tot[k] / cnt[k]:10.1f} {100 * tot[k] / s:6.1f}%")
    print(f"(durations in the unit ncu reports for gpu__time_duration.sum; cold-cache, serialised)")


if __name__ == "__main__":
    p = sys.argv[1]
    full(p) if p.endswith(".ncu-rep") else launches(p)
