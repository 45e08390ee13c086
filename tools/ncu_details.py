"""Print selected 'details' metrics of ncu reports side by side.
    python tools/ncu_details.py a.ncu-rep [b.ncu-rep ...]"""
import csv
import io
import subprocess
import sys

WANT = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'Issue Slots Busy', 'Executed Ipc Active',
        'Eligible Warps Per Scheduler', 'Active Warps Per Scheduler', 'No Eligible', 'L2 Hit Rate',
        'Warp Cycles Per Issued Instruction', 'Executed Instructions', 'Registers Per Thread', 'Achieved Occupancy',
        'L1/TEX Cache Throughput', 'L2 Cache Throughput', 'Mem Busy', 'Max Bandwidth', 'Compute (SM) Throughput']

for path in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h = r[0]
    seen = set()
    for row in r[1:]:
        k = row[h.index('Kernel Name')][:50]
        name = row[h.index('Metric Name')]
        if name in WANT and (k, name) not in seen:
            seen.add((k, name))
            print(f"{path.split('/')[-1][:20]:20s} {k:50s} {name:36s} {row[h.index('Metric Value')]:>14s} "
                  f"{row[h.index('Metric Unit')]}")
