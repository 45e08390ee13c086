"""STAGED transport's pack / unpack kernels on a ROW <-> COL
repartition: one process drives 2 GPUs (hda_init(2, P=2); STAGED is single-process),
16384^2 fp32, SCALE under ROW then COL.  Each redistribution packs a 256 MiB strided block
(8192 runs of 32 KiB, pitch 64 KiB) into contiguous staging on the writer, copies it over
NVLink on the copy engine, and unpacks it on the reader.  Run under ncu with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:copy_runs
to get the pack/unpack HBM bandwidth; prints the CUDA-event step time itself.
    python tools/staged_pack.py [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1809_05657_b200 as H  # noqa: E402
import synth  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
n = 16384
h = H.HDArray(n_gpus=2, n_devices=2)
h.set_transport(1)  # STAGED
X = h.create(H.F32, (n, n), synth.uniform(3, (n, n), "f32"))
rp, cp = h.partition(H.ROW, (n, n)), h.partition(H.COL, (n, n))
for i in range(4):
    h.apply(H.K_SCALE, rp if i % 2 == 0 else cp, [(X, [(0, 0)], [(0, 0)])], [1.0])
h.sync()
s0 = torch.cuda.ExternalStream(h.stream(0), device=torch.device("cuda", 0))
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.device(0):
    a.record(s0)
for i in range(steps):
    h.apply(H.K_SCALE, rp if i % 2 == 0 else cp, [(X, [(0, 0)], [(0, 0)])], [1.0])
with torch.cuda.device(0):
    b.record(s0)
h.sync()
ms = a.elapsed_time(b) / steps
moved = (n // 2) * (n // 2) * 4  # one 8192^2 fp32 block each way per redistribution
print(f"STAGED repartition 16384^2 f32 on 2 GPUs: {ms:.3f} ms per call, {moved / ms / 1e6:.0f} GB/s per GPU "
      f"(pack + copy-engine transfer + unpack + SCALE)")
h.close()
