"""Single-process multi-GPU Jacobi (one process drives G GPUs, hda_init(G, P=G)):
device-timed steps (max over GPUs) and host issue time per step.  Not the bench
contract's launch mode (that is one process per GPU); this checks whether the
single-process runtime is host-bound.   python tools/sp_bench.py G [steps] [n]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1809_05657_b200 as H  # noqa: E402
import synth  # noqa: E402

G = int(sys.argv[1])
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 500
n = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
J = [(0, -1), (0, 1), (-1, 0), (1, 0)]
h = H.HDArray(n_gpus=G, n_devices=G)
u0 = synth.eigenmode2d(n, n, 37, 61)
X, Y = h.create(H.F64, (n, n), u0), h.create(H.F64, (n, n), u0)
w = h.partition(H.ROW, (n, n), (1, 1), (n - 1, n - 1))
calls = [h.prepare(H.K_JACOBI5, w, [(d, [], [(0, 0)]), (s, J, [])]) for s, d in ((X, Y), (Y, X))]
for i in range(20):
    calls[i % 2]()
h.sync()
streams = []
for d in range(G):
    with torch.cuda.device(d):
        streams.append(torch.cuda.ExternalStream(h.stream(d), device=torch.device("cuda", d)))
ev = []
for d in range(G):
    with torch.cuda.device(d):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(streams[d])
        ev.append((a, b))
t0 = time.perf_counter()
for i in range(steps):
    calls[i % 2]()
host_us = (time.perf_counter() - t0) / steps * 1e6
for d in range(G):
    with torch.cuda.device(d):
        ev[d][1].record(streams[d])
h.sync()
ms = max(a.elapsed_time(b) for a, b in ev)
pts = (n - 2) ** 2
print(f"G={G} {pts * steps / (ms * 1e-3) / 1e9:.1f} GPoints/s  {ms / steps * 1e3:.1f} us/step  "
      f"host issue {host_us:.1f} us/step  launches={h.stats()['kernel_launches']}")
h.close()
