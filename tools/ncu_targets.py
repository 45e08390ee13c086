"""Two launches each of the configs[2] 9-point (16384^2 f64), the configs[4] 3-D
7-point (1024^3 f32) and the configs[4] bf16 GEMM (16384^2) kernels through the C-ABI,
in ONE process, for a single `ncu --set full` capture:

    ncu --set full --clock-control none --import-source on \
        -k regex:"stencil2d_kernel|stencil7_kernel|gemm_kernel" -c 6 \
        -o gpurun_out/targets python tools/ncu_targets.py
Not part of the library."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_05657_b200 as H  # noqa: E402
import synth  # noqa: E402

N9 = [(i, j) for i in (-1, 0, 1) for j in (-1, 0, 1) if i or j]
N7 = [(0, 0, -1), (0, 0, 1), (0, -1, 0), (0, 1, 0), (-1, 0, 0), (1, 0, 0)]

h = H.HDArray(n_gpus=1, n_devices=1)
n = 16384
u = np.ones((n, n))
X, Y = h.create(H.F64, (n, n), u), h.create(H.F64, (n, n), u)
w = h.partition(H.BLOCK, (n, n), (1, 1), (n - 1, n - 1))
for s, d in ((X, Y), (Y, X)):
    h.apply(H.K_STENCIL9, w, [(d, [], [(0, 0)]), (s, N9, [])])
h.sync()
h.free(X)
h.free(Y)

m = 1024
v = np.ones((m, m, m), np.float32)
X, Y = h.create(H.F32, (m,) * 3, v), h.create(H.F32, (m,) * 3, v)
w = h.partition(H.ROW, (m,) * 3, (1, 1, 1), (m - 1,) * 3)
for s, d in ((X, Y), (Y, X)):
    h.apply(H.K_STENCIL7_3D, w, [(d, [], [(0, 0, 0)]), (s, N7, [])])
h.sync()
h.free(X)
h.free(Y)

S = H.STAR
A, B, C = h.create(H.BF16, (n, n)), h.create(H.BF16, (n, n)), h.create(H.F32, (n, n))
p = h.partition(H.ROW, (n, n))
h.write(A, p, synth.int_bf16(51, (n, n)))
h.write(B, p, synth.int_bf16(52, (n, n)))
for _ in range(2):
    h.apply(H.K_GEMM, p, [(C, [], [(0, 0)]), (A, [(0, S)], []), (B, [(S, 0)], [])], [1.0, 0.0])
h.sync()
h.close()
print("ok")
