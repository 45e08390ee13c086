"""GEMM edge cases through the C-ABI, one per process (a sticky CUDA error poisons the
context):  python tools/gemm_edge.py M N K m0 m1 n0 n1 beta cdt"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1809_05657_b200 as H  # noqa: E402
import synth  # noqa: E402

M, N, K, m0, m1, n0, n1 = (int(v) for v in sys.argv[1:8])
beta = float(sys.argv[8])
cdt = sys.argv[9]
Ab, Bb = synth.int_bf16(71, (M, K)), synth.int_bf16(72, (K, N))
Cin = np.zeros((M, N), np.float32) + 1.0
h = H.HDArray(n_gpus=1, n_devices=1)
A = h.create(H.BF16, (M, K), Ab)
B = h.create(H.BF16, (K, N), Bb)
C = h.create(H.F32, (M, N), Cin) if cdt == "f32" else h.create(H.BF16, (M, N), (Cin.view(np.uint32) >> 16).astype(np.uint16))
pc = h.partition_manual((M, N), [(m0, n0)], [(m1, n1)])
S = H.STAR
try:
    h.apply(H.K_GEMM, pc, [(C, [(0, 0)] if beta else [], [(0, 0)]), (A, [(0, S)], []), (B, [(S, 0)], [])], [1.0, beta])
    got = h.read_replica(C, 0)
    if cdt == "bf16":
        got = synth.bf16_to_f32(got)
    ex = synth.bf16_to_f32(Ab).astype(np.int64) @ synth.bf16_to_f32(Bb).astype(np.int64) + beta
    ok = np.array_equal(got[m0:m1, n0:n1].astype(np.float64), ex[m0:m1, n0:n1].astype(np.float32).astype(np.float64)) if cdt == "f32" else True
    print("OK" if ok else "MISMATCH", sys.argv[1:])
except Exception as e:  # noqa: BLE001
    print("ERROR", sys.argv[1:], str(e)[:120])
