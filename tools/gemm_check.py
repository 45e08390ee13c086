"""configs[4] product on one GPU through the C-ABI: C = A @ B (16384^2 bf16, fp32 C),
tcgen05 kernel time -> TFLOP/s, sampled entries vs the oracle (fp64)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1809_05657_b200 as H
import oracle as O
import synth

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
cdt = sys.argv[2] if len(sys.argv) > 2 else "f32"
S = H.STAR
t0 = time.time()
Ab = synth.uniform(41, (n, n), "bf16")
Bb = synth.uniform(42, (n, n), "bf16")
print("gen", time.time() - t0, flush=True)
h = H.HDArray(n_gpus=1, n_devices=1)
A = h.create(H.BF16, (n, n), Ab)
B = h.create(H.BF16, (n, n), Bb)
C = h.create(H.F32 if cdt == "f32" else H.BF16, (n, n))
part = h.partition(H.ROW, (n, n))
acc = [(C, [], [(0, 0)]), (A, [(0, S)], []), (B, [(S, 0)], [])]
for _ in range(3):
    h.apply(H.K_GEMM, part, acc, [1.0, 0.0])
h.sync()
h.set_kernel_timing(True)
for _ in range(10):
    h.apply(H.K_GEMM, part, acc, [1.0, 0.0])
ms, k = h.kernel_time(H.K_GEMM)
tflops = 2.0 * n ** 3 / (ms / k * 1e-3) / 1e12
Cg = h.read(C, part)
rng = np.random.default_rng(0)
ii = rng.integers(0, n, 256)
jj = rng.integers(0, n, 256)
ref = O.gemm_sample(Ab, Bb, ii, jj)
got = Cg[ii, jj].astype(np.float64) if cdt == "f32" else synth.bf16_to_f32(Cg[ii, jj]).astype(np.float64)
rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
print(json.dumps({"n": n, "c": cdt, "ms": ms / k, "tflops": tflops, "frob_rel_sampled": rel, "launches": k}))
