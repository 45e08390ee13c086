"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, element by
element on the same seeded inputs.

Bars (BASELINE.json north_star): message sets, owner maps and exchanged data
bit-exact; stencils within 1e-12 normwise (they are in fact compared bit-exactly:
both sides use the same operand order and IEEE operations); the product within
1e-2 relative Frobenius (integer cases bit-exact).  Every replica of every device is
compared, so out-of-region writes and stale halos are caught.
"""
import os

import numpy as np
import pytest

import oracle as O
import synth
from programs import LibAdapter, gen_program, run_program

pytestmark = pytest.mark.gpu

J = [(0, -1), (0, 1), (-1, 0), (1, 0)]
N9 = [(i, j) for i in (-1, 0, 1) for j in (-1, 0, 1) if i or j]
N7 = [(0, 0, -1), (0, 0, 1), (0, -1, 0), (0, 1, 0), (-1, 0, 0), (1, 0, 0)]


@pytest.fixture(scope="module")
def H():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_1809_05657_b200 as H
    H.lib()
    return H


def ngpus():
    import torch
    return torch.cuda.device_count()


def assert_same_msgs(h, w):
    a = O.msgs_by_pair(LibAdapter(h).msgs())
    b = O.msgs_by_pair(w.msgs())
    assert a.keys() == b.keys()
    for k in b:
        np.testing.assert_array_equal(a[k], b[k])


def assert_replicas(h, w, arrs, P):
    for a in arrs:
        np.testing.assert_array_equal(h.owner_map(a), w.owner_map(a))
        for d in range(P):
            g = h.read_replica(a, d)
            o = w.replica(a, d)
            assert g.tobytes() == o.tobytes(), f"array {a} device {d}: replica differs"


# ------------------------------------------------------------------ config 1
@pytest.mark.parametrize("transport", [0, 1, 2])
def test_config1_virtual_devices(H, transport):
    """BASELINE configs[0]: 16x16 fp64 Jacobi, 4 row partitions, +-1 offsets; paper
    2-call form on one GPU with 4 virtual devices."""
    n, P = 16, 4
    h = H.HDArray(n_gpus=1, n_devices=P)
    h.set_transport(transport)
    w = O.Oracle(P)
    init_a = synth.uniform(synth.SEED0 + 0, (n, n))
    init_b = synth.uniform(synth.SEED0 + 100, (n, n))
    for be in (h, w):
        A = be.create(H.F64, (n, n))
        B = be.create(H.F64, (n, n))
        data = be.partition(H.ROW, (n, n))
        work = be.partition(H.ROW, (n, n), (1, 1), (n - 1, n - 1))
        be.write(A, data, init_a)
        be.write(B, data, init_b)
    assert_replicas(h, w, [A, B], P)
    for s in range(3):
        for be in (h, w):
            be.apply(H.K_JACOBI5, work, [(A, [], [(0, 0)]), (B, J, [])])
        assert_same_msgs(h, w)
        assert_replicas(h, w, [A, B], P)
        for be in (h, w):
            be.apply(H.K_COPY, work, [(B, [], [(0, 0)]), (A, [(0, 0)], [])])
        assert_same_msgs(h, w)
        assert_replicas(h, w, [A, B], P)
    got = h.read(B, data)
    ref = w.read(B, data)
    assert_same_msgs(h, w)
    assert got.tobytes() == ref.tobytes()
    assert h.stats()["plan_hits"] > 0
    h.close()


# ------------------------------------------------------------------ random programs
@pytest.mark.parametrize("P,transport", [(2, 0), (3, 1), (4, 0), (8, 0), (8, 1)])
def test_random_programs_bit_exact(H, P, transport):
    """STAMP writes distinctive raw bits (NaN payloads included) on arbitrary def
    shapes; reads/writes/partition switches move them; every replica must match."""
    for seed in range(12):
        for ndim in (2, 3):
            prog = gen_program(50_000 + 100 * P + seed, P, ndim=ndim, n_ops=8, with_kernels=True)
            w = O.Oracle(P)
            h = H.HDArray(n_gpus=1, n_devices=P)
            h.set_transport(transport)
            lib = LibAdapter(h)
            states = {}

            def on_o(step, op, arrs, st):
                states[step] = (st, O.msgs_by_pair(w.msgs()) if st == 0 else None,
                                [[w.replica(a, d).tobytes() for d in range(P)] for a in arrs])

            def on_l(step, op, arrs, st):
                st_o, m_o, reps = states[step]
                assert st == st_o
                if st == 0:
                    m_l = O.msgs_by_pair(lib.msgs())
                    assert m_l.keys() == m_o.keys()
                for ai, a in enumerate(arrs):
                    for d in range(P):
                        assert h.read_replica(a, d).tobytes() == reps[ai][d], (seed, step, op, a, d)

            run_program(prog, w, on_o)
            run_program(prog, lib, on_l)
            h.close()


# ------------------------------------------------------------------ stencils
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("shape,kind,P", [((150, 700), "ROW", 3), ((130, 1030), "BLOCK", 4),
                                          ((37, 53), "COL", 2), ((300, 260), "BLOCK", 8)])
def test_stencil2d_bit_exact(H, dtype, shape, kind, P):
    DT = H.F64 if dtype == "f64" else H.F32
    npdt = np.float64 if dtype == "f64" else np.float32
    u0 = synth.uniform(synth.SEED0 + 1, shape, dtype)
    for K, uses in ((H.K_JACOBI5, J), (H.K_STENCIL9, N9)):
        h = H.HDArray(n_gpus=1, n_devices=P)
        w = O.Oracle(P)
        for be in (h, w):
            X = be.create(DT, shape, u0)
            Y = be.create(DT, shape, u0)
            part = be.partition(getattr(H, kind), shape, (1, 1), (shape[0] - 1, shape[1] - 1))
            for s in range(4):
                src, dst = (X, Y) if s % 2 == 0 else (Y, X)
                be.apply(K, part, [(dst, [], [(0, 0)]), (src, uses, [])])
        assert_replicas(h, w, [X, Y], P)
        assert h.read_replica(X, 0).dtype == npdt
        h.close()


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_stencil7_3d_bit_exact(H, dtype):
    DT = H.F64 if dtype == "f64" else H.F32
    shape, P = (40, 36, 70), 3
    u0 = synth.uniform(synth.SEED0 + 4, shape, dtype)
    h = H.HDArray(n_gpus=1, n_devices=P)
    w = O.Oracle(P)
    for be in (h, w):
        X = be.create(DT, shape, u0)
        Y = be.create(DT, shape, u0)
        part = be.partition(H.ROW, shape, (1, 1, 1), tuple(s - 1 for s in shape))
        for s in range(3):
            src, dst = (X, Y) if s % 2 == 0 else (Y, X)
            be.apply(H.K_STENCIL7_3D, part, [(dst, [], [(0, 0, 0)]), (src, N7, [])])
    assert_replicas(h, w, [X, Y], P)
    h.close()


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_stencil_division_edge_values(H, dtype):
    """Stencils on fields with +Inf, signed zeros, subnormals, tiny and huge normals
    mixed into uniform data (the divisions by 20 and 6 on their slow paths, Inf
    propagation, sign of zero): every replica bit-identical to the oracle, on the
    default kernels (the TMA-ring ones: test_stencil2d_tma_shapes).  2-D boxes with
    full 16-row tiles (ROW) and thin strips (COL, 4 devices)."""
    DT = H.F64 if dtype == "f64" else H.F32
    cases = [((90, 420), "ROW", 2, H.K_STENCIL9, N9), ((37, 53), "COL", 4, H.K_STENCIL9, N9),
             ((20, 26, 140), "ROW", 2, H.K_STENCIL7_3D, N7)]
    for i, (shape, kind, P, K, uses) in enumerate(cases):
        u0 = synth.special_values(synth.SEED0 + 40 + i, shape, dtype)
        h = H.HDArray(n_gpus=1, n_devices=P)
        w = O.Oracle(P)
        for be in (h, w):
            X = be.create(DT, shape, u0)
            Y = be.create(DT, shape, u0)
            part = be.partition(getattr(H, kind), shape, (1,) * len(shape), tuple(s - 1 for s in shape))
            for s in range(3):
                src, dst = (X, Y) if s % 2 == 0 else (Y, X)
                be.apply(K, part, [(dst, [], [(0,) * len(shape)]), (src, uses, [])])
        assert_replicas(h, w, [X, Y], P)
        h.close()


def test_div20_matches_ieee(tmp_path):
    """The 9-point stencil's fp64 division (csrc/divc.cuh: Markstein correction with a
    constant reciprocal on [2^-1000, 2^1000], the IEEE division elsewhere) is bit-
    identical to a / 20.0 on 2^32 inputs covering every exponent, both range edges,
    zeros, subnormals, Inf and NaN; the 3-D stencil's fp32 division by 6 (same scheme)
    identical to a / 6.0f on all 2^32 fp32 inputs (tools/div20_check.cu, built here
    with nvcc)."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "div20_check")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-I",
                    os.path.join(root, "paper_1809_05657_b200", "csrc"), os.path.join(root, "tools", "div20_check.cu"),
                    "-o", exe], check=True, timeout=300)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count(" 0 mismatches") == 2, r.stdout


# ------------------------------------------------------------------ repartition
@pytest.mark.parametrize("dtype", ["f32", "bf16", "f64"])
@pytest.mark.parametrize("transport", [0, 1])
def test_repartition_row_col(H, dtype, transport):
    """configs[3] at test scale: ROW SCALE then COL SCALE on X; each switch is a full
    P(P-1)-block redistribution."""
    DT = {"f32": H.F32, "bf16": H.BF16, "f64": H.F64}[dtype]
    shape, P = (96, 160), 4
    v = synth.uniform(9, shape, dtype)
    h = H.HDArray(n_gpus=1, n_devices=P)
    h.set_transport(transport)
    w = O.Oracle(P)
    for be in (h, w):
        X = be.create(DT, shape)
        rowp = be.partition(H.ROW, shape)
        colp = be.partition(H.COL, shape)
        be.write(X, rowp, v)
    for it in range(3):
        for part in (colp, rowp):
            for be in (h, w):
                be.apply(H.K_SCALE, part, [(X, [(0, 0)], [(0, 0)])], [1.5 if it % 2 else 0.5])
            assert_same_msgs(h, w)
            n_blocks = len(O.msgs_by_pair(w.msgs()))
            assert n_blocks == P * (P - 1)
            assert_replicas(h, w, [X], P)
    h.close()


def test_raw_bits_repartition(H):
    """random bit patterns (NaN payloads, denormals, infinities) survive the exchange
    bit-exactly: write under ROW, read under COL (pure copies)."""
    shape, P = (64, 96), 4
    for dt, name in ((H.F64, "f64"), (H.F32, "f32"), (H.BF16, "bf16")):
        bits = synth.random_bits(77, shape, name)
        for transport in (0, 1):
            h = H.HDArray(n_gpus=1, n_devices=P)
            h.set_transport(transport)
            X = h.create(dt, shape)
            h.write(X, h.partition(H.ROW, shape), bits)
            got = h.read(X, h.partition(H.COL, shape))
            assert got.tobytes() == np.ascontiguousarray(bits).tobytes()
            assert h.stats()["last_msgs"] == P * (P - 1)
            h.close()


# ------------------------------------------------------------------ GEMM
@pytest.mark.parametrize("cdt", ["f32", "bf16"])
def test_gemm_integer_exact_and_allgather(H, cdt):
    """Listing 2 with integer bf16 inputs: fp32 accumulation is exact
    (|sum| < 2^24), so C is bit-exact vs int64 matmul; call 1 all-gathers B."""
    M, N, K, P = 256, 384, 512, 2
    Ab = synth.int_bf16(21, (M, K))
    Bb = synth.int_bf16(22, (K, N))
    exact = synth.bf16_to_f32(Ab).astype(np.int64) @ synth.bf16_to_f32(Bb).astype(np.int64)
    CT = H.F32 if cdt == "f32" else H.BF16
    h = H.HDArray(n_gpus=1, n_devices=P)
    w = O.Oracle(P)
    S = H.STAR
    for be in (h, w):
        A = be.create(H.BF16, (M, K))
        B = be.create(H.BF16, (K, N))
        C = be.create(CT, (M, N))
        pa, pb, pc = be.partition(H.ROW, (M, K)), be.partition(H.ROW, (K, N)), be.partition(H.ROW, (M, N))
        be.write(A, pa, Ab)
        be.write(B, pb, Bb)
        be.apply(H.K_GEMM, pc, [(C, [], [(0, 0)]), (A, [(0, S)], []), (B, [(S, 0)], [])], [1.0, 0.0])
    assert_same_msgs(h, w)
    assert len(O.msgs_by_pair(w.msgs())) == P * (P - 1)
    got = h.read(C, pc)
    ref = w.read(C, pc)
    assert got.tobytes() == ref.tobytes()
    if cdt == "f32":
        np.testing.assert_array_equal(got.astype(np.int64), exact)
    for be in (h, w):
        be.apply(H.K_GEMM, pc, [(C, [], [(0, 0)]), (A, [(0, S)], []), (B, [(S, 0)], [])], [1.0, 0.0])
    assert h.stats()["last_msgs"] == 0 and len(w.msgs()) == 0
    h.close()


def test_gemm_random_frobenius(H):
    M, N, K, P = 320, 256, 448, 4
    Ab = synth.uniform(31, (M, K), "bf16")
    Bb = synth.uniform(32, (K, N), "bf16")
    h = H.HDArray(n_gpus=1, n_devices=P)
    w = O.Oracle(P)
    S = H.STAR
    Cin = synth.uniform(33, (M, N), "f32")
    for be in (h, w):
        A = be.create(H.BF16, (M, K), Ab)
        B = be.create(H.BF16, (K, N), Bb)
        C = be.create(H.F32, (M, N), Cin)
        pc = be.partition(H.BLOCK, (M, N))
        be.apply(H.K_GEMM, pc, [(C, [(0, 0)], [(0, 0)]), (A, [(0, S)], []), (B, [(S, 0)], [])], [1.25, -0.5])
    got = h.read(C, pc).astype(np.float64)
    ref = w.read(C, pc).astype(np.float64)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-2
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-5  # fp32 accumulation
    h.close()


# ------------------------------------------------------------------ full scale
def test_config2_full_scale_eigenmode(H):
    """configs[1] at full size on one GPU: 8192^2 fp64 Jacobi, ROW, ping-pong, 100
    sweeps, in the bench launch configuration.  Closed form u = lambda^s u0
    within 1e-12 normwise, plus sampled cells against the oracle on windows."""
    n, sweeps, a, b = 8192, 100, 37, 61
    u0 = synth.eigenmode2d(n, n, a, b)
    lam = (np.cos(a * np.pi / (n - 1)) + np.cos(b * np.pi / (n - 1))) / 2
    h = H.HDArray(n_gpus=1, n_devices=1)
    X = h.create(H.F64, (n, n), u0)
    Y = h.create(H.F64, (n, n), u0)
    part = h.partition(H.ROW, (n, n), (1, 1), (n - 1, n - 1))
    for s in range(sweeps):
        src, dst = (X, Y) if s % 2 == 0 else (Y, X)
        h.apply(H.K_JACOBI5, part, [(dst, [], [(0, 0)]), (src, J, [])])
    got = h.read(X, h.partition(H.ROW, (n, n)))
    ref = lam ** sweeps * u0
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < 1e-12
    # sampled cells: the oracle on a (2s+3)^2 window around each sample, from the
    # random initial field (a window of radius s+1 makes the centre exact)
    s = 6
    v0 = synth.uniform(synth.SEED0 + 1, (n, n))
    h2 = H.HDArray(n_gpus=1, n_devices=1)
    X = h2.create(H.F64, (n, n), v0)
    Y = h2.create(H.F64, (n, n), v0)
    part2 = h2.partition(H.ROW, (n, n), (1, 1), (n - 1, n - 1))
    for k in range(s):
        src, dst = (X, Y) if k % 2 == 0 else (Y, X)
        h2.apply(H.K_JACOBI5, part2, [(dst, [], [(0, 0)]), (src, J, [])])
    full = h2.read(X, h2.partition(H.ROW, (n, n)))
    rng = np.random.default_rng(5)
    pts = [(1, 1), (n - 2, n - 2), (1, n - 2), (4000, 17)] + [tuple(rng.integers(1, n - 1, 2)) for _ in range(6)]
    r = s + 1
    for (i, j) in pts:
        i0, i1 = max(i - r, 0), min(i + r + 1, n)
        j0, j1 = max(j - r, 0), min(j + r + 1, n)
        win = np.ascontiguousarray(v0[i0:i1, j0:j1])
        w = O.Oracle(1)
        WX = w.create(O.F64, win.shape, win)
        WY = w.create(O.F64, win.shape, win)
        # interior of the window; array borders keep their ghost role
        lb = (1 if i0 == 0 else 1, 1 if j0 == 0 else 1)
        wp = w.partition(O.ROW, win.shape, lb, (win.shape[0] - 1, win.shape[1] - 1))
        for k in range(s):
            src, dst = (WX, WY) if k % 2 == 0 else (WY, WX)
            w.apply(O.K_JACOBI5, wp, [(dst, [], [(0, 0)]), (src, J, [])])
        ow = w.replica(WX, 0)
        assert ow[i - i0, j - j0] == full[i, j], (i, j)
    h.close()
    h2.close()


# ------------------------------------------------------------------ multi-GPU
@pytest.mark.parametrize("G,P", [(2, 2), (2, 4), (4, 8)])
def test_multi_gpu_single_process(H, G, P):
    """P devices over G physical GPUs (NVLink peer pulls + cross-GPU sync words; at P=8
    the BLOCK grid is 4x2 and same-GPU and cross-GPU neighbours mix)."""
    if ngpus() < G:
        pytest.skip(f"needs {G} GPUs")
    shape = (258, 514)
    u0 = synth.uniform(3, shape)
    for transport in (0, 1, 2):
        h = H.HDArray(n_gpus=G, n_devices=P)
        h.set_transport(transport)
        w = O.Oracle(P)
        for be in (h, w):
            X = be.create(H.F64, shape, u0)
            Y = be.create(H.F64, shape, u0)
            part = be.partition(H.ROW, shape, (1, 1), (shape[0] - 1, shape[1] - 1))
            colp = be.partition(H.COL, shape)
            for s in range(6):
                src, dst = (X, Y) if s % 2 == 0 else (Y, X)
                be.apply(H.K_JACOBI5, part, [(dst, [], [(0, 0)]), (src, J, [])])
            for s in range(4):
                src, dst = (X, Y) if s % 2 == 0 else (Y, X)
                be.apply(H.K_STENCIL9, part, [(dst, [], [(0, 0)]), (src, N9, [])])
            blk = be.partition(H.BLOCK, shape, (1, 1), (shape[0] - 1, shape[1] - 1))
            for s in range(2):
                src, dst = (X, Y) if s % 2 == 0 else (Y, X)
                be.apply(H.K_STENCIL9, blk, [(dst, [], [(0, 0)]), (src, N9, [])])
            be.apply(H.K_SCALE, colp, [(X, [(0, 0)], [(0, 0)])], [2.0])
        assert_replicas(h, w, [X, Y], P)
        h.close()
    # bulk repartition: blocks >= 1 MiB take the copy-engine path under AUTO
    big = (1024, 2048)
    v = synth.uniform(8, big, "f32")
    for transport in (0, 2):
        h = H.HDArray(n_gpus=G, n_devices=P)
        h.set_transport(transport)
        w = O.Oracle(P)
        for be in (h, w):
            Z = be.create(H.F32, big)
            rp = be.partition(H.ROW, big)
            cp = be.partition(H.COL, big)
            be.write(Z, rp, v)
            for it in range(3):
                be.apply(H.K_SCALE, cp, [(Z, [(0, 0)], [(0, 0)])], [2.0])
                be.apply(H.K_SCALE, rp, [(Z, [(0, 0)], [(0, 0)])], [0.5])
        assert_replicas(h, w, [Z], P)
        h.close()


@pytest.mark.skipif("ngpus() < 2")
@pytest.mark.parametrize("mode", [0, 1])
def test_multi_gpu_halo_modes(mode):
    """Both 2-D halo launch shapes give the oracle's replicas for both stencils:
    HDA_HALO_MODE=1 (pull blocks + interior + gated boundary strips in one launch) and
    0 (comm-stream pull, interior launch, boundary launch); the default mixes them per
    kernel.  The mode is read once per process, hence the subprocess."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, HDA_HALO_MODE=str(mode))
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        f"{__file__}::test_multi_gpu_single_process"], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


# ------------------------------------------------------------------ 2MM
@pytest.mark.parametrize("kind", ["ROW", "COL"])
def test_2mm_chain_partition_choice(H, kind):
    """2MM: D = A x B ; E = C x D, iterated.  ROW moves B once and D every
    iteration; COL moves A and C once.  Integer bf16 inputs keep every product exact,
    so E (fp32) is bit-exact vs the oracle; messages equal element by element."""
    n, P, iters = 256, 4, 3
    S = H.STAR
    Ab, Bb, Cb = (synth.int_bf16(60 + i, (n, n), -2, 2) for i in range(3))
    h = H.HDArray(n_gpus=1, n_devices=P)
    w = O.Oracle(P)
    moved = []
    for be in (h, w):
        A = be.create(H.BF16, (n, n))
        B = be.create(H.BF16, (n, n))
        C = be.create(H.BF16, (n, n))
        D = be.create(H.BF16, (n, n))
        E = be.create(H.F32, (n, n))
        part = be.partition(getattr(H, kind), (n, n))
        for X, v in ((A, Ab), (B, Bb), (C, Cb)):
            be.write(X, part, v)
    for it in range(iters):
        for be in (h, w):
            be.apply(H.K_GEMM, part, [(D, [], [(0, 0)]), (A, [(0, S)], []), (B, [(S, 0)], [])], [1.0, 0.0])
        assert_same_msgs(h, w)
        m1 = {k[0] for k in O.msgs_by_pair(w.msgs())}
        for be in (h, w):
            be.apply(H.K_GEMM, part, [(E, [], [(0, 0)]), (C, [(0, S)], []), (D, [(S, 0)], [])], [1.0, 0.0])
        assert_same_msgs(h, w)
        m2 = {k[0] for k in O.msgs_by_pair(w.msgs())}
        moved.append((m1, m2))
    if kind == "ROW":
        assert moved[0] == ({B}, {D}) and all(m == (set(), {D}) for m in moved[1:])
    else:
        assert moved[0] == ({A}, {C}) and all(m == (set(), set()) for m in moved[1:])
    assert_replicas(h, w, [D, E], P)
    h.close()


# ------------------------------------------------------------------ Reduce (§8(f)-3)
@pytest.mark.parametrize("dtype", ["f64", "f32", "bf16", "i64"])
def test_reduce_vs_oracle(H, dtype):
    """Table 2 Reduce: same coherence messages as a read, then a
    device reduction + combine.  Integer-valued data: SUM/MAX/MIN exact; random data:
    SUM within 1e-12 of the sequential fp64 oracle relative to sum|x|."""
    DT = {"f64": H.F64, "f32": H.F32, "bf16": H.BF16, "i64": H.I64}[dtype]
    shape, P = (130, 270), 3
    rng = np.random.default_rng(3)
    ints = rng.integers(-50, 50, size=shape)
    vals = {"f64": ints.astype(np.float64), "f32": ints.astype(np.float32),
            "bf16": synth.int_bf16(5, shape, -50, 50), "i64": ints.astype(np.int64)}[dtype]
    h = H.HDArray(n_gpus=1, n_devices=P)
    w = O.Oracle(P)
    for be in (h, w):
        X = be.create(DT, shape)
        rowp = be.partition(H.ROW, shape)
        blk = be.partition(H.BLOCK, shape, (3, 5), (120, 250))
        be.write(X, rowp, vals)
    for part in (blk, rowp):
        for op in (H.SUM, H.MAX, H.MIN):
            g = h.reduce(X, part, op)
            o = w.reduce(X, part, op)
            assert g == o, (op, g, o)
            assert_same_msgs(h, w)
    if dtype == "f64":
        r = synth.uniform(7, shape)
        for be in (h, w):
            be.write(X, rowp, r)
        g, o = h.reduce(X, blk, H.SUM), w.reduce(X, blk, H.SUM)
        assert abs(g - o) <= 1e-12 * np.abs(r).sum()
        p2 = np.where(synth.uniform(8, shape) < 0.5, 0.5, 2.0)
        for be in (h, w):
            be.write(X, rowp, p2)
        assert h.reduce(X, rowp, H.PROD) == w.reduce(X, rowp, H.PROD)  # powers of two: exact
    h.close()


# ------------------------------------------------------------------ absolute sections (§8(f)-2)
def test_absolute_sections_triangular_gpu(H):
    """Correlation-style triangular access with a Listing-1 manual partition
    (P:L197-208): each device STAMPs the upper-triangle rows of its slab,
    then every device reads the whole upper triangle; replicas bit-exact vs oracle."""
    n, P = 96, 2
    h = H.HDArray(n_gpus=1, n_devices=P)
    w = O.Oracle(P)
    up = H.trapezoid([(0, 0), (0, n - 1), (n - 1, n - 1), (n - 1, n - 1)])
    cut = 28  # ~ n(1 - 1/sqrt 2): halves the triangle's work (Listing 1's 3008/10240)
    defs = [[b for b in up if b[0][0] < cut], [b for b in up if b[0][0] >= cut]]
    for be in (h, w):
        X = be.create(H.F64, (n, n))
        part = be.partition_manual((n, n), [[0, 0], [cut, 0]], [[cut, n], [n, n]])
    for be in (h, w):
        be.apply_abs(H.K_STAMP, part, [(X, [[], []], defs)], [9.0])
    for be in (h, w):
        be.apply_abs(H.K_NONE, part, [(X, [up, up], [[], []])])
    assert_same_msgs(h, w)
    assert len(w.msgs()) > 0
    assert_replicas(h, w, [X], P)
    h.close()


def test_trace_rows(H):
    """hda_set_trace / hda_trace: one exchange + one kernel span per call, ordered."""
    n, P = 64, 2
    h = H.HDArray(n_gpus=1, n_devices=P)
    X = h.create(H.F64, (n, n), synth.uniform(1, (n, n)))
    Y = h.create(H.F64, (n, n))
    part = h.partition(H.ROW, (n, n), (1, 1), (n - 1, n - 1))
    h.set_trace(True)
    for s in range(4):
        src, dst = (X, Y) if s % 2 == 0 else (Y, X)
        h.apply(H.K_JACOBI5, part, [(dst, [], [(0, 0)]), (src, J, [])])
    t = h.trace()
    h.set_trace(False)
    assert len(t) >= 8  # >= one kernel span per device per call
    assert (t[:, 4] >= t[:, 3]).all() and (t[:, 3] >= 0).all()
    assert set(t[:, 1].astype(int)) == {0, 1}
    h.close()


# ------------------------------------------------------------------ frontend (§8(f)-4)
def test_frontend_program_on_gpu(H):
    """config 1 driven through `#pragma hdarray` sources and file M on the GPU: every
    replica bit-exact with the oracle's explicit-offset run."""
    from paper_1809_05657_b200 import frontend as F
    src = r"""
#pragma hdarray use(B,(0,-1)) use(B,(0,1)) use(B,(-1,0)) use(B,(1,0)) def(A,(0,0))
__global__ void jacobi_step(double *A, const double *B) { }
#pragma hdarray use(A,(0,0)) def(B,(0,0))
__global__ void copy_back(double *B, const double *A) { }
"""
    n, P = 16, 4
    h = H.HDArray(n_gpus=1, n_devices=P)
    prog = F.Program(h, F.parse(src))
    prog.bind("jacobi_step", H.K_JACOBI5, arrays=["A", "B"])
    prog.bind("copy_back", H.K_COPY, arrays=["B", "A"])
    w = O.Oracle(P)
    ia, ib = synth.uniform(21, (n, n)), synth.uniform(22, (n, n))
    hs = {}
    for be in (h, w):
        A, B = be.create(H.F64, (n, n)), be.create(H.F64, (n, n))
        data = be.partition(H.ROW, (n, n))
        work = be.partition(H.ROW, (n, n), (1, 1), (n - 1, n - 1))
        be.write(A, data, ia)
        be.write(B, data, ib)
        hs[be] = (A, B, work)
    A, B, work = hs[h]
    Aw, Bw, workw = hs[w]
    for s in range(3):
        prog.apply_kernel("jacobi_step", work, A, B)
        prog.apply_kernel("copy_back", work, B, A)
        w.apply(O.K_JACOBI5, workw, [(Aw, [], [(0, 0)]), (Bw, J, [])])
        w.apply(O.K_COPY, workw, [(Bw, [], [(0, 0)]), (Aw, [(0, 0)], [])])
    assert_replicas(h, w, [A, B], P)
    h.close()


def test_gemm_single_cta_kernel():
    """The single-CTA tcgen05 GEMM (HDA_GEMM_2SM=0; the default is the CTA-pair kernel)
    passes the same GEMM parity tests; the switch is read once per process."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, HDA_GEMM_2SM="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-p", "no:cacheprovider", "-k",
                        "gemm and not single_cta or 2mm", __file__], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("cdt", ["f32", "bf16"])
@pytest.mark.parametrize("P", [1, 2])
def test_gemm_cta_pair_ragged(H, cdt, P):
    """The CTA-pair kernel's edges: work boxes whose rows and columns are not multiples of
    the 256x256 pair tile and do not start at 0, K not a multiple of 64-wide stages, and
    beta != 0 (C read).  Integer inputs keep every value exact, so C is bit-exact."""
    M, N, K = 1100, 776, 456
    Ab = synth.int_bf16(71, (M, K))
    Bb = synth.int_bf16(72, (K, N))
    Cin = (synth.int_bf16(73, (M, N)).astype(np.int64) % 7).astype(np.float32) - 3.0
    if cdt == "bf16":
        Cin = synth.bf16_to_f32(((Cin.view(np.uint32) >> 16).astype(np.uint16)))
    CT = H.F32 if cdt == "f32" else H.BF16
    h = H.HDArray(n_gpus=1, n_devices=P)
    w = O.Oracle(P)
    S = H.STAR
    lbs = [(37, 5), (600, 5)][:P] if P == 2 else [(37, 5)]
    ubs = [(600, 771), (1090, 771)][:P] if P == 2 else [(1090, 771)]
    for be in (h, w):
        A = be.create(H.BF16, (M, K), Ab)
        B = be.create(H.BF16, (K, N), Bb)
        cinit = Cin if cdt == "f32" else ((Cin.view(np.uint32) >> 16).astype(np.uint16))
        C = be.create(CT, (M, N), cinit)
        pc = be.partition_manual((M, N), lbs, ubs)
        be.apply(H.K_GEMM, pc, [(C, [(0, 0)], [(0, 0)]), (A, [(0, S)], []), (B, [(S, 0)], [])], [1.0, 2.0])
    assert_replicas(h, w, [C], P)
    h.close()


# ------------------------------------------------------------------ WAR races
def _scenario(name, G, **env):
    import os
    import subprocess
    import sys
    e = dict(os.environ, HDA_TIMEOUT_MS="20000", **env)
    script = os.path.join(os.path.dirname(os.path.abspath(__file__)), "gpu_scenarios.py")
    return subprocess.run([sys.executable, script, name, str(G)], env=e, capture_output=True, text=True,
                          timeout=600)


@pytest.mark.parametrize("G", [2, 3])
def test_pull_war_three_devices(G):
    """Reader-side WAR with three devices and an asymmetric slow reader (device 1's
    pulls sleep 20 ms): a pull into q's replica waits for the ACK of every peer that
    earlier pulled those cells from q.  Negative control: with the WAR waits switched
    off (HDA_DEBUG_NO_WAR) the same program breaks parity, so the scenario has teeth."""
    if ngpus() < G:
        pytest.skip(f"needs {G} GPUs")
    slow = dict(HDA_DEBUG_PULL_DELAY_US="20000", HDA_DEBUG_PULL_DELAY_DEV="1")
    r = _scenario("pull_war", G, **slow)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    neg = _scenario("pull_war", G, HDA_DEBUG_NO_WAR="1", **slow)
    assert neg.returncode == 1 and "MISMATCH" in neg.stdout, neg.stdout[-3000:] + neg.stderr[-3000:]


@pytest.mark.parametrize("G", [1, 2])
def test_staged_plan_replay_after_regrow(G):
    """STAGED: cached small-message plans replayed after a larger plan regrew the
    staging buffers stay bit-exact (the staging pointers are bound at issue)."""
    if ngpus() < G:
        pytest.skip(f"needs {G} GPUs")
    r = _scenario("staged_regrow", G)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("gate", ["1", "2", "0"])
def test_gemm_gated_allgather(G, gate):
    """The all-gather of B / D fused into the product (2MM ROW on G GPUs, 256 KiB copy
    threshold so 1024^2 blocks take the copy engine): bit-exact vs the oracle, gated
    (HDA_GEMM_GATE=1, every incoming row block waited for per k-block inside the GEMM),
    split (2: fp32 C with whole k-blocks per source as two launches, resident rows
    beside the copies and the arrived rows after them; the rest as in 1) and joined
    (0)."""
    if ngpus() < G:
        pytest.skip(f"needs {G} GPUs")
    r = _scenario("gemm_gate", G, HDA_GEMM_GATE=gate, HDA_CE_BYTES="262144")
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("mode", ["0", "1", "2"])
def test_stencil2d_tma_shapes(mode):
    """The TMA-ring 2-D stencils (HDA_TMA=1: 9-point, 2: both, 0: register march only)
    on multi-strip, multi-row-block boxes with ragged and unaligned edges, bit-exact
    against the oracle for every replica."""
    r = _scenario("tma_shapes", 1, HDA_TMA=mode)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
