"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(one context per GPU, the workload's own partition): closed forms that hold at any size
 plus cells sampled against the oracle one by one (windowed oracle runs:
after s sweeps a cell depends only on the (2s+1)-neighbourhood of the initial field, so
an oracle run on a window of radius s+1 reproduces the centre bit for bit)."""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu

N9 = [(i, j) for i in (-1, 0, 1) for j in (-1, 0, 1) if i or j]
N7 = [(0, 0, -1), (0, 0, 1), (0, -1, 0), (0, 1, 0), (-1, 0, 0), (1, 0, 0)]


@pytest.fixture(scope="module")
def H():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_1809_05657_b200 as H
    H.lib()
    return H


def _window_oracle(v0, centre, s, kernel, uses, dtype):
    """oracle value at `centre` after s sweeps of `kernel`, from a window of v0."""
    r = s + 1
    sl = tuple(slice(max(c - r, 0), min(c + r + 1, n)) for c, n in zip(centre, v0.shape))
    win = np.ascontiguousarray(v0[sl])
    nd = win.ndim
    w = O.Oracle(1)
    A = w.create(dtype, win.shape, win)
    B = w.create(dtype, win.shape, win)
    part = w.partition(O.ROW, win.shape, (1,) * nd, tuple(x - 1 for x in win.shape))
    for k in range(s):
        src, dst = (A, B) if k % 2 == 0 else (B, A)
        w.apply(kernel, part, [(dst, [], [(0,) * nd]), (src, uses, [])])
    return w.replica(A, 0)[tuple(c - x.start for c, x in zip(centre, sl))]


def test_config3_stencil9_full_scale(H):
    """configs[2]: 16384^2 fp64 9-point stencil (R12) over the interior, 20 ping-pong
    sweeps: the eigenmode closed form within 1e-12 normwise; 8 cells from a random field
    against windowed oracle runs, bit for bit."""
    n, sweeps, a, b = 16384, 20, 3, 4
    c0, c1 = np.cos(a * np.pi / (n - 1)), np.cos(b * np.pi / (n - 1))
    lam = (8 * (c0 + c1) + 4 * c0 * c1) / 20
    h = H.HDArray(n_gpus=1, n_devices=1)
    u0 = synth.eigenmode2d(n, n, a, b)
    X = h.create(H.F64, (n, n), u0)
    Y = h.create(H.F64, (n, n), u0)
    work = h.partition(H.BLOCK, (n, n), (1, 1), (n - 1, n - 1))
    data = h.partition(H.ROW, (n, n))
    for k in range(sweeps):
        src, dst = (X, Y) if k % 2 == 0 else (Y, X)
        h.apply(H.K_STENCIL9, work, [(dst, [], [(0, 0)]), (src, N9, [])])
    got = h.read(X, data)
    ref = lam ** sweeps * u0
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < 1e-12
    del got, ref, u0
    s = 4
    v0 = synth.uniform(synth.SEED0 + 3, (n, n))
    h.write(X, data, v0)
    h.write(Y, data, v0)
    for k in range(s):
        src, dst = (X, Y) if k % 2 == 0 else (Y, X)
        h.apply(H.K_STENCIL9, work, [(dst, [], [(0, 0)]), (src, N9, [])])
    full = h.read(X, data)
    rng = np.random.default_rng(9)
    pts = [(1, 1), (n - 2, n - 2), (1, n - 2), (8191, 8192)] + [tuple(rng.integers(1, n - 1, 2)) for _ in range(4)]
    for p in pts:
        assert _window_oracle(v0, p, s, O.K_STENCIL9, N9, O.F64) == full[p], p
    h.close()


def test_config5a_stencil7_full_scale(H):
    """configs[4] 3-D half: 1024^3 fp32 7-point (R13), slab (ROW) partition of the
    interior, 10 sweeps: the 3-D eigenmode closed form (fp32: 1e-5 normwise) and 6 cells
    against windowed fp32 oracle runs, bit for bit."""
    n, sweeps, (a, b, c) = 1024, 10, (5, 7, 9)
    lam = sum(np.cos(m * np.pi / (n - 1)) for m in (a, b, c)) / 3
    sz, sy, sx = (np.sin(m * np.pi * np.arange(n) / (n - 1)) for m in (a, b, c))
    for v in (sz, sy, sx):
        v[0] = v[-1] = 0.0
    u0 = np.empty((n, n, n), np.float32)
    yx = np.outer(sy, sx)
    for z in range(n):
        u0[z] = (sz[z] * yx).astype(np.float32)
    h = H.HDArray(n_gpus=1, n_devices=1)
    X = h.create(H.F32, (n,) * 3, u0)
    Y = h.create(H.F32, (n,) * 3, u0)
    work = h.partition(H.ROW, (n,) * 3, (1, 1, 1), (n - 1,) * 3)
    data = h.partition(H.ROW, (n,) * 3)
    for k in range(sweeps):
        src, dst = (X, Y) if k % 2 == 0 else (Y, X)
        h.apply(H.K_STENCIL7_3D, work, [(dst, [], [(0, 0, 0)]), (src, N7, [])])
    got = h.read(X, data)
    zs = slice(0, n, 64)  # normwise check on every 64th plane (the closed form holds everywhere)
    ref = (lam ** sweeps) * u0[zs].astype(np.float64)
    assert np.max(np.abs(got[zs] - ref)) / np.max(np.abs(ref)) < 1e-5
    del got, ref
    s = 3
    v0 = np.random.default_rng(synth.SEED0 + 5).random((n, n, n), dtype=np.float32)  # 4 GiB, fast
    h.write(X, data, v0)
    h.write(Y, data, v0)
    for k in range(s):
        src, dst = (X, Y) if k % 2 == 0 else (Y, X)
        h.apply(H.K_STENCIL7_3D, work, [(dst, [], [(0, 0, 0)]), (src, N7, [])])
    full = h.read(X, data)
    rng = np.random.default_rng(13)
    pts = [(1, 1, 1), (n - 2, n - 2, n - 2), (511, 512, 1)] + [tuple(rng.integers(1, n - 1, 3)) for _ in range(3)]
    for p in pts:
        assert _window_oracle(v0, p, s, O.K_STENCIL7_3D, N7, O.F32).tobytes() == full[p].tobytes(), p
    h.close()


def test_config5b_gemm_full_scale(H):
    """configs[4] product half: 16384^2 bf16 inputs in [-4,4] (P7: every partial sum
    is an integer below 2^24, so fp32 accumulation is exact in any order), fp32 C:
    256 sampled entries equal the oracle's sampled product exactly."""
    n = 16384
    Ab = synth.int_bf16(51, (n, n))
    Bb = synth.int_bf16(52, (n, n))
    h = H.HDArray(n_gpus=1, n_devices=1)
    S = H.STAR
    A, B, C = h.create(H.BF16, (n, n)), h.create(H.BF16, (n, n)), h.create(H.F32, (n, n))
    part = h.partition(H.ROW, (n, n))
    h.write(A, part, Ab)
    h.write(B, part, Bb)
    h.apply(H.K_GEMM, part, [(C, [], [(0, 0)]), (A, [(0, S)], []), (B, [(S, 0)], [])], [1.0, 0.0])
    got = h.read(C, part)
    rng = np.random.default_rng(3)
    ii = np.concatenate([[0, n - 1, 127, 128], rng.integers(0, n, 252)])
    jj = np.concatenate([[0, n - 1, 255, 256], rng.integers(0, n, 252)])
    ref = O.gemm_sample(Ab, Bb, ii, jj)
    np.testing.assert_array_equal(got[ii, jj].astype(np.float64), ref)
    h.close()


def test_config4_repartition_full_scale(H):
    """configs[3]: 32768^2 fp32 ROW <-> COL at P = 8 (virtual devices on one B200, 32 GiB
    of replicas): each redistribution is exactly P(P-1) blocks of 4096^2 (P10), and the
    raw bits of sampled rows survive two redistributions (SCALE by 1.0; NaN payloads
    compared as NaN)."""
    n, P = 32768, 8
    h = H.HDArray(n_gpus=1, n_devices=P)
    X = h.create(H.F32, (n, n))
    rowp = h.partition(H.ROW, (n, n))
    colp = h.partition(H.COL, (n, n))
    seed = 4242
    h.apply(H.K_STAMP, rowp, [(X, [], [(0, 0)])], [float(seed)])
    for part in (colp, rowp):
        h.apply(H.K_SCALE, part, [(X, [(0, 0)], [(0, 0)])], [1.0])
        plan = h.last_plan()
        assert len(plan) == P * (P - 1)
        assert all(int(np.prod(np.subtract(ub, lb))) == (n // P) ** 2 for _, _, _, lb, ub in plan)
    got = h.read(X, rowp)
    for r in (0, 4095, 4096, 20000, n - 1):
        exp = synth.splitmix64_stream(seed, r * n, n)
        e32 = (exp & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.float32)
        g = got[r]
        ok = (g.view(np.uint32) == e32.view(np.uint32)) | (np.isnan(g) & np.isnan(e32))
        assert ok.all(), r
    h.close()
