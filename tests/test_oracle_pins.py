"""Pins of the CPU oracle against what the paper and the mathematics fix.

Nothing here compares the oracle with itself or with the CUDA path.  Each test names
the passage (PAPER.md "P:Lnnn") or the closed form it checks.  A plausible mistake in
the oracle (a dropped offset, a wrong sign or index, a transposed operand, a stale
replica, a missing commit) fails at least one of them.
"""
import itertools
import os

import numpy as np
import pytest

import synth

HERE = os.path.dirname(os.path.abspath(__file__))
S = None  # oracle.STAR, filled by fixture


@pytest.fixture(autouse=True)
def _star(oracle_mod):
    global S
    S = oracle_mod.STAR


JAC_USES = [(0, -1), (0, 1), (-1, 0), (1, 0)]
ZERO2 = [(0, 0)]


def load_golden(path):
    steps = {}
    with open(path) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            step, arr, src, dst, row, c0, c1 = line.split()
            steps.setdefault(step, {}).setdefault((arr, int(src), int(dst)), set()).update(
                (int(row), c) for c in range(int(c0), int(c1)))
    return steps


def msgs_as_cells(m, names, ncols):
    out = {}
    for arr, src, dst, c in m:
        out.setdefault((names[int(arr)], int(src), int(dst)), set()).add((int(c) // ncols, int(c) % ncols))
    return out


# ---------------------------------------------------------------------------
# P3: the config-1 worked example (tests/golden/config1_messages.txt)
# ---------------------------------------------------------------------------
def test_config1_worked_example(oracle_mod):
    O = oracle_mod
    gold = load_golden(os.path.join(HERE, "golden", "config1_messages.txt"))
    n = 16
    w = O.Oracle(4)
    A = w.create(O.F64, (n, n))
    B = w.create(O.F64, (n, n))
    names = {A: "A", B: "B"}
    data = w.partition(O.ROW, (n, n))
    work = w.partition(O.ROW, (n, n), (1, 1), (n - 1, n - 1))
    assert [w.region(work, d, 2) for d in range(4)] == [
        ((1, 1), (5, 15)), ((5, 1), (9, 15)), ((9, 1), (12, 15)), ((12, 1), (15, 15))]
    w.write(A, data, synth.uniform(synth.SEED0 + 0, (n, n)))
    w.write(B, data, synth.uniform(synth.SEED0 + 100, (n, n)))
    assert len(w.msgs()) == 0
    total = 0
    for s in (1, 2):
        w.apply(O.K_JACOBI5, work, [(A, [], ZERO2), (B, JAC_USES, [])])
        got = msgs_as_cells(w.msgs(), names, n)
        assert got == gold.get(f"s{s}_jacobi", {}), f"sweep {s} jacobi"
        if s == 1:
            total = sum(len(v) for v in got.values())
        w.apply(O.K_COPY, work, [(B, [], ZERO2), (A, ZERO2, [])])
        assert msgs_as_cells(w.msgs(), names, n) == gold.get(f"s{s}_copy", {}), f"sweep {s} copy"
    assert total == 88  # 88 cells = 704 B in sweep 1
    w.read(B, data)
    assert msgs_as_cells(w.msgs(), names, n) == gold["read_B"]


# ---------------------------------------------------------------------------
# composition: per-work-item brute force written here (offsets are
# relative to each work item; '*' = all elements of that dimension)
# ---------------------------------------------------------------------------
def brute_luse(shape, lb, ub, tuples):
    cells = set()
    if any(l >= u for l, u in zip(lb, ub)):
        return cells
    for w_ in itertools.product(*[range(l, u) for l, u in zip(lb, ub)]):
        for d in tuples:
            axes = [range(s) if dk == S else [wk + dk] for wk, dk, s in zip(w_, d, shape)]
            for c in itertools.product(*axes):
                if all(0 <= ck < s for ck, s in zip(c, shape)):
                    cells.add(c)
    return cells


def random_program(rng, O, P, shape, n_calls):
    """SPEC-style random program: offsets in [-2,2] and '*', partition switches."""
    w = O.Oracle(P, with_data=True)
    nd = len(shape)
    arrs = [w.create(O.F64, shape) for _ in range(2)]
    parts = [w.partition(k, shape) for k in (O.ROW, O.COL, O.BLOCK)]
    parts.append(w.partition(O.ROW, shape, [1] * nd, [s - 1 for s in shape]))
    log = []
    for k in range(n_calls):
        part = parts[rng.integers(len(parts))]
        x = arrs[rng.integers(2)]
        y = arrs[1 - arrs.index(x)]
        nu = int(rng.integers(1, 4))
        uses = []
        for _ in range(nu):
            t = tuple(int(v) if rng.random() > 0.15 else S for v in rng.integers(-2, 3, size=nd))
            uses.append(t)
        acc = [(x, uses, [])]
        if rng.random() < 0.8:
            acc.append((y, [], [(0,) * nd]))
        if rng.random() < 0.3:
            w.write(x, part, np.full(shape, float(k)))
            log.append(("write", x, part, None))
        w.apply(O.K_NONE, part, acc)
        log.append(("apply", acc, part, w.msgs()))
    return w, log


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_messages_only_flow_from_other_writers_to_users(oracle_mod, P):
    """P4: communication only for cells defined on one device and used on another;
    every message cell lies in the reader's LUSE (brute-force composition here);
    P=1 never communicates; a repeated use-only call has an empty plan."""
    O = oracle_mod
    rng = np.random.default_rng(1000 + P)
    shape = (9, 7)
    w = O.Oracle(P)
    X = w.create(O.F64, shape)
    Y = w.create(O.F64, shape)
    parts = [w.partition(k, shape) for k in (O.ROW, O.COL, O.BLOCK)]
    owner_before = w.owner_map(X)
    valid_before = w.valid_map(X)
    for k in range(40):
        part = parts[rng.integers(3)]
        uses = [tuple(int(v) if rng.random() > 0.15 else S for v in rng.integers(-2, 3, size=2))
                for _ in range(int(rng.integers(1, 4)))]
        defs = [(0, 0)] if rng.random() < 0.7 else []
        w.apply(O.K_NONE, part, [(X, uses, []), (Y, [], [(0, 0)])])
        m = w.msgs()
        if P == 1:
            assert len(m) == 0
        for arr, src, dst, c in m:
            assert arr == X and src != dst
            cell = np.unravel_index(int(c), shape)
            assert owner_before[cell] == src                    # last writer sends
            assert not (int(valid_before[cell]) >> int(dst)) & 1  # reader lacked it
            lb, ub = w.region(part, int(dst), 2)
            assert tuple(int(v) for v in cell) in brute_luse(shape, lb, ub, uses)
        # completeness: every used cell that the reader lacks and another device wrote is sent
        sent = {(int(d), int(c)) for _, _, d, c in m}
        for q in range(P):
            lb, ub = w.region(part, q, 2)
            for cell in brute_luse(shape, lb, ub, uses):
                c = int(np.ravel_multi_index(cell, shape))
                o = int(owner_before[cell])
                if o >= 0 and o != q and not (int(valid_before[cell]) >> q) & 1:
                    assert (q, c) in sent
        # the identical use-only call again: nothing left to send (P4)
        w.apply(O.K_NONE, part, [(X, uses, [])])
        assert len(w.msgs()) == 0
        # now redefine X under a random partition
        w.apply(O.K_NONE, parts[rng.integers(3)], [(X, [], defs or [(0, 0)])])
        owner_before = w.owner_map(X)
        valid_before = w.valid_map(X)
        if defs:
            pass


def test_unchanged_partition_zero_offsets_no_messages(oracle_mod):
    """P4 (north_star): an unchanged partition with zero use offsets generates no messages."""
    O = oracle_mod
    for P in (2, 4, 8):
        w = O.Oracle(P)
        X = w.create(O.F64, (32, 24))
        for kind in (O.ROW, O.COL, O.BLOCK):
            part = w.partition(kind, (32, 24))
            w.write(X, part, synth.uniform(1, (32, 24)))
            for _ in range(3):
                w.apply(O.K_SCALE, part, [(X, ZERO2, ZERO2)], [2.0])
                assert len(w.msgs()) == 0


def test_owner_and_valid_after_defs(oracle_mod):
    """Eq. 3-4 with last-writer semantics: after a def by p the cell is owned by p and
    valid only on p; a later read moves it and marks the reader valid."""
    O = oracle_mod
    w = O.Oracle(2)
    X = w.create(O.F64, (8, 8))
    rowp = w.partition(O.ROW, (8, 8))
    colp = w.partition(O.COL, (8, 8))
    w.apply(O.K_NONE, rowp, [(X, [], ZERO2)])
    own = w.owner_map(X)
    assert (own[:4] == 0).all() and (own[4:] == 1).all()
    w.apply(O.K_NONE, colp, [(X, [], ZERO2)])
    own = w.owner_map(X)
    assert (own[:, :4] == 0).all() and (own[:, 4:] == 1).all()
    # the SURVEY A7 counterexample: literal Eq. 3-4 would resend stale cells here;
    # last-writer semantics send nothing (everything used is own)
    w.apply(O.K_NONE, colp, [(X, ZERO2, [])])
    assert len(w.msgs()) == 0
    w.read(X, rowp)
    m = w.msgs()
    assert len(m) == 32  # each row half needs the other device's column half: 2 x 16
    assert set(map(tuple, m[:, 1:3].tolist())) == {(0, 1), (1, 0)}


# ---------------------------------------------------------------------------
# P5: GEMM all-gather ("detects and generates all-gather collective
# communication"), then silence on repeat (P:L390-393 reuse; nothing new defined)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("P", [2, 4])
def test_gemm_allgather_then_silence(oracle_mod, P):
    O = oracle_mod
    ni, nj, nk = 12, 10, 8
    w = O.Oracle(P)
    A = w.create(O.BF16, (ni, nk))
    B = w.create(O.BF16, (nk, nj))
    C = w.create(O.F32, (ni, nj))
    pa = w.partition(O.ROW, (ni, nk))
    pb = w.partition(O.ROW, (nk, nj))
    pc = w.partition(O.ROW, (ni, nj))
    w.write(A, pa, synth.uniform(3, (ni, nk), "bf16"))
    w.write(B, pb, synth.uniform(4, (nk, nj), "bf16"))
    w.write(C, pc, np.zeros((ni, nj), np.float32))
    acc = [(C, [], ZERO2), (A, [(0, S)], []), (B, [(S, 0)], [])]
    w.apply(O.K_GEMM, pc, acc, [1.0, 0.0])
    by = O.msgs_by_pair(w.msgs())
    assert len(by) == P * (P - 1)
    for (arr, src, dst), cells in by.items():
        assert arr == B
        lb, ub = w.region(pb, src, 2)
        expect = np.arange(lb[0] * nj, ub[0] * nj)
        np.testing.assert_array_equal(cells, expect)
    w.apply(O.K_GEMM, pc, acc, [1.0, 0.0])
    assert len(w.msgs()) == 0


# ---------------------------------------------------------------------------
# P6: Dirichlet eigenmodes (closed form) through the whole distributed pipeline
# ---------------------------------------------------------------------------
def _pingpong(O, w, kernel, part, X, Y, uses, sweeps):
    for s in range(sweeps):
        src, dst = (X, Y) if s % 2 == 0 else (Y, X)
        w.apply(kernel, part, [(dst, [], [(0,) * len(uses[0])]), (src, uses, [])])
    return X if sweeps % 2 == 0 else Y


@pytest.mark.parametrize("kernel,P,kind", [("jacobi", 4, "ROW"), ("jacobi", 3, "COL"),
                                           ("stencil9", 4, "BLOCK"), ("stencil9", 2, "ROW")])
def test_eigenmode_2d(oracle_mod, kernel, P, kind):
    O = oracle_mod
    # |lambda|^s kept in [0.05, 0.95]: rounding noise in slow modes does not swamp a
    # decayed mode, and a stale halo still changes the result by far more than 1e-12
    n0, n1, sweeps = 34, 40, 12
    a, b = (29, 35) if kernel == "jacobi" else (3, 4)
    u0 = synth.eigenmode2d(n0, n1, a, b)
    ta, tb = a * np.pi / (n0 - 1), b * np.pi / (n1 - 1)
    if kernel == "jacobi":
        lam = (np.cos(ta) + np.cos(tb)) / 2
        K, uses = O.K_JACOBI5, JAC_USES
    else:
        lam = (8 * (np.cos(ta) + np.cos(tb)) + 4 * np.cos(ta) * np.cos(tb)) / 20
        K, uses = O.K_STENCIL9, [(i, j) for i in (-1, 0, 1) for j in (-1, 0, 1) if i or j]
    w = O.Oracle(P)
    X = w.create(O.F64, (n0, n1), u0)
    Y = w.create(O.F64, (n0, n1), u0)
    part = w.partition(getattr(O, kind), (n0, n1), (1, 1), (n0 - 1, n1 - 1))
    R = _pingpong(O, w, K, part, X, Y, uses, sweeps)
    full = w.partition(O.ROW, (n0, n1))
    got = w.read(R, full)
    ref = lam ** sweeps * u0
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < 1e-12
    # the interior really changed (lambda^s is far from 1)
    assert 0.05 < abs(lam ** sweeps) < 0.95


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-12), ("f32", 2e-5)])
def test_eigenmode_3d(oracle_mod, dtype, tol):
    O = oracle_mod
    n, a, b, c, sweeps, P = 14, 11, 10, 12, 6, 4
    npdt = np.float64 if dtype == "f64" else np.float32
    u0 = synth.eigenmode3d(n, n, n, a, b, c, npdt)
    th = [k * np.pi / (n - 1) for k in (a, b, c)]
    lam = sum(np.cos(t) for t in th) / 3
    uses = [(0, 0, -1), (0, 0, 1), (0, -1, 0), (0, 1, 0), (-1, 0, 0), (1, 0, 0)]
    w = O.Oracle(P)
    DT = O.F64 if dtype == "f64" else O.F32
    X = w.create(DT, (n, n, n), u0)
    Y = w.create(DT, (n, n, n), u0)
    part = w.partition(O.ROW, (n, n, n), (1, 1, 1), (n - 1, n - 1, n - 1))
    R = _pingpong(O, w, O.K_STENCIL7_3D, part, X, Y, uses, sweeps)
    got = w.read(R, w.partition(O.ROW, (n, n, n))).astype(np.float64)
    ref = lam ** sweeps * u0.astype(np.float64)
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < tol


# ---------------------------------------------------------------------------
# P7: integer harmonic fields are exact fixed points
# ---------------------------------------------------------------------------
def test_harmonic_fixed_points(oracle_mod):
    O = oracle_mod
    n0, n1 = 20, 18
    u = synth.harmonic2d(n0, n1)
    for K, uses in ((O.K_JACOBI5, JAC_USES),
                    (O.K_STENCIL9, [(i, j) for i in (-1, 0, 1) for j in (-1, 0, 1) if i or j])):
        w = O.Oracle(4)
        X = w.create(O.F64, (n0, n1), u)
        Y = w.create(O.F64, (n0, n1), np.zeros((n0, n1)))
        part = w.partition(O.BLOCK, (n0, n1), (1, 1), (n0 - 1, n1 - 1))
        w.apply(K, part, [(Y, [], ZERO2), (X, uses, [])])
        got = w.read(Y, part)
        np.testing.assert_array_equal(got[1:-1, 1:-1], u[1:-1, 1:-1])
        assert (got[0] == 0).all() and (got[:, 0] == 0).all()  # outside work: untouched
    u3 = synth.harmonic3d(10, 9, 8)
    w = O.Oracle(2)
    X = w.create(O.F32, u3.shape, u3)
    Y = w.create(O.F32, u3.shape)
    part = w.partition(O.ROW, u3.shape, (1, 1, 1), tuple(s - 1 for s in u3.shape))
    uses = [(0, 0, -1), (0, 0, 1), (0, -1, 0), (0, 1, 0), (-1, 0, 0), (1, 0, 0)]
    w.apply(O.K_STENCIL7_3D, part, [(Y, [], [(0, 0, 0)]), (X, uses, [])])
    got = w.read(Y, part)
    np.testing.assert_array_equal(got[1:-1, 1:-1, 1:-1], u3[1:-1, 1:-1, 1:-1])


def test_asymmetric_stencil_orientation(oracle_mod):
    """A field that is harmonic along rows but not columns distinguishes the two axes:
    u = i (linear in the row index) is a Jacobi fixed point; u = i^2 is not (second
    difference 2 -> each sweep adds 2/4 = 0.5 exactly)."""
    O = oracle_mod
    n0, n1 = 10, 12
    i = np.arange(n0, dtype=np.float64)[:, None] * np.ones((1, n1))
    for u, delta in ((i, 0.0), (i * i, 0.5), ((i * i).T.copy() if n0 == n1 else None, None)):
        if u is None:
            continue
        w = O.Oracle(2)
        X = w.create(O.F64, u.shape, u)
        Y = w.create(O.F64, u.shape)
        part = w.partition(O.ROW, u.shape, (1, 1), (n0 - 1, n1 - 1))
        w.apply(O.K_JACOBI5, part, [(Y, [], ZERO2), (X, JAC_USES, [])])
        got = w.read(Y, part)
        np.testing.assert_array_equal(got[1:-1, 1:-1], u[1:-1, 1:-1] + delta)
    # columns: u = j^2 also gains 0.5 exactly
    j = np.arange(n1, dtype=np.float64)[None, :] * np.ones((n0, 1))
    w = O.Oracle(3)
    X = w.create(O.F64, j.shape, j * j)
    Y = w.create(O.F64, j.shape)
    part = w.partition(O.COL, j.shape, (1, 1), (n0 - 1, n1 - 1))
    w.apply(O.K_JACOBI5, part, [(Y, [], ZERO2), (X, JAC_USES, [])])
    np.testing.assert_array_equal(w.read(Y, part)[1:-1, 1:-1], (j * j)[1:-1, 1:-1] + 0.5)


# ---------------------------------------------------------------------------
# COPY / SCALE / STAMP / bf16 rounding
# ---------------------------------------------------------------------------
def test_copy_raw_bits_and_scale(oracle_mod):
    O = oracle_mod
    shape = (11, 13)
    bits = synth.random_bits(7, shape, "f64")  # NaN payloads, denormals, infinities
    w = O.Oracle(3)
    X = w.create(O.F64, shape)
    Y = w.create(O.F64, shape)
    rowp = w.partition(O.ROW, shape)
    colp = w.partition(O.COL, shape)
    w.write(X, rowp, bits)
    w.apply(O.K_COPY, colp, [(Y, [], ZERO2), (X, ZERO2, [])])
    got = w.read(Y, colp)
    assert got.view(np.uint64).tolist() == bits.view(np.uint64).tolist()
    v = synth.uniform(8, shape)
    w.write(X, rowp, v)
    w.apply(O.K_SCALE, colp, [(X, ZERO2, ZERO2)], [2.0])
    np.testing.assert_array_equal(w.read(X, rowp), 2.0 * v)  # power-of-two scaling is exact


def test_splitmix64_vector_and_stamp(oracle_mod):
    O = oracle_mod
    # published first outputs of splitmix64 seeded with 0 (Vigna, splitmix64.c)
    assert O.splitmix64(0) == 0xE220A8397B1DCDAF
    assert O.splitmix64(0x9E3779B97F4A7C15) == 0x6E789E6AA1B965F4
    # STAMP: cell c of seed s gets splitmix64(s*GOLDEN + c); cell 0 of seeds 0 and 1
    # are therefore the first two published outputs
    for seed, first in ((0, 0xE220A8397B1DCDAF), (1, 0x6E789E6AA1B965F4)):
        w = O.Oracle(2)
        X = w.create(O.I64, (4, 6))
        part = w.partition(O.ROW, (4, 6))
        w.apply(O.K_STAMP, part, [(X, [], [(0, 0)])], [float(seed)])
        got = w.read(X, part).view(np.uint64).reshape(-1)
        assert int(got[0]) == first
        assert len(set(got.tolist())) == 24
        assert w.owner_map(X).tolist() == [[0] * 6] * 2 + [[1] * 6] * 2


def test_bf16_rounding_pins(oracle_mod):
    O = oracle_mod
    # round-to-nearest-even at 8 significant bits
    assert O.f64_to_bf16(257.0) == 0x4380  # tie between 256 and 258 -> even (256)
    assert O.f64_to_bf16(259.0) == 0x4382  # tie between 258 and 260 -> even (260)
    assert O.f64_to_bf16(1.0 / 3.0) == 0x3EAB
    assert O.f32_to_bf16(np.float32(1.0 / 3.0)) == 0x3EAB
    assert O.f64_to_bf16(-2.0) == 0xC000
    assert O.f64_to_bf16(2.0**-133) == 0x0001  # smallest subnormal
    assert O.f64_to_bf16(1e39) == 0x7F80       # overflow -> inf
    assert O.f64_to_bf16(float("nan")) & 0x7FC0 == 0x7FC0


# ---------------------------------------------------------------------------
# P7: GEMM with integer bf16 inputs is exact; compare with int64 matmul
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("cdt", ["f32", "bf16"])
def test_gemm_integer_exact(oracle_mod, cdt):
    O = oracle_mod
    ni, nj, nk, P = 12, 9, 40, 3
    Ab = synth.int_bf16(11, (ni, nk))
    Bb = synth.int_bf16(12, (nk, nj))
    Ai = synth.bf16_to_f32(Ab).astype(np.int64)
    Bi = synth.bf16_to_f32(Bb).astype(np.int64)
    exact = Ai @ Bi
    w = O.Oracle(P)
    A = w.create(O.BF16, (ni, nk), Ab)
    B = w.create(O.BF16, (nk, nj), Bb)
    C = w.create(O.F32 if cdt == "f32" else O.BF16, (ni, nj))
    pc = w.partition(O.ROW, (ni, nj))
    w.apply(O.K_GEMM, pc, [(C, [], ZERO2), (A, [(0, S)], []), (B, [(S, 0)], [])], [1.0, 0.0])
    got = w.read(C, pc)
    if cdt == "f32":
        np.testing.assert_array_equal(got.astype(np.int64), exact)
    else:
        vals = synth.bf16_to_f32(got).astype(np.float64)
        # |exact| < 2^11 here, so bf16 (8 significant bits) error is < 2^3; check RNE bound
        assert np.all(np.abs(vals - exact) <= np.maximum(1.0, np.abs(exact) * 2.0**-8))
    # alpha/beta: C = 2*A@B - 1*C
    w.apply(O.K_GEMM, pc, [(C, ZERO2, ZERO2), (A, [(0, S)], []), (B, [(S, 0)], [])], [2.0, -1.0])
    if cdt == "f32":
        np.testing.assert_array_equal(w.read(C, pc).astype(np.int64), exact)
    samp = O.gemm_sample(Ab, Bb, [0, 5, 11], [0, 3, 8])
    np.testing.assert_array_equal(samp, exact[[0, 5, 11], [0, 3, 8]].astype(np.float64))


# ---------------------------------------------------------------------------
# partitions (Listing 1)
# ---------------------------------------------------------------------------
def test_partitions(oracle_mod):
    O = oracle_mod
    w = O.Oracle(4)
    p = w.partition(O.ROW, (10, 8))
    sizes = [w.region(p, d, 2)[1][0] - w.region(p, d, 2)[0][0] for d in range(4)]
    assert sizes == [3, 3, 2, 2]
    w8 = O.Oracle(8)
    b = w8.partition(O.BLOCK, (16, 16))
    regs = [w8.region(b, d, 2) for d in range(8)]
    assert regs[0] == ((0, 0), (4, 8)) and regs[1] == ((0, 8), (4, 16)) and regs[7] == ((12, 8), (16, 16))
    # Listing 1 read as (start, length) (reading R2): tiles the 10240 rows exactly
    w2 = O.Oracle(2)
    w2.partition_manual((10240, 10240), [[0, 0], [3008, 0]], [[3008, 10240], [10240, 10240]])
    with pytest.raises(O.OracleError) as e:
        w2.partition_manual((16, 16), [[0, 0], [4, 0]], [[8, 16], [16, 16]])
    assert e.value.code == O.EOVERLAP
    with pytest.raises(O.OracleError) as e:
        O.Oracle(2).partition(O.COL, (16,))
    assert e.value.code == O.EUNSUPPORTED


def test_race_and_validation(oracle_mod):
    O = oracle_mod
    w = O.Oracle(2)
    X = w.create(O.F64, (8, 8))
    Y = w.create(O.F64, (8, 8))
    part = w.partition(O.ROW, (8, 8))
    inner = w.partition(O.ROW, (8, 8), (1, 1), (7, 7))
    with pytest.raises(O.OracleError) as e:
        w.apply(O.K_NONE, part, [(X, [], [(0, 0), (1, 0)])])
    assert e.value.code == O.ERACE
    with pytest.raises(O.OracleError) as e:  # undeclared footprint
        w.apply(O.K_JACOBI5, inner, [(Y, [], ZERO2), (X, JAC_USES[:3], [])])
    assert e.value.code == O.EINVAL
    with pytest.raises(O.OracleError) as e:  # work + halo outside the array
        w.apply(O.K_JACOBI5, part, [(Y, [], ZERO2), (X, JAC_USES, [])])
    assert e.value.code == O.ERANGE
    with pytest.raises(O.OracleError) as e:  # in-place stencil
        w.apply(O.K_JACOBI5, inner, [(X, [], ZERO2), (X, JAC_USES, [])])
    assert e.value.code == O.EINVAL


# ---------------------------------------------------------------------------
# P9: Table 3 communication patterns as closed forms
# ---------------------------------------------------------------------------
def test_jacobi_volume_closed_form(oracle_mod):
    """Jacobi paper form: steady state 2(P-1) rows of interior width per sweep
    (Table 3: 473 GB = 1e5 * 2(P-1) * 20480 * 4 B at P=32)."""
    O = oracle_mod
    P, n0, n1 = 32, 98, 12
    w = O.Oracle(P, with_data=False)
    A = w.create(O.F32, (n0, n1))
    B = w.create(O.F32, (n0, n1))
    data = w.partition(O.ROW, (n0, n1))
    work = w.partition(O.ROW, (n0, n1), (1, 1), (n0 - 1, n1 - 1))
    w.write(A, data, None)
    w.write(B, data, None)
    vols = []
    for s in range(4):
        w.apply(O.K_JACOBI5, work, [(A, [], ZERO2), (B, JAC_USES, [])])
        vols.append(len(w.msgs()))
        w.apply(O.K_COPY, work, [(B, [], ZERO2), (A, ZERO2, [])])
        assert len(w.msgs()) == 0
    assert vols[1:] == [2 * (P - 1) * (n1 - 2)] * 3


def test_2mm_row_vs_col(oracle_mod):
    """2MM: ROW sends B once and D every iteration; COL sends A and C once."""
    O = oracle_mod
    P, n, iters = 4, 16, 3
    for kind in ("ROW", "COL"):
        w = O.Oracle(P, with_data=False)
        A, B, C, D, E = (w.create(O.BF16, (n, n)) for _ in range(5))
        E = w.create(O.F32, (n, n))
        D = w.create(O.BF16, (n, n))
        part = w.partition(getattr(O, kind), (n, n))
        for X in (A, B, C):
            w.write(X, part, None)
        per_iter = []
        for it in range(iters):
            w.apply(O.K_GEMM, part, [(D, [], ZERO2), (A, [(0, S)], []), (B, [(S, 0)], [])], [1.0, 0.0])
            m1 = O.msgs_by_pair(w.msgs())
            w.apply(O.K_GEMM, part, [(E, [], ZERO2), (C, [(0, S)], []), (D, [(S, 0)], [])], [1.0, 0.0])
            m2 = O.msgs_by_pair(w.msgs())
            per_iter.append(({k[0] for k in m1}, {k[0] for k in m2},
                             sum(len(v) for v in m1.values()) + sum(len(v) for v in m2.values())))
        full = (P - 1) * n * n
        if kind == "ROW":
            assert per_iter[0] == ({B}, {D}, 2 * full)
            assert all(p == (set(), {D}, full) for p in per_iter[1:])
        else:
            assert per_iter[0] == ({A}, {C}, 2 * full)
            assert all(p == (set(), set(), 0) for p in per_iter[1:])


def test_read_after_write_same_partition_is_local(oracle_mod):
    O = oracle_mod
    w = O.Oracle(4)
    X = w.create(O.F32, (10, 10))
    part = w.partition(O.BLOCK, (10, 10))
    v = synth.uniform(5, (10, 10), "f32")
    w.write(X, part, v)
    np.testing.assert_array_equal(w.read(X, part), v)
    assert len(w.msgs()) == 0


# ---------------------------------------------------------------------------
# Reduce (Table 2): closed forms after a redistribution
# ---------------------------------------------------------------------------
def test_reduce_closed_forms(oracle_mod):
    O = oracle_mod
    n0, n1, P = 12, 10, 3
    i = np.arange(n0)[:, None]
    j = np.arange(n1)[None, :]
    u = (i * n1 + j + 1).astype(np.float64)  # 1 .. n0*n1
    w = O.Oracle(P)
    X = w.create(O.F64, (n0, n1))
    rowp = w.partition(O.ROW, (n0, n1))
    colp = w.partition(O.COL, (n0, n1))
    inner = w.partition(O.BLOCK, (n0, n1), (2, 3), (9, 8))
    w.write(X, rowp, u)
    N = n0 * n1
    assert w.reduce(X, colp, O.SUM) == N * (N + 1) / 2       # Gauss
    assert len(w.msgs()) > 0                                 # coherence moved data (ROW -> COL)
    assert w.reduce(X, colp, O.MAX) == N and w.reduce(X, colp, O.MIN) == 1
    sub = u[2:9, 3:8]
    assert w.reduce(X, inner, O.SUM) == sub.sum() and w.reduce(X, inner, O.MAX) == sub.max()
    # PROD of powers of two is exact: 2^(sum of exponents)
    e = ((i + j) % 5 - 2).astype(np.float64)
    w.write(X, rowp, 2.0 ** e)
    assert w.reduce(X, rowp, O.PROD) == 2.0 ** e.sum()
    Y = w.create(O.I64, (n0, n1))
    w.write(Y, colp, -(i * n1 + j).astype(np.int64))
    assert w.reduce(Y, rowp, O.SUM) == -(N - 1) * N / 2 and w.reduce(Y, rowp, O.MIN) == -(N - 1)


# ---------------------------------------------------------------------------
# absolute sections + trapezoids (Table 1 use@/def@, Table 2 SetAbsolute*/SetTrapezoid*)
# ---------------------------------------------------------------------------
def test_trapezoid_closed_forms(oracle_mod):
    O = oracle_mod
    # upper-triangular n x n incl. diagonal: row r spans [r, n-1] -> n(n+1)/2 cells
    n = 9
    boxes = O.trapezoid([(0, 0), (0, n - 1), (n - 1, n - 1), (n - 1, n - 1)])
    assert len(boxes) == n and sum(u[1] - l[1] for l, u in boxes) == n * (n + 1) // 2
    assert boxes[3] == ((3, 3), (4, n))
    # lower triangle: row r spans [0, r]
    boxes = O.trapezoid([(2, 0), (2, 0), (6, 0), (6, 4)])
    assert [(l[1], u[1]) for l, u in boxes] == [(0, 1), (0, 2), (0, 3), (0, 4), (0, 5)]
    # rectangle, and a single row
    assert O.trapezoid([(1, 2), (1, 5), (3, 2), (3, 5)]) == [((r, 2), (r + 1, 6)) for r in (1, 2, 3)]
    assert O.trapezoid([(4, 1), (4, 3), (4, 1), (4, 3)]) == [((4, 1), (5, 4))]
    # round half up on the interpolated edge: width 3 over 2 steps -> 0, 2 (1.5 -> 2), 3
    assert [l[1] for l, _ in O.trapezoid([(0, 0), (0, 9), (2, 3), (2, 9)])] == [0, 2, 3]


def test_absolute_sections_triangular(oracle_mod):
    """Correlation-style symmetric fill: device p defines the
    upper-triangle rows of its manual row block, then every device uses the full
    rows of the mirrored lower triangle -> only defined-elsewhere cells move."""
    O = oracle_mod
    n, P = 12, 2
    w = O.Oracle(P)
    X = w.create(O.F64, (n, n))
    part = w.partition_manual((n, n), [[0, 0], [4, 0]], [[4, n], [n, n]])  # Listing 1 style (R2)
    up = O.trapezoid([(0, 0), (0, n - 1), (n - 1, n - 1), (n - 1, n - 1)])
    defs = [[b for b in up if b[0][0] < 4], [b for b in up if b[0][0] >= 4]]
    uses = [[((0, 0), (4, n))], [((4, 0), (n, n))]]
    w.apply_abs(O.K_STAMP, part, [(X, [[], []], defs)], [3.0])
    own = w.owner_map(X)
    assert (own[np.triu_indices(n)] == np.where(np.triu_indices(n)[0] < 4, 0, 1)).all()
    assert (own[np.tril_indices(n, -1)] == -1).all()
    w.apply_abs(O.K_NONE, part, [(X, uses, [[], []])])
    m = w.msgs()
    # device 0 (rows 0-3) owns all of its rows' upper part: nothing to receive;
    # device 1 (rows 4-11) owns its upper part too: the triangles never cross
    assert len(m) == 0
    # now device 1 reads all rows: it needs device 0's triangle rows 0-3 (cols r..n-1)
    w.apply_abs(O.K_NONE, part, [(X, [[], [((0, 0), (n, n))]], [[], []])])
    cells = set(int(c) for c in w.msgs()[:, 3])
    expect = {r * n + c for r in range(4) for c in range(r, n)}
    assert cells == expect
    with pytest.raises(O.OracleError) as e:
        w.apply_abs(O.K_NONE, part, [(X, [[], []], [[((0, 0), (2, 2))], [((1, 1), (3, 3))]])])
    assert e.value.code == O.ERACE
