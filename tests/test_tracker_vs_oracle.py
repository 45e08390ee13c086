"""The library's rect-algebra tracker (plan-only contexts, no GPU) against the
per-element oracle: element-set equality of every message set and of every owner
map on random programs with partition switches (SPEC S:L676 acceptance 1), plus
the paper's closed forms at paper scale (Table 3)."""
import numpy as np
import pytest

import oracle as O
from programs import LibAdapter, gen_program, run_program

import paper_1809_05657_b200 as H


def compare_program(seed, P, ndim):
    prog = gen_program(seed, P, ndim=ndim, n_ops=10)
    w = O.Oracle(P, with_data=False)
    h = H.HDArray(n_gpus=0, n_devices=P)
    lib = LibAdapter(h)
    rec = {}

    def on_oracle(step, op, arrs, status):
        rec[step] = (status, O.msgs_by_pair(w.msgs()) if status == 0 else None,
                     [w.owner_map(a) for a in arrs])

    def on_lib(step, op, arrs, status):
        st_o, msgs_o, own_o = rec[step]
        assert status == st_o, (seed, step, op, status, st_o)
        if status == 0:
            msgs_l = O.msgs_by_pair(lib.msgs())
            assert msgs_l.keys() == msgs_o.keys(), (seed, step, op)
            for k in msgs_o:
                np.testing.assert_array_equal(msgs_l[k], msgs_o[k])
        for a, own in zip(arrs, own_o):
            np.testing.assert_array_equal(h.owner_map(a), own)

    run_program(prog, w, on_oracle)
    run_program(prog, lib, on_lib)
    h.close()
    return prog


@pytest.mark.parametrize("P", [1, 2, 3, 4, 5, 8])
def test_random_programs_2d(P):
    for s in range(60):
        compare_program(10_000 * P + s, P, 2)


@pytest.mark.parametrize("P", [2, 4, 8])
def test_random_programs_3d_and_1d(P):
    for s in range(20):
        compare_program(20_000 * P + s, P, 3)
        compare_program(30_000 * P + s, P, 1)


def test_plan_cache_is_transparent():
    """Cache on vs off: identical plans on every call; steady
    state of a Jacobi sweep is served by the cache."""
    J = [(0, -1), (0, 1), (-1, 0), (1, 0)]
    plans = []
    for cache in (True, False):
        h = H.HDArray(n_gpus=0, n_devices=4)
        h.set_plan_cache(cache)
        A = h.create(H.F64, (40, 30))
        B = h.create(H.F64, (40, 30))
        data = h.partition(H.ROW, (40, 30))
        work = h.partition(H.BLOCK, (40, 30), (1, 1), (39, 29))
        h.write(A, data, None)
        h.write(B, data, None)
        seq = []
        for s in range(6):
            h.apply(H.K_JACOBI5, work, [(A, [], [(0, 0)]), (B, J, [])])
            seq.append(h.last_plan())
            h.apply(H.K_COPY, work, [(B, [], [(0, 0)]), (A, [(0, 0)], [])])
            seq.append(h.last_plan())
        st = h.stats()
        if cache:
            assert st["plan_hits"] >= 8
        else:
            assert st["plan_hits"] == 0
        plans.append(seq)
    assert plans[0] == plans[1]


def _gib(b):
    return b / 2**30


def test_table3_closed_forms_at_paper_scale():
    """Table 3 at 32 processes, 10240^2 fp32 arrays, plan-only:
    GEMM B all-gather, 2MM row vs custom (column) partitions, Jacobi per sweep."""
    P = 32
    n = 10240
    S = H.STAR
    # GEMM: exact message sets carry (P-1)|B|; the paper counts P|B| = 12.5 GiB
    h = H.HDArray(n_gpus=0, n_devices=P)
    A, B = h.create(H.BF16, (n, n)), h.create(H.BF16, (n, n))
    C = h.create(H.F32, (n, n))
    part = h.partition(H.ROW, (n, n))
    for X in (A, B, C):
        h.write(X, part, None)
    bytes_B = n * n * 4  # the paper's fp32 elements
    tot = 0
    for it in range(100):
        h.apply(H.K_GEMM, part, [(C, [], [(0, 0)]), (A, [(0, S)], []), (B, [(S, 0)], [])], [1.0, 0.0])
        tot += sum(np.prod(np.subtract(ub, lb)) for _, _, _, lb, ub in h.last_plan())
    assert tot == (P - 1) * n * n
    assert round(_gib(P * bytes_B), 1) == 12.5
    # 2MM: D = A x B ; E = C x D, 100 iterations
    for kind, expect_cells in ((H.ROW, (P - 1) * n * n * 101), (H.COL, (P - 1) * n * n * 2)):
        h = H.HDArray(n_gpus=0, n_devices=P)
        A, B, Cm, D = (h.create(H.BF16, (n, n)) for _ in range(4))
        E = h.create(H.F32, (n, n))
        part = h.partition(kind, (n, n))
        for X in (A, B, Cm):
            h.write(X, part, None)
        tot = 0
        for it in range(100):
            h.apply(H.K_GEMM, part, [(D, [], [(0, 0)]), (A, [(0, S)], []), (B, [(S, 0)], [])], [1.0, 0.0])
            tot += sum(np.prod(np.subtract(ub, lb)) for _, _, _, lb, ub in h.last_plan())
            h.apply(H.K_GEMM, part, [(E, [], [(0, 0)]), (Cm, [(0, S)], []), (D, [(S, 0)], [])], [1.0, 0.0])
            tot += sum(np.prod(np.subtract(ub, lb)) for _, _, _, lb, ub in h.last_plan())
        assert tot == expect_cells
        # the paper's P|X| accounting reproduces the printed numbers
        paper = expect_cells // (P - 1) * P * 4
        assert round(_gib(paper)) == (1262 if kind == H.ROW else 25)
    # Jacobi paper form, 20480 columns (+ghost ring), 10 sweeps -> per-sweep volume
    J = [(0, -1), (0, 1), (-1, 0), (1, 0)]
    rows, cols = 24080 + 2, 20480 + 2
    h = H.HDArray(n_gpus=0, n_devices=P)
    A, B = h.create(H.F32, (rows, cols)), h.create(H.F32, (rows, cols))
    data = h.partition(H.ROW, (rows, cols))
    work = h.partition(H.ROW, (rows, cols), (1, 1), (rows - 1, cols - 1))
    h.write(A, data, None)
    h.write(B, data, None)
    vols = []
    for s in range(5):
        h.apply(H.K_JACOBI5, work, [(A, [], [(0, 0)]), (B, J, [])])
        vols.append(h.stats()["last_bytes"])
        h.apply(H.K_COPY, work, [(B, [], [(0, 0)]), (A, [(0, 0)], [])])
        assert h.stats()["last_bytes"] == 0
    per_sweep = 2 * (P - 1) * 20480 * 4
    assert vols[2:] == [per_sweep] * 3
    assert round(_gib(1e5 * per_sweep)) == 473
    assert h.stats()["plan_hits"] >= 4


def test_trapezoid_helper_matches_oracle():
    rng = np.random.default_rng(11)
    for _ in range(300):
        top = int(rng.integers(0, 20))
        bottom = top + int(rng.integers(0, 15))
        c = [(top, int(rng.integers(0, 30))), (top, int(rng.integers(0, 30))),
             (bottom, int(rng.integers(0, 30))), (bottom, int(rng.integers(0, 30)))]
        assert H.trapezoid(c) == O.trapezoid(c), c


@pytest.mark.parametrize("P", [2, 3, 4])
def test_absolute_sections_random(P):
    """Random per-device absolute sections (triangles, rectangles) for uses and defs:
    message element sets and owner maps equal to the oracle."""
    rng = np.random.default_rng(100 + P)
    n = 16
    for trial in range(25):
        w = O.Oracle(P, with_data=False)
        h = H.HDArray(n_gpus=0, n_devices=P)
        parts = []
        for be in (w, h):
            X = be.create(H.F64, (n, n))
            parts.append(be.partition(H.ROW, (n, n)))
        # disjoint defs: row slabs, each a trapezoid clipped to its slab
        cuts = np.sort(rng.integers(0, n + 1, P - 1))
        bounds = [0] + list(cuts) + [n]
        for step in range(4):
            defs, uses = [], []
            for q in range(P):
                r0, r1 = int(bounds[q]), int(bounds[q + 1])
                if r1 > r0 and rng.random() < 0.8:
                    c = [(r0, int(rng.integers(0, n))), (r0, int(rng.integers(0, n))),
                         (r1 - 1, int(rng.integers(0, n))), (r1 - 1, int(rng.integers(0, n)))]
                    defs.append(H.trapezoid(c))
                else:
                    defs.append([])
                ub = []
                for _ in range(int(rng.integers(0, 3))):
                    a0, a1 = sorted(rng.integers(0, n + 1, 2))
                    b0, b1 = sorted(rng.integers(0, n + 1, 2))
                    ub.append(((int(a0), int(b0)), (int(a1), int(b1))))
                uses.append(ub)
            w.apply_abs(O.K_NONE, parts[0], [(X, uses, defs)])
            h.apply_abs(H.K_NONE, parts[1], [(X, uses, defs)])
            mo = O.msgs_by_pair(w.msgs())
            from programs import LibAdapter
            ml = O.msgs_by_pair(LibAdapter(h).msgs())
            assert mo.keys() == ml.keys()
            for k in mo:
                np.testing.assert_array_equal(mo[k], ml[k])
            np.testing.assert_array_equal(w.owner_map(X), h.owner_map(X))
        h.close()
