"""GPU scenarios run in a subprocess (the delay hooks and kernel switches are read once
per process): WAR races, the TMA stencil shapes, the gated product.

    python tests/gpu_scenarios.py pull_war <n_gpus>
    python tests/gpu_scenarios.py staged_regrow <n_gpus>
    HDA_TMA=2 python tests/gpu_scenarios.py tma_shapes 1
    HDA_CE_BYTES=262144 python tests/gpu_scenarios.py gemm_gate <n_gpus>

Each prints "OK" or a mismatch description and exits 0 / 1.  Test code only: the
library runs the program, the oracle replays it, every replica is compared bit for bit.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import paper_1809_05657_b200 as H  # noqa: E402
import synth  # noqa: E402


def _compare(h, w, arrs, P):
    bad = []
    for a in arrs:
        if not (h.owner_map(a) == w.owner_map(a)).all():
            bad.append(f"array {a}: owner map")
        for d in range(P):
            if h.read_replica(a, d).tobytes() != w.replica(a, d).tobytes():
                bad.append(f"array {a} device {d}: replica differs")
    return bad


def pull_war(G):
    """Three devices, reader-side WAR: q=0 writes rows 0-3 of X; r=1 pulls
    them from q (r's pulls sleep, HDA_DEBUG_PULL_DELAY_DEV=1); p=2 redefines them
    (waiting on no one: r read q's replica, not p's); then q pulls them back from p
    into its own replica.  Unless q's pull waits for r's ACK, r reads p's new values
    out of q's replica and its copy Y differs from the oracle's."""
    P, shape = 3, (12, 64)
    h = H.HDArray(n_gpus=G, n_devices=P)
    w = O.Oracle(P)
    x0 = synth.uniform(21, shape)
    empty = ([0, 0], [0, 0])

    def manual(be, rows):  # device d works on rows[d] (None = empty region)
        lbs, ubs = [], []
        for r in rows:
            if r is None:
                lbs.append(list(empty[0]))
                ubs.append(list(empty[1]))
            else:
                lbs.append([r[0], 0])
                ubs.append([r[1], shape[1]])
        return be.partition_manual(shape, lbs, ubs)

    parts = {}
    for be in (h, w):
        X, Y, Z = (be.create(H.F64, shape) for _ in range(3))
        D = manual(be, [(0, 4), (4, 8), (8, 12)])
        W1 = manual(be, [None, (0, 4), None])
        W2 = manual(be, [None, None, (0, 4)])
        W3 = manual(be, [(0, 4), None, None])
        parts[be] = (X, Y, Z, D, W1, W2, W3)
    bad = []
    for it in range(3):
        for be in (h, w):
            X, Y, Z, D, W1, W2, W3 = parts[be]
            be.write(X, D, x0 + it)
            be.apply(H.K_COPY, W1, [(Y, [], [(0, 0)]), (X, [(0, 0)], [])])             # r pulls from q
            be.apply(H.K_STAMP, W2, [(X, [], [(0, 0)])], [float(100 + it)])            # p redefines
            be.apply(H.K_COPY, W3, [(Z, [], [(0, 0)]), (X, [(0, 0)], [])])             # q pulls from p
        X, Y, Z = parts[h][:3]
        bad += [f"it{it}: {b}" for b in _compare(h, w, [X, Y, Z], P)]
    h.close()
    return bad


def staged_regrow(G):
    """STAGED transport: a cached small-message plan (Jacobi halos) is
    replayed after a larger plan (a ROW->COL repartition with 2 MiB blocks) has grown
    the staging buffers; the replay must use the new buffers."""
    P = 2
    h = H.HDArray(n_gpus=G, n_devices=P)
    h.set_transport(1)
    w = O.Oracle(P)
    J = [(0, -1), (0, 1), (-1, 0), (1, 0)]
    shape, big = (34, 130), (1024, 1024)
    u0, v0 = synth.uniform(3, shape), synth.uniform(4, big, "f32")
    arrs = {}
    for be in (h, w):
        Xa, Ya = be.create(H.F64, shape, u0), be.create(H.F64, shape, u0)
        part = be.partition(H.ROW, shape, (1, 1), (shape[0] - 1, shape[1] - 1))
        Zb = be.create(H.F32, big)
        rp, cp = be.partition(H.ROW, big), be.partition(H.COL, big)
        be.write(Zb, rp, v0)
        arrs[be] = (Xa, Ya, part, Zb, rp, cp)

    def jacobi(n):
        for s in range(n):
            for be in (h, w):
                Xa, Ya, part = arrs[be][:3]
                src, dst = (Xa, Ya) if s % 2 == 0 else (Ya, Xa)
                be.apply(H.K_JACOBI5, part, [(dst, [], [(0, 0)]), (src, J, [])])

    jacobi(6)                       # small plans cached, staging at its 1 MiB minimum
    for be in (h, w):
        Zb, rp, cp = arrs[be][3:]
        be.apply(H.K_SCALE, cp, [(Zb, [(0, 0)], [(0, 0)])], [2.0])   # 2 MiB blocks: regrow
        be.apply(H.K_SCALE, rp, [(Zb, [(0, 0)], [(0, 0)])], [0.5])
    jacobi(6)                       # cached small plans replayed
    Xa, Ya, _, Zb = arrs[h][:4]
    bad = _compare(h, w, [Xa, Ya, Zb], P)
    h.close()
    return bad


def tma_shapes(G):
    """TMA-ring 2-D stencils (stencil_tma.cu) on boxes spanning several 252/248-column
    strips and several row blocks, with ragged ends, boxes that start off the 32-byte
    strip alignment and partitions whose devices get different tile heights; every
    replica against the oracle, bit for bit, f64 and f32, 5- and 9-point, uniform and
    special-value inputs."""
    J = [(0, -1), (0, 1), (-1, 0), (1, 0)]
    N9 = [(i, j) for i in (-1, 0, 1) for j in (-1, 0, 1) if i or j]
    bad = []
    cases = [((517, 1111), 1, (1, 1), None), ((300, 1500), 2, (5, 7), (291, 1433)), ((1000, 600), 3, (1, 3), None),
             ((133, 2050), 1, (40, 250), (100, 1900))]
    for dt, name in ((H.F64, "f64"), (H.F32, "f32")):
        # the first shape also with Inf / signed zeros / subnormals / huge values mixed in
        # (the divisions' slow paths inside the TMA consumers)
        for ci, (shape, P, lb, ub, u0) in enumerate(
                [(c[0], c[1], c[2], c[3], synth.uniform(31, c[0], name)) for c in cases] +
                [(cases[0][0], 2, cases[0][2], None, synth.special_values(32, cases[0][0], name))]):
            ub = ub or (shape[0] - 1, shape[1] - 1)
            for K, uses in ((H.K_JACOBI5, J), (H.K_STENCIL9, N9)):
                h = H.HDArray(n_gpus=G, n_devices=P)
                w = O.Oracle(P)
                for be in (h, w):
                    X = be.create(dt, shape, u0)
                    Y = be.create(dt, shape, u0)
                    part = be.partition(H.ROW, shape, lb, ub)
                    for s in range(3):
                        src, dst = (X, Y) if s % 2 == 0 else (Y, X)
                        be.apply(K, part, [(dst, [], [(0, 0)]), (src, uses, [])])
                bad += [f"{name} {shape} P={P} K={K}: {b}" for b in _compare(h, w, [X, Y], P)]
                h.close()
    return bad


def gemm_gate(G):
    """2MM under ROW: D = A x B, E = C x D on P = G GPUs.  Every incoming
    message is a full-width row block of B (call 1) or D (every call) from another GPU
    on the copy engine, so the product runs gated on their arrival (KGate, own rows
    first) instead of after a join.  Integer bf16 inputs in [-1, 1]: D rounds to bf16
    the same way on both sides and |E| <= 2^20, so E (fp32) is exact in any k order and
    every replica must equal the oracle's bit for bit.  HDA_GEMM_GATE=2 (the default)
    splits the fp32 products into a launch beside the copies and one after them, 1 gates
    inside the kernel, 0 joins (the A/B).  Exits nonzero on a mismatch or when no product was gated
    though gating is on."""
    P, S = G, H.STAR
    bad, gated = [], 0
    # 1024: k-block aligned row blocks; 1064: blocks of 532 / 266 rows, so k-blocks
    # straddle two sources (or own rows and a source) and the segments are ragged
    for n in (1024, 1064):
        Ab, Bb, Cb = (synth.int_bf16(70 + i, (n, n), -1, 1) for i in range(3))
        h = H.HDArray(n_gpus=G, n_devices=P)
        w = O.Oracle(P)
        for be in (h, w):
            A, B, C, D = (be.create(H.BF16, (n, n)) for _ in range(4))
            E = be.create(H.F32, (n, n))
            part = be.partition(H.ROW, (n, n))
            for X, v in ((A, Ab), (B, Bb), (C, Cb)):
                be.write(X, part, v)
            for it in range(3):
                be.apply(H.K_GEMM, part, [(D, [], [(0, 0)]), (A, [(0, S)], []), (B, [(S, 0)], [])], [1.0, 0.0])
                be.apply(H.K_GEMM, part, [(E, [], [(0, 0)]), (C, [(0, S)], []), (D, [(S, 0)], [])], [1.0, 0.0])
        bad += [f"n={n}: {b}" for b in _compare(h, w, [B, D, E], P)]
        gated += h.stats()["gated_products"]
        h.close()
    # the gated kernel is the CTA-pair one (HDA_GEMM_2SM=0 selects the single-CTA kernel)
    mode = os.environ.get("HDA_GEMM_GATE", "2") if os.environ.get("HDA_GEMM_2SM", "1") != "0" else "0"
    # 1: per size B once and D three times on every device; 2 (split): only the fp32 E
    # products with whole k-blocks per source (1024, not 1064), the bf16 D products join
    want = {"0": 0, "1": 2 * 4 * P, "2": 3 * P}[mode]
    if gated != want:
        bad.append(f"gated products {gated}, expected {want}")
    print(f"gated products: {gated}")
    return bad


if __name__ == "__main__":
    name, G = sys.argv[1], int(sys.argv[2])
    bad = {"pull_war": pull_war, "staged_regrow": staged_regrow, "tma_shapes": tma_shapes,
           "gemm_gate": gemm_gate}[name](G)
    print("OK" if not bad else "MISMATCH " + "; ".join(bad[:8]))
    sys.exit(1 if bad else 0)
