"""Random HDArray programs, replayed identically on the oracle and on the library.

A program is data: a list of ops over arrays and partitions.  The generator follows
SPEC S:L676 (shapes <= 32^2, P in 1..8, offsets in [-2,2] and '*', ROW/COL/BLOCK/manual
partitions, partition switches) and adds 3-D arrays.  Test code only.
"""
from __future__ import annotations

import numpy as np

import synth

STAR = -(2**31)


def gen_program(seed: int, P: int, ndim: int = 2, n_ops: int = 8, with_kernels: bool = False):
    rng = np.random.default_rng(seed)
    if ndim == 2:
        shape = (int(rng.integers(max(P, 3), 24)), int(rng.integers(3, 24)))
    elif ndim == 3:
        shape = (int(rng.integers(max(P, 3), 10)), int(rng.integers(3, 9)), int(rng.integers(3, 9)))
    else:
        shape = (int(rng.integers(max(P, 3), 60)),)
    dtype = int(rng.choice([0, 1, 2, 4]))  # f64 f32 bf16 i64
    parts = [("auto", 0, None, None)]
    if ndim >= 2:
        parts += [("auto", 1, None, None), ("auto", 2, None, None)]
    # interior ROW partition (ghost-cell style)
    if all(s >= 3 for s in shape) and shape[0] - 2 >= 1:
        parts.append(("auto", 0, [1] * ndim, [s - 1 for s in shape]))
    # a manual partition: random disjoint row slabs, some devices empty
    cuts = np.sort(rng.integers(0, shape[0] + 1, size=P - 1)) if P > 1 else np.array([], int)
    bounds = [0] + [int(c) for c in cuts] + [shape[0]]
    perm = rng.permutation(P)
    lbs = np.zeros((P, ndim), np.int64)
    ubs = np.zeros((P, ndim), np.int64)
    for d in range(P):
        k = int(perm[d])
        lbs[d, 0], ubs[d, 0] = bounds[k], bounds[k + 1]
        for j in range(1, ndim):
            lbs[d, j], ubs[d, j] = 0, shape[j]
    parts.append(("manual", None, lbs, ubs))
    ops = []
    n_arr = 2
    for i in range(n_arr):
        ops.append(("write", i, int(rng.integers(len(parts))), int(seed * 7 + i)))
    for k in range(n_ops):
        part = int(rng.integers(len(parts)))
        r = rng.random()
        if r < 0.12:
            ops.append(("write", int(rng.integers(n_arr)), part, int(seed * 31 + k)))
        elif r < 0.22:
            ops.append(("read", int(rng.integers(n_arr)), part))
        else:
            x = int(rng.integers(n_arr))
            y = 1 - x
            uses = []
            for _ in range(int(rng.integers(1, 4))):
                uses.append(tuple(int(v) if rng.random() > 0.15 else STAR for v in rng.integers(-2, 3, size=ndim)))
            acc_y_def = rng.random() < 0.85
            defs = [(0,) * ndim]
            if rng.random() < 0.3:
                defs.append(tuple(int(v) for v in rng.integers(-1, 2, size=ndim)))
            kernel = "stamp" if (with_kernels and acc_y_def) else "none"
            ops.append(("apply", kernel, part, x, uses, y, defs if acc_y_def else [], int(seed * 131 + k)))
    return dict(shape=shape, ndim=ndim, dtype=dtype, P=P, parts=parts, ops=ops, n_arr=n_arr)


def run_program(prog, backend, on_step=None):
    """backend: object with create/partition/partition_manual/apply/write/read/msgs API
    (oracle.Oracle or an adapter of HDArray).  Returns list of per-op results."""
    shape, dt = prog["shape"], prog["dtype"]
    arrs = [backend.create(dt, shape) for _ in range(prog["n_arr"])]
    parts = []
    for kind, k, lb, ub in prog["parts"]:
        if kind == "auto":
            parts.append(backend.partition(k, shape, lb, ub))
        else:
            parts.append(backend.partition_manual(shape, lb, ub))
    npdt = {0: np.float64, 1: np.float32, 2: np.uint16, 4: np.int64}[dt]
    for step, op in enumerate(prog["ops"]):
        status = 0
        if op[0] == "write":
            _, a, p, seed = op
            data = synth.random_bits(seed, shape, {0: "f64", 1: "f32", 2: "bf16", 4: "i64"}[dt]).astype(npdt, copy=False)
            backend.write(arrs[a], parts[p], data)
        elif op[0] == "read":
            _, a, p = op
            backend.read(arrs[a], parts[p])
        else:
            _, kernel, p, x, uses, y, ydefs, seed = op
            acc = [(arrs[y], [], ydefs), (arrs[x], uses, [])] if kernel == "stamp" else \
                [(arrs[x], uses, []), (arrs[y], [], ydefs)]
            kid = 7 if kernel == "stamp" else 0
            if kernel == "stamp" and not ydefs:
                kid = 0
            try:
                backend.apply(kid, parts[p], acc, [float(seed)] if kid == 7 else [])
            except Exception as e:  # validation errors must agree between backends
                status = getattr(e, "code", -999)
        if on_step:
            on_step(step, op, arrs, status)
    return arrs


class LibAdapter:
    """HDArray with the oracle's method names and message format."""

    def __init__(self, h):
        self.h = h

    def create(self, dt, shape):
        return self.h.create(dt, shape)

    def partition(self, kind, shape, lb, ub):
        return self.h.partition(kind, shape, lb, ub)

    def partition_manual(self, shape, lbs, ubs):
        return self.h.partition_manual(shape, lbs, ubs)

    def apply(self, k, part, acc, scalars):
        return self.h.apply(k, part, acc, scalars)

    def write(self, a, part, data):
        if self.h.plan_only:
            return self.h.write(a, part, None)
        return self.h.write(a, part, data)

    def read(self, a, part):
        if self.h.plan_only:
            return self.h.L.hda_read(self.h.h, a, part, None)
        return self.h.read(a, part)

    def msgs(self):
        """(n,4) int64 (array, src, dst, linear index) sorted, like oracle.msgs()."""
        rows = []
        for a, s, d, lb, ub in self.h.last_plan():
            shp = self.h.shapes[a]
            idx = np.ravel_multi_index(np.meshgrid(*[np.arange(l, u) for l, u in zip(lb, ub)], indexing="ij"),
                                       shp).reshape(-1)
            rows.append(np.stack([np.full_like(idx, a), np.full_like(idx, s), np.full_like(idx, d), idx], 1))
        if not rows:
            return np.zeros((0, 4), np.int64)
        m = np.concatenate(rows).astype(np.int64)
        order = np.lexsort((m[:, 3], m[:, 2], m[:, 1], m[:, 0]))
        return m[order]
