"""CPU oracle of the HDArray def/use exchange path (arXiv:1809.05657).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline legs (``cpu_baseline`` and ``--impl reference``) may
import this package.  The product library (``paper_1809_05657_b200``) never imports
it, and the two share no code: this wrapper loads ``oracle/liboracle.so`` built
from ``hda_oracle.c`` (plain C, per-element last-writer maps, brute force).

Parity status of each oracle function:
  messages / owner maps (orc_apply, orc_read, orc_write)  pinned: P3 worked example,
      P4 invariants, P5 GEMM all-gather, P9 closed-form volumes (tests/test_oracle_pins.py)
  JACOBI5 / STENCIL9 / STENCIL7_3D                         pinned: eigenmode closed form
      (P6) and harmonic fixed points (P7)
  COPY / SCALE / STAMP                                      pinned: identity, exact scaling,
      splitmix64 published test vector
  GEMM (orc_apply, orc_gemm_sample)                         pinned: integer case vs exact
      int64 numpy matmul (P7)
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

STAR = -(2**31)
F64, F32, BF16, I32, I64 = 0, 1, 2, 3, 4
ROW, COL, BLOCK = 0, 1, 2
K_NONE, K_JACOBI5, K_COPY, K_STENCIL9, K_STENCIL7_3D, K_SCALE, K_GEMM, K_STAMP = range(8)
OK, EINVAL, ERANGE, EOVERLAP, ERACE, ENOMEM = 0, -1, -2, -3, -4, -5
SUM, PROD, MAX, MIN = 0, 1, 2, 3
EUNSUPPORTED, ESTALE = -8, -10

NP_DTYPE = {F64: np.float64, F32: np.float32, BF16: np.uint16, I32: np.int32, I64: np.int64}


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no FP contraction, no fast-math)."""
    src = os.path.join(_HERE, "hda_oracle.c")
    hdr = os.path.join(_HERE, "hda_oracle.h")
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= max(os.path.getmtime(src), os.path.getmtime(hdr))):
        return _LIB_PATH
    tmp = _LIB_PATH + f".tmp{os.getpid()}"
    cmd = ["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
           "-Wall", "-Wextra", "-Wno-unused-parameter", "-o", tmp, src, "-lm"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        i64p = ctypes.POINTER(ctypes.c_int64)
        i32p = ctypes.POINTER(ctypes.c_int32)
        L.orc_new.restype = ctypes.c_void_p
        L.orc_new.argtypes = [ctypes.c_int, ctypes.c_int]
        L.orc_free.argtypes = [ctypes.c_void_p]
        L.orc_error.restype = ctypes.c_char_p
        L.orc_error.argtypes = [ctypes.c_void_p]
        L.orc_create.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, i64p, ctypes.c_void_p]
        L.orc_partition.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, i64p, i64p, i64p]
        L.orc_partition_manual.argtypes = [ctypes.c_void_p, ctypes.c_int, i64p, i64p, i64p]
        L.orc_region.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, i64p, i64p]
        L.orc_apply.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, i32p, i32p,
                                i32p, i32p, i32p, ctypes.POINTER(ctypes.c_double), ctypes.c_int]
        L.orc_write.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        L.orc_read.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        L.orc_apply_abs.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, i32p, i32p, i64p,
                                    i32p, i64p, ctypes.POINTER(ctypes.c_double), ctypes.c_int]
        L.orc_trapezoid.argtypes = [i64p, i64p, ctypes.c_int]
        L.orc_reduce.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                 ctypes.POINTER(ctypes.c_double)]
        L.orc_msg_count.restype = ctypes.c_int64
        L.orc_msg_count.argtypes = [ctypes.c_void_p]
        L.orc_msgs.restype = ctypes.c_int64
        L.orc_msgs.argtypes = [ctypes.c_void_p, i64p, ctypes.c_int64]
        L.orc_owner_map.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
        L.orc_valid_map.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
        L.orc_replica.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        L.orc_gemm_sample.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                      i64p, i64p, ctypes.c_int64, ctypes.c_void_p]
        L.orc_splitmix64.restype = ctypes.c_uint64
        L.orc_splitmix64.argtypes = [ctypes.c_uint64]
        L.orc_f32_to_bf16.restype = ctypes.c_uint16
        L.orc_f32_to_bf16.argtypes = [ctypes.c_float]
        L.orc_f64_to_bf16.restype = ctypes.c_uint16
        L.orc_f64_to_bf16.argtypes = [ctypes.c_double]
        _lib = L
    return _lib


def _i64(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def _i32(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


class Oracle:
    """P simulated devices with full-size replicas in one address space."""

    def __init__(self, P: int, with_data: bool = True):
        self.L = lib()
        self.P = P
        self.h = self.L.orc_new(P, 1 if with_data else 0)
        if not self.h:
            raise OracleError(EINVAL, "orc_new failed")
        self.shapes = {}
        self.dtypes = {}

    def close(self):
        if self.h:
            self.L.orc_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, rc):
        if rc < 0:
            raise OracleError(rc, self.L.orc_error(self.h).decode())
        return rc

    def create(self, dtype, shape, init=None):
        shp, p = _i64(shape)
        buf = None
        if init is not None:
            buf = np.ascontiguousarray(init, dtype=NP_DTYPE[dtype]).reshape(-1)
            assert buf.size == int(np.prod(shape))
        a = self._chk(self.L.orc_create(self.h, dtype, len(shape), p,
                                        buf.ctypes.data if buf is not None else None))
        self.shapes[a] = tuple(int(s) for s in shape)
        self.dtypes[a] = dtype
        return a

    def partition(self, kind, domain, lb=None, ub=None):
        nd = len(domain)
        lb = [0] * nd if lb is None else lb
        ub = list(domain) if ub is None else ub
        d, dp = _i64(domain)
        l, lp = _i64(lb)
        u, up = _i64(ub)
        return self._chk(self.L.orc_partition(self.h, kind, nd, dp, lp, up))

    def partition_manual(self, domain, lbs, ubs):
        nd = len(domain)
        d, dp = _i64(domain)
        l, lp = _i64(np.asarray(lbs).reshape(-1))
        u, up = _i64(np.asarray(ubs).reshape(-1))
        return self._chk(self.L.orc_partition_manual(self.h, nd, dp, lp, up))

    def region(self, part, dev, ndim):
        lb = np.zeros(ndim, np.int64)
        ub = np.zeros(ndim, np.int64)
        self._chk(self.L.orc_region(self.h, part, dev, lb.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                    ub.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
        return tuple(lb), tuple(ub)

    def apply(self, kernel, part, acc, scalars=()):
        """acc: list of (array, uses, defs), uses/defs lists of offset tuples."""
        arrays = [a for a, _, _ in acc]
        n_use = [len(u) for _, u, _ in acc]
        n_def = [len(d) for _, _, d in acc]
        uses = [x for _, u, _ in acc for t in u for x in t] or [0]
        defs = [x for _, _, d in acc for t in d for x in t] or [0]
        a, ap = _i32(arrays or [0])
        nu, nup = _i32(n_use or [0])
        nd, ndp = _i32(n_def or [0])
        us, usp = _i32(uses)
        ds, dsp = _i32(defs)
        sc = np.ascontiguousarray(list(scalars) or [0.0], dtype=np.float64)
        return self._chk(self.L.orc_apply(self.h, kernel, part, len(acc), ap, nup, usp, ndp, dsp,
                                          sc.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                          len(scalars)))

    def apply_abs(self, kernel, part, acc, scalars=()):
        """acc: list of (array, uses, defs); uses/defs: per device a list of boxes
        ((lb...), (ub...)) (absolute sections, Table 1 use@/def@)."""
        P = self.P
        arrays = [a for a, _, _ in acc]
        n_use, n_def, ub, db = [], [], [], []
        for a, uses, defs in acc:
            for q in range(P):
                n_use.append(len(uses[q]))
                n_def.append(len(defs[q]))
                for lb_, ub_ in uses[q]:
                    ub += list(lb_) + list(ub_)
                for lb_, ub_ in defs[q]:
                    db += list(lb_) + list(ub_)
        a, ap = _i32(arrays)
        nu, nup = _i32(n_use)
        nd, ndp = _i32(n_def)
        u, up = _i64(ub or [0])
        d, dp = _i64(db or [0])
        sc = np.ascontiguousarray(list(scalars) or [0.0], dtype=np.float64)
        return self._chk(self.L.orc_apply_abs(self.h, kernel, part, len(acc), ap, nup, up, ndp, dp,
                                              sc.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(scalars)))

    def write(self, arr, part, host):
        if host is None:  # plan-only worlds carry no data
            return self._chk(self.L.orc_write(self.h, arr, part, None))
        buf = np.ascontiguousarray(host, dtype=NP_DTYPE[self.dtypes[arr]]).reshape(-1)
        return self._chk(self.L.orc_write(self.h, arr, part, buf.ctypes.data))

    def read(self, arr, part, out=None):
        if out is None:
            out = np.zeros(self.shapes[arr], dtype=NP_DTYPE[self.dtypes[arr]])
        self._chk(self.L.orc_read(self.h, arr, part, out.ctypes.data))
        return out

    def reduce(self, arr, part, op):
        out = ctypes.c_double()
        self._chk(self.L.orc_reduce(self.h, arr, part, op, ctypes.byref(out)))
        return out.value

    def msgs(self):
        """(n, 4) int64: (array, src, dst, linear index), sorted."""
        n = self.L.orc_msg_count(self.h)
        out = np.zeros((max(n, 1), 4), np.int64)
        self.L.orc_msgs(self.h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), n)
        return out[:n]

    def owner_map(self, arr):
        out = np.zeros(self.shapes[arr], np.int8)
        self._chk(self.L.orc_owner_map(self.h, arr, out.ctypes.data))
        return out

    def valid_map(self, arr):
        out = np.zeros(self.shapes[arr], np.uint64)
        self._chk(self.L.orc_valid_map(self.h, arr, out.ctypes.data))
        return out

    def replica(self, arr, dev):
        out = np.zeros(self.shapes[arr], NP_DTYPE[self.dtypes[arr]])
        self._chk(self.L.orc_replica(self.h, arr, dev, out.ctypes.data))
        return out


def msgs_by_pair(m):
    """dict (array, src, dst) -> sorted np.int64 array of linear indices."""
    out = {}
    if len(m) == 0:
        return out
    keys = m[:, :3]
    brk = np.nonzero(np.any(keys[1:] != keys[:-1], axis=1))[0] + 1
    starts = np.concatenate([[0], brk])
    ends = np.concatenate([brk, [len(m)]])
    for s, e in zip(starts, ends):
        out[tuple(int(x) for x in m[s, :3])] = m[s:e, 3].copy()
    return out


def gemm_sample(A_bits, B_bits, ii, jj, alpha=1.0, beta=0.0, Cin=None):
    """fp64 sampled C entries of Listing 2 over bf16 (uint16 bit pattern) inputs."""
    L = lib()
    A = np.ascontiguousarray(A_bits, np.uint16)
    B = np.ascontiguousarray(B_bits, np.uint16)
    ni, nk = A.shape
    nk2, nj = B.shape
    assert nk == nk2
    i, ip = _i64(ii)
    j, jp = _i64(jj)
    out = np.zeros(len(i), np.float64)
    C = None if Cin is None else np.ascontiguousarray(Cin, np.float64)
    L.orc_gemm_sample(A.ctypes.data, B.ctypes.data, C.ctypes.data if C is not None else None,
                      ni, nj, nk, alpha, beta, ip, jp, len(i), out.ctypes.data)
    return out


def trapezoid(corners):
    """per-row boxes ((r, l), (r+1, r_+1)) of a trapezoid with inclusive corners
    [(top, ul), (top, ur), (bottom, bl), (bottom, br)]."""
    L = lib()
    k, kp = _i64([x for c in corners for x in c])
    n = L.orc_trapezoid(kp, None, 0)
    out = np.zeros(max(4 * n, 4), np.int64)
    L.orc_trapezoid(kp, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), n)
    return [((int(out[4 * i]), int(out[4 * i + 1])), (int(out[4 * i + 2]), int(out[4 * i + 3]))) for i in range(n)]


def splitmix64(x: int) -> int:
    return int(lib().orc_splitmix64(x))


def f32_to_bf16(f: float) -> int:
    return int(lib().orc_f32_to_bf16(f))


def f64_to_bf16(d: float) -> int:
    return int(lib().orc_f64_to_bf16(d))
