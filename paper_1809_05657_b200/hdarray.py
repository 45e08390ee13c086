"""Thin ctypes binding of libhdarray.so (include/hdarray.h).

Argument marshalling only: every step of the path (tracking, planning, packing,
transfers, kernels) runs inside the C++/CUDA library.  Function names are the
C-ABI names; ``HDArray`` is a small convenience object over them.  There is no
fallback: if the library is missing this module raises at import.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import build as _build

STAR = -(2**31)
F64, F32, BF16, I32, I64 = 0, 1, 2, 3, 4
ROW, COL, BLOCK = 0, 1, 2
(K_NONE, K_JACOBI5, K_COPY, K_STENCIL9, K_STENCIL7_3D, K_SCALE, K_GEMM, K_STAMP) = range(8)
XPORT_FUSED, XPORT_STAGED, XPORT_AUTO = 0, 1, 2
SUM, PROD, MAX, MIN = 0, 1, 2, 3
OK, EINVAL, ERANGE, EOVERLAP, ERACE, ENOMEM, ECUDA, ETIMEOUT, EUNSUPPORTED, ESTATE = (
    0, -1, -2, -3, -4, -5, -6, -7, -8, -9)
HANDLE_BYTES = 128
NP_DTYPE = {F64: np.float64, F32: np.float32, BF16: np.uint16, I32: np.int32, I64: np.int64}
ELEM = {F64: 8, F32: 4, BF16: 2, I32: 4, I64: 8}


class hda_access_t(ctypes.Structure):
    _fields_ = [("array", ctypes.c_int32), ("n_use", ctypes.c_int32), ("use", ctypes.POINTER(ctypes.c_int32)),
                ("n_def", ctypes.c_int32), ("def_", ctypes.POINTER(ctypes.c_int32))]


class hda_abs_access_t(ctypes.Structure):
    _fields_ = [("array", ctypes.c_int32), ("n_use", ctypes.POINTER(ctypes.c_int32)),
                ("use", ctypes.POINTER(ctypes.c_int64)), ("n_def", ctypes.POINTER(ctypes.c_int32)),
                ("def_", ctypes.POINTER(ctypes.c_int64))]


class hda_msg_t(ctypes.Structure):
    _fields_ = [("array", ctypes.c_int32), ("src", ctypes.c_int32), ("dst", ctypes.c_int32),
                ("ndim", ctypes.c_int32), ("lb", ctypes.c_int64 * 3), ("ub", ctypes.c_int64 * 3)]


class hda_stats_t(ctypes.Structure):
    _fields_ = [("n_apply", ctypes.c_int64), ("plan_hits", ctypes.c_int64), ("plan_misses", ctypes.c_int64),
                ("msgs_total", ctypes.c_int64), ("bytes_total", ctypes.c_int64), ("last_msgs", ctypes.c_int64),
                ("last_bytes", ctypes.c_int64), ("kernel_launches", ctypes.c_int64), ("tracker_us", ctypes.c_double),
                ("gated_products", ctypes.c_int64)]


EXPORTS = [
    "hda_init", "hda_init_spmd", "hda_finalize", "hda_num_devices", "hda_is_local", "hda_spmd_export",
    "hda_spmd_import", "hda_create", "hda_create_ext", "hda_free", "hda_device_ptr", "hda_partition",
    "hda_partition_manual", "hda_partition_region", "hda_apply", "hda_apply_abs", "hda_trapezoid", "hda_sync", "hda_write", "hda_read", "hda_reduce",
    "hda_set_transport", "hda_set_overlap", "hda_set_plan_cache", "hda_set_kernel_timing", "hda_kernel_time", "hda_exchange_time",
    "hda_stream", "hda_set_trace", "hda_trace", "hda_last_plan", "hda_owner_map", "hda_read_replica", "hda_stats", "hda_reset_stats",
    "hda_last_error", "hda_version",
]

_lib = None
LIB_PATH = _build.LIB


def lib():
    """Load libhdarray.so (building it in-tree with nvcc if stale)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH) or os.environ.get("HDA_AUTOBUILD", "1") == "1":
            _build.build()
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        P = ctypes.POINTER
        sig = {
            "hda_init": [P(vp), i32, P(i32), i32],
            "hda_init_spmd": [P(vp), i32, i32, i32],
            "hda_finalize": [vp],
            "hda_num_devices": [vp, P(i32)],
            "hda_is_local": [vp, i32, P(i32)],
            "hda_spmd_export": [vp, i32, vp],
            "hda_spmd_import": [vp, i32, vp],
            "hda_create": [vp, i32, i32, P(i64), vp, P(i32)],
            "hda_create_ext": [vp, i32, i32, P(i64), P(vp), P(i32)],
            "hda_free": [vp, i32],
            "hda_device_ptr": [vp, i32, i32, P(vp)],
            "hda_partition": [vp, i32, i32, P(i64), P(i64), P(i64), P(i32)],
            "hda_partition_manual": [vp, i32, P(i64), P(i64), P(i64), P(i32)],
            "hda_partition_region": [vp, i32, i32, P(i64), P(i64)],
            "hda_apply": [vp, i32, i32, P(hda_access_t), i32, P(ctypes.c_double), i32],
            "hda_sync": [vp],
            "hda_apply_abs": [vp, i32, i32, P(hda_abs_access_t), i32, P(ctypes.c_double), i32],
            "hda_trapezoid": [P(i64), P(i64), i32, P(i32)],
            "hda_write": [vp, i32, i32, vp],
            "hda_read": [vp, i32, i32, vp],
            "hda_reduce": [vp, i32, i32, i32, P(ctypes.c_double)],
            "hda_set_transport": [vp, i32],
            "hda_set_plan_cache": [vp, i32],
            "hda_set_overlap": [vp, i32],
            "hda_set_kernel_timing": [vp, i32],
            "hda_kernel_time": [vp, i32, P(ctypes.c_double), P(i64)],
            "hda_exchange_time": [vp, P(ctypes.c_double), P(i64)],
            "hda_stream": [vp, i32, P(vp)],
            "hda_set_trace": [vp, i32],
            "hda_trace": [vp, P(ctypes.c_double), i32, P(i32)],
            "hda_last_plan": [vp, P(hda_msg_t), i32, P(i32)],
            "hda_owner_map": [vp, i32, vp],
            "hda_read_replica": [vp, i32, i32, vp],
            "hda_stats": [vp, P(hda_stats_t)],
            "hda_reset_stats": [vp],
            "hda_last_error": [vp],
            "hda_version": [],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        L.hda_last_error.restype = ctypes.c_char_p
        L.hda_version.restype = ctypes.c_char_p
        _lib = L
    return _lib


class HDAError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"hdarray error {code}: {msg}")
        self.code = code


def _i64(v):
    a = np.ascontiguousarray(v, dtype=np.int64)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def _tuples(ts, nd):
    flat = [int(x) for t in ts for x in t]
    assert all(len(t) == nd for t in ts), "offset arity must equal the array rank"
    arr = (ctypes.c_int32 * max(len(flat), 1))(*flat)
    return arr


class HDArray:
    """One runtime context (hda_ctx_t*) and convenience wrappers of every call."""

    def __init__(self, n_gpus: int = 1, n_devices: int | None = None, gpu_ids=None, _spmd=None):
        self.L = lib()
        self.h = ctypes.c_void_p()
        self.shapes, self.dtypes = {}, {}
        self.group = None
        if _spmd is None:
            P = n_devices if n_devices is not None else max(n_gpus, 1)
            ids = None if gpu_ids is None else (ctypes.c_int32 * len(gpu_ids))(*gpu_ids)
            rc = self.L.hda_init(ctypes.byref(self.h), n_gpus, ids, P)
            self.spmd = False
            self.rank = None
        else:
            P, rank, gpu_id, group = _spmd
            rc = self.L.hda_init_spmd(ctypes.byref(self.h), P, rank, gpu_id)
            self.spmd = True
            self.rank = rank
            self.group = group
        self.P = P
        self.plan_only = (n_gpus == 0) if _spmd is None else (_spmd[2] < 0)
        self._chk(rc)
        if self.spmd and not self.plan_only and P > 1:
            self._swap(-1)

    @classmethod
    def spmd(cls, n_devices: int, rank: int, gpu_id: int, group=None):
        """The paper's SPMD model: this process is device `rank`."""
        return cls(_spmd=(n_devices, rank, gpu_id, group))

    def _swap(self, arr):
        import torch.distributed as dist
        blob = (ctypes.c_char * HANDLE_BYTES)()
        self._chk(self.L.hda_spmd_export(self.h, arr, blob))
        mine = bytes(blob)
        allb = [None] * self.P
        dist.all_gather_object(allb, mine, group=self.group)
        buf = (ctypes.c_char * (HANDLE_BYTES * self.P)).from_buffer_copy(b"".join(allb))
        self._chk(self.L.hda_spmd_import(self.h, arr, buf))

    def close(self):
        if self.h:
            self.L.hda_finalize(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, rc):
        if rc != OK:
            msg = self.L.hda_last_error(self.h).decode() if self.h else ""
            raise HDAError(rc, msg)
        return rc

    # ---- arrays / partitions
    def create(self, dtype, shape, init=None):
        shp, sp = _i64(shape)
        buf = None
        if init is not None:
            buf = np.ascontiguousarray(init, dtype=NP_DTYPE[dtype]).reshape(-1)
            assert buf.size == int(np.prod(shape))
        out = ctypes.c_int32()
        self._chk(self.L.hda_create(self.h, dtype, len(shape), sp, buf.ctypes.data if buf is not None else None,
                                    ctypes.byref(out)))
        a = out.value
        self.shapes[a] = tuple(int(s) for s in shape)
        self.dtypes[a] = dtype
        if self.spmd and not self.plan_only and self.P > 1:
            self._swap(a)
        return a

    def free(self, a):
        self._chk(self.L.hda_free(self.h, a))

    def partition(self, kind, domain, lb=None, ub=None):
        nd = len(domain)
        d, dp = _i64(domain)
        l, lp = _i64([0] * nd if lb is None else lb)
        u, up = _i64(list(domain) if ub is None else ub)
        out = ctypes.c_int32()
        self._chk(self.L.hda_partition(self.h, kind, nd, dp, lp, up, ctypes.byref(out)))
        return out.value

    def partition_manual(self, domain, lbs, ubs):
        nd = len(domain)
        d, dp = _i64(domain)
        l, lp = _i64(np.asarray(lbs).reshape(-1))
        u, up = _i64(np.asarray(ubs).reshape(-1))
        out = ctypes.c_int32()
        self._chk(self.L.hda_partition_manual(self.h, nd, dp, lp, up, ctypes.byref(out)))
        return out.value

    def region(self, part, dev, ndim):
        lb = (ctypes.c_int64 * 3)()
        ub = (ctypes.c_int64 * 3)()
        self._chk(self.L.hda_partition_region(self.h, part, dev, lb, ub))
        return tuple(lb[:ndim]), tuple(ub[:ndim])

    # ---- hot path
    def apply(self, kernel, part, acc, scalars=()):
        """acc: list of (array, use_tuples, def_tuples) in kernel-parameter order."""
        n = len(acc)
        entries = (hda_access_t * max(n, 1))()
        keep = []
        for i, (a, uses, defs) in enumerate(acc):
            nd = len(self.shapes[a])
            u = _tuples(uses, nd)
            d = _tuples(defs, nd)
            keep += [u, d]
            entries[i].array = a
            entries[i].n_use = len(uses)
            entries[i].use = ctypes.cast(u, ctypes.POINTER(ctypes.c_int32))
            entries[i].n_def = len(defs)
            entries[i].def_ = ctypes.cast(d, ctypes.POINTER(ctypes.c_int32))
        sc = (ctypes.c_double * max(len(scalars), 1))(*[float(s) for s in scalars])
        self._chk(self.L.hda_apply(self.h, kernel, part, entries, n, sc, len(scalars)))

    def apply_abs(self, kernel, part, acc, scalars=()):
        """acc: list of (array, uses, defs); uses/defs: per device a list of boxes
        ((lb...), (ub...)) — absolute sections (Table 1 use@/def@)."""
        n = len(acc)
        entries = (hda_abs_access_t * n)()
        keep = []
        for i, (a, uses, defs) in enumerate(acc):
            for fld_n, fld_b, lists in (("n_use", "use", uses), ("n_def", "def_", defs)):
                cnt = (ctypes.c_int32 * self.P)(*[len(lists[q]) for q in range(self.P)])
                flat = [int(v) for q in range(self.P) for lb, ub in lists[q] for v in list(lb) + list(ub)]
                arr = (ctypes.c_int64 * max(len(flat), 1))(*flat)
                keep += [cnt, arr]
                setattr(entries[i], fld_n, ctypes.cast(cnt, ctypes.POINTER(ctypes.c_int32)))
                setattr(entries[i], fld_b, ctypes.cast(arr, ctypes.POINTER(ctypes.c_int64)))
            entries[i].array = a
        sc = (ctypes.c_double * max(len(scalars), 1))(*[float(s) for s in scalars])
        self._chk(self.L.hda_apply_abs(self.h, kernel, part, entries, n, sc, len(scalars)))

    def prepare(self, kernel, part, acc, scalars=()):
        """Marshal an hda_apply call once; the returned callable re-issues it with no
        Python-side re-marshalling (steady-state loops)."""
        n = len(acc)
        entries = (hda_access_t * max(n, 1))()
        keep = []
        for i, (a, uses, defs) in enumerate(acc):
            nd = len(self.shapes[a])
            u = _tuples(uses, nd)
            d = _tuples(defs, nd)
            keep += [u, d]
            entries[i].array = a
            entries[i].n_use = len(uses)
            entries[i].use = ctypes.cast(u, ctypes.POINTER(ctypes.c_int32))
            entries[i].n_def = len(defs)
            entries[i].def_ = ctypes.cast(d, ctypes.POINTER(ctypes.c_int32))
        sc = (ctypes.c_double * max(len(scalars), 1))(*[float(s) for s in scalars])
        fn, h, ns = self.L.hda_apply, self.h, len(scalars)

        def run():
            rc = fn(h, kernel, part, entries, n, sc, ns)
            if rc:
                self._chk(rc)

        run._keep = (entries, keep, sc)
        return run

    def sync(self):
        self._chk(self.L.hda_sync(self.h))

    def write(self, a, part, host):
        if host is None:
            self._chk(self.L.hda_write(self.h, a, part, None))
            return
        buf = np.ascontiguousarray(host, dtype=NP_DTYPE[self.dtypes[a]]).reshape(-1)
        assert buf.size == int(np.prod(self.shapes[a]))
        self._chk(self.L.hda_write(self.h, a, part, buf.ctypes.data))

    def write_ptr(self, a, part, host_ptr: int):
        """write from a raw host pointer (e.g. pinned torch tensor), global layout."""
        self._chk(self.L.hda_write(self.h, a, part, ctypes.c_void_p(host_ptr)))

    def read(self, a, part, out=None):
        if out is None:
            out = np.zeros(self.shapes[a], dtype=NP_DTYPE[self.dtypes[a]])
        self._chk(self.L.hda_read(self.h, a, part, out.ctypes.data))
        return out

    def reduce(self, a, part, op):
        out = ctypes.c_double()
        self._chk(self.L.hda_reduce(self.h, a, part, op, ctypes.byref(out)))
        return out.value

    def read_ptr(self, a, part, host_ptr: int):
        self._chk(self.L.hda_read(self.h, a, part, ctypes.c_void_p(host_ptr)))

    # ---- tuning / timing
    def set_transport(self, t):
        self._chk(self.L.hda_set_transport(self.h, t))

    def set_overlap(self, on):
        self._chk(self.L.hda_set_overlap(self.h, 1 if on else 0))

    def set_plan_cache(self, on):
        self._chk(self.L.hda_set_plan_cache(self.h, 1 if on else 0))

    def set_kernel_timing(self, on):
        self._chk(self.L.hda_set_kernel_timing(self.h, 1 if on else 0))

    def kernel_time(self, kernel):
        ms = ctypes.c_double()
        n = ctypes.c_int64()
        self._chk(self.L.hda_kernel_time(self.h, kernel, ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    def exchange_time(self):
        ms = ctypes.c_double()
        n = ctypes.c_int64()
        self._chk(self.L.hda_exchange_time(self.h, ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    def set_trace(self, on):
        self._chk(self.L.hda_set_trace(self.h, 1 if on else 0))

    def trace(self):
        """rows (epoch, device, phase, start_us, end_us); phase 0 exchange, 1 kernel,
        2 interior, 3 dependent."""
        n = ctypes.c_int32()
        self._chk(self.L.hda_trace(self.h, None, 0, ctypes.byref(n)))
        out = (ctypes.c_double * max(5 * n.value, 5))()
        self._chk(self.L.hda_trace(self.h, out, n.value, ctypes.byref(n)))
        return np.array(out[:5 * n.value]).reshape(-1, 5)

    def stream(self, dev):
        s = ctypes.c_void_p()
        self._chk(self.L.hda_stream(self.h, dev, ctypes.byref(s)))
        return s.value

    def device_ptr(self, a, dev):
        p = ctypes.c_void_p()
        self._chk(self.L.hda_device_ptr(self.h, a, dev, ctypes.byref(p)))
        return p.value

    # ---- introspection
    def last_plan(self):
        n = ctypes.c_int32()
        self._chk(self.L.hda_last_plan(self.h, None, 0, ctypes.byref(n)))
        buf = (hda_msg_t * max(n.value, 1))()
        self._chk(self.L.hda_last_plan(self.h, buf, n.value, ctypes.byref(n)))
        return [(m.array, m.src, m.dst, tuple(m.lb[:m.ndim]), tuple(m.ub[:m.ndim])) for m in buf[:n.value]]

    def owner_map(self, a):
        out = np.zeros(self.shapes[a], np.int8)
        self._chk(self.L.hda_owner_map(self.h, a, out.ctypes.data))
        return out

    def read_replica(self, a, dev):
        out = np.zeros(self.shapes[a], NP_DTYPE[self.dtypes[a]])
        self._chk(self.L.hda_read_replica(self.h, a, dev, out.ctypes.data))
        return out

    def stats(self):
        s = hda_stats_t()
        self._chk(self.L.hda_stats(self.h, ctypes.byref(s)))
        return {k: getattr(s, k) for k, _ in hda_stats_t._fields_}

    def reset_stats(self):
        self._chk(self.L.hda_reset_stats(self.h))


def trapezoid(corners):
    """per-row 2-D boxes of a trapezoid, corners [(top,ul),(top,ur),(bottom,bl),(bottom,br)]."""
    L = lib()
    c = (ctypes.c_int64 * 8)(*[int(x) for cc in corners for x in cc])
    n = ctypes.c_int32()
    rc = L.hda_trapezoid(c, None, 0, ctypes.byref(n))
    if rc:
        raise HDAError(rc, "bad trapezoid corners")
    out = (ctypes.c_int64 * max(4 * n.value, 4))()
    L.hda_trapezoid(c, out, n.value, ctypes.byref(n))
    return [((out[4 * i], out[4 * i + 1]), (out[4 * i + 2], out[4 * i + 3])) for i in range(n.value)]


def plan_cells(plan, shapes):
    """expand a plan into {(array, src, dst): sorted linear indices} (for parity)."""
    out = {}
    for a, s, d, lb, ub in plan:
        shp = shapes[a]
        idx = np.ravel_multi_index(np.meshgrid(*[np.arange(l, u) for l, u in zip(lb, ub)], indexing="ij"), shp)
        out.setdefault((a, s, d), []).append(idx.reshape(-1))
    return {k: np.sort(np.concatenate(v)) for k, v in out.items()}
