"""Error behaviour of the C-ABI as include/hdarray.h states it (plan-only contexts, so
no GPU): negative codes, a message from hda_last_error, and validation errors that
leave the context's state untouched (SPEC-style "the call has no effect")."""
import ctypes

import numpy as np
import pytest

import oracle as O
from programs import LibAdapter

import paper_1809_05657_b200 as H

J = [(0, -1), (0, 1), (-1, 0), (1, 0)]


@pytest.fixture
def h():
    ctx = H.HDArray(n_gpus=0, n_devices=4)
    yield ctx
    ctx.close()


def test_init_rejects_bad_device_counts():
    L = H.lib()
    out = ctypes.c_void_p()
    assert L.hda_init(ctypes.byref(out), 0, None, 0) == H.EINVAL          # P < 1
    assert L.hda_init(ctypes.byref(out), 0, None, 65) == H.EINVAL         # P > 64
    assert L.hda_init(ctypes.byref(out), 2, None, 1) == H.EINVAL          # n_gpus > P
    assert L.hda_init_spmd(ctypes.byref(out), 4, 4, -1) == H.EINVAL       # rank out of range
    assert L.hda_init(None, 0, None, 2) == H.EINVAL                      # null out


def test_null_context_and_null_arguments(h):
    L = H.lib()
    assert L.hda_sync(None) == H.EINVAL
    assert L.hda_finalize(None) == H.EINVAL
    a = ctypes.c_int32()
    shape = (ctypes.c_int64 * 2)(8, 8)
    assert L.hda_create(h.h, H.F64, 2, None, None, ctypes.byref(a)) == H.EINVAL
    assert L.hda_create(h.h, H.F64, 2, shape, None, None) == H.EINVAL
    assert b"null" in L.hda_last_error(h.h)


def test_unknown_handles_and_kernels(h):
    X = h.create(H.F64, (8, 8))
    p = h.partition(H.ROW, (8, 8))
    for bad in (lambda: h.apply(99, p, [(X, [], [(0, 0)])]),                 # unknown kernel
                lambda: h.apply(H.K_NONE, 1234, [(X, [], [(0, 0)])])):        # unknown partition
        with pytest.raises(H.HDAError) as e:
            bad()
        assert e.value.code == H.EINVAL, e.value
    L = H.lib()
    # unknown array handles straight through the C-ABI (the binding checks them itself)
    d = (ctypes.c_int32 * 2)(0, 0)
    acc = (H.hda_access_t * 1)()
    acc[0].array, acc[0].n_use, acc[0].n_def = 777, 0, 1
    acc[0].def_ = ctypes.cast(d, ctypes.POINTER(ctypes.c_int32))
    assert L.hda_apply(h.h, H.K_NONE, p, acc, 1, None, 0) == H.EINVAL
    assert L.hda_read(h.h, 777, p, None) == H.EINVAL
    assert L.hda_free(h.h, 777) == H.EINVAL
    assert b"unknown array" in L.hda_last_error(h.h)
    assert L.hda_set_transport(h.h, 7) == H.EINVAL


def test_partition_out_of_domain_is_erange(h):
    with pytest.raises(H.HDAError) as e:
        h.partition(H.ROW, (8, 8), (0, 0), (9, 8))
    assert e.value.code == H.ERANGE
    with pytest.raises(H.HDAError) as e:
        h.partition_manual((8, 8), [[0, 0], [2, 0], [4, 0], [6, 0]], [[2, 8], [4, 8], [6, 8], [8, 9]])
    assert e.value.code == H.ERANGE


def test_reduce_needs_data(h):
    X = h.create(H.F64, (8, 8))
    p = h.partition(H.ROW, (8, 8))
    with pytest.raises(H.HDAError) as e:
        h.reduce(X, p, H.SUM)
    assert e.value.code == H.ESTATE


def test_rejected_calls_leave_no_trace():
    """A rejected call (race, bad footprint) changes nothing: the following program
    plans exactly the oracle's messages for the program without the rejected calls."""
    n, P = 12, 4
    h = H.HDArray(n_gpus=0, n_devices=P)
    w = O.Oracle(P, with_data=False)
    arrs = {}
    for be in (h, w):
        A, B = be.create(H.F64, (n, n)), be.create(H.F64, (n, n))
        data = be.partition(H.ROW, (n, n))
        work = be.partition(H.ROW, (n, n), (1, 1), (n - 1, n - 1))
        be.write(A, data, None)
        be.write(B, data, None)
        arrs[be] = (A, B, data, work)
    A, B, data, work = arrs[h]
    for bad in ([(A, [], [(0, 0), (1, 0)])],                          # two devices define one cell
                [(A, [], [(0, 0)]), (B, [(0, 1)], [])]):              # JACOBI5 footprint not declared
        with pytest.raises(H.HDAError):
            h.apply(H.K_JACOBI5 if len(bad) == 2 else H.K_NONE, work, bad)
    Aw, Bw, _, workw = arrs[w]
    for s in range(3):
        h.apply(H.K_JACOBI5, work, [(A, [], [(0, 0)]), (B, J, [])])
        w.apply(O.K_JACOBI5, workw, [(Aw, [], [(0, 0)]), (Bw, J, [])])
        got, ref = O.msgs_by_pair(LibAdapter(h).msgs()), O.msgs_by_pair(w.msgs())
        assert got.keys() == ref.keys()
        for k in ref:
            np.testing.assert_array_equal(got[k], ref[k])
        h.apply(H.K_COPY, work, [(B, [], [(0, 0)]), (A, [(0, 0)], [])])
        w.apply(O.K_COPY, workw, [(Bw, [], [(0, 0)]), (Aw, [(0, 0)], [])])
    np.testing.assert_array_equal(h.owner_map(A), w.owner_map(Aw))
    np.testing.assert_array_equal(h.owner_map(B), w.owner_map(Bw))
    h.close()


def test_scalar_count_checked_on_cache_hits(h):
    """The per-kernel scalar minimum holds on every call, not only the first: a valid
    SCALE / GEMM call caches its spec, and the same call with too few scalars is still
    EINVAL (the GPU path would otherwise read scalars[0] / scalars[1] past the array)."""
    X = h.create(H.F64, (8, 8))
    p = h.partition(H.ROW, (8, 8))
    acc = [(X, [(0, 0)], [(0, 0)])]
    h.apply(H.K_SCALE, p, acc, (2.0,))
    for bad in ((), ):
        with pytest.raises(H.HDAError) as e:
            h.apply(H.K_SCALE, p, acc, bad)
        assert e.value.code == H.EINVAL and "scalars" in str(e.value)
    A, B, C = (h.create(H.BF16, (8, 8)) for _ in range(3))
    g = [(C, [], [(0, 0)]), (A, [(0, H.STAR)], []), (B, [(H.STAR, 0)], [])]
    h.apply(H.K_GEMM, p, g, (1.0, 0.0))
    for bad in ((), (1.0,)):
        with pytest.raises(H.HDAError) as e:
            h.apply(H.K_GEMM, p, g, bad)
        assert e.value.code == H.EINVAL
    h.apply(H.K_SCALE, p, acc, (2.0,))  # the context is still usable
