"""`#pragma hdarray` frontend: the paper's listings parse to the clauses
they state, and a program driven through the file-M table produces exactly the message
sets of the same calls written with explicit offsets (oracle, plan-only library)."""
import numpy as np
import pytest

import oracle as O
from programs import LibAdapter

import paper_1809_05657_b200 as H
from paper_1809_05657_b200 import frontend as F

# Listing 3, GEMM device code, verbatim apart from the LaTeX
GEMM_CL = r"""
#pragma hdarray use(A,(0,*)) use(B,(*,0)) def(C,(0,0))
__kernel void gemm(__global float *A, __global float *B, __global float *C,
                   float alph, float beta, int ni, int nj, int nk) {
  int i = get_global_id(1), j = get_global_id(0);
  if ((i < ni) && (j < nj)) {
     C[i * nj + j] *= beta;
     for(int k=0; k < nk; k++)
        C[i*nj+j] += alph * A[i*nk+k] * B[k*nj+j];
  }
}
"""

# Listing 1, manually partitioned Correlation host code
CORR_HOST = r"""
#pragma hdarray partition(part0,        (10240,10240),\
                          dev:0,   (0,3008),(0,10240),\
                          dev:1,(3008,7232),(0,10240))
HDArrayApplyKernel("corr_ker1", part0, ... );
"""

# the paper's Jacobi pair as CUDA-style sources
JACOBI_CU = r"""
#pragma hdarray use(B,(0,-1)) use(B,(0,+1)) use(B,(-1,0)) use(B,(1,0)) \
                def(A,(0,0))
extern "C" __global__ void jacobi_step(double *A, const double *B, int n) { }

#pragma hdarray use(A,(0,0)) def(B,(0,0))
__global__ void copy_back(double *B, const double *A, int n) { }
"""

J = [(0, -1), (0, 1), (-1, 0), (1, 0)]


def test_gemm_listing_clauses():
    fm = F.parse(GEMM_CL)
    k = fm["kernels"]["gemm"]
    assert [p["name"] for p in k["params"]] == ["A", "B", "C", "alph", "beta", "ni", "nj", "nk"]
    assert [p["array"] for p in k["params"]] == [True, True, True, False, False, False, False, False]
    assert k["access"]["A"]["use"] == [(0, "*")] and k["access"]["A"]["def"] == []
    assert k["access"]["B"]["use"] == [("*", 0)]
    assert k["access"]["C"]["def"] == [(0, 0)] and k["access"]["C"]["use"] == []


def test_listing1_partition_start_length():
    """R2: (start, length) tuples tile the 10240 rows exactly."""
    p = F.parse(CORR_HOST)["partitions"]["part0"]
    assert p["domain"] == [10240, 10240]
    assert p["lb"] == [[0, 0], [3008, 0]] and p["ub"] == [[3008, 10240], [10240, 10240]]


def test_file_m_roundtrip(tmp_path):
    fm = F.parse(GEMM_CL + CORR_HOST + JACOBI_CU)
    path = str(tmp_path / "M.json")
    F.write_file_m(fm, path)
    assert F.load_file_m(path) == fm


def test_config1_through_the_frontend_equals_explicit_offsets():
    """The config-1 worked example (tests/golden) driven by HDArrayApplyKernel over
    file M: every message set and owner map equals the oracle's explicit-offset run."""
    n, P = 16, 4
    fm = F.parse(JACOBI_CU)
    h = H.HDArray(n_gpus=0, n_devices=P)
    prog = F.Program(h, fm)
    prog.bind("jacobi_step", H.K_JACOBI5, arrays=["A", "B"])
    prog.bind("copy_back", H.K_COPY, arrays=["B", "A"])
    w = O.Oracle(P, with_data=False)
    arrs = {}
    for be in (h, w):
        A = be.create(H.F64, (n, n))
        B = be.create(H.F64, (n, n))
        data = be.partition(H.ROW, (n, n))
        work = be.partition(H.ROW, (n, n), (1, 1), (n - 1, n - 1))
        be.write(A, data, None)
        be.write(B, data, None)
        arrs[be] = (A, B, data, work)
    A, B, data, work = arrs[h]
    Aw, Bw, _, workw = arrs[w]
    sizes = []
    for s in range(2):
        prog.apply_kernel("jacobi_step", work, A, B, n)
        w.apply(O.K_JACOBI5, workw, [(Aw, [], [(0, 0)]), (Bw, J, [])])
        got, ref = O.msgs_by_pair(LibAdapter(h).msgs()), O.msgs_by_pair(w.msgs())
        assert got.keys() == ref.keys()
        for key in ref:
            np.testing.assert_array_equal(got[key], ref[key])
        sizes.append(sum(len(v) for v in ref.values()))
        prog.apply_kernel("copy_back", work, B, A, n)
        w.apply(O.K_COPY, workw, [(Bw, [], [(0, 0)]), (Aw, [(0, 0)], [])])
        assert len(w.msgs()) == 0 and len(LibAdapter(h).msgs()) == 0
        for X, Xw in ((A, Aw), (B, Bw)):
            np.testing.assert_array_equal(h.owner_map(X), w.owner_map(Xw))
    assert sizes == [88, 84]  # golden: 88 cells in sweep 1, 6 x 14 afterwards
    h.close()


def test_absolute_and_trapezoid_clauses_equal_apply_abs():
    """use@/def@ kernels take their boxes from set_absolute_* / set_trapezoid_* (Table 2)
    and plan exactly like the oracle's absolute-section call."""
    src = r"""
#pragma hdarray use@(X) def@(Y)
__kernel void tri(__global double *Y, __global double *X) { }
"""
    n, P = 12, 2
    h = H.HDArray(n_gpus=0, n_devices=P)
    prog = F.Program(h, F.parse(src))
    prog.bind("tri", H.K_NONE, arrays=["Y", "X"])
    w = O.Oracle(P, with_data=False)
    handles = {}
    for be in (h, w):
        X = be.create(H.F64, (n, n))
        Y = be.create(H.F64, (n, n))
        rows = be.partition(H.ROW, (n, n))
        be.write(X, rows, None)
        handles[be] = (X, Y, rows)
    X, Y, rows = handles[h]
    Xw, Yw, rowsw = handles[w]
    use = [[((0, 0), (n, 3))], []]           # dev 0 reads the first 3 columns everywhere
    tri_def = [(0, 0), (0, n - 1), (5, 5), (5, n - 1)]
    defs = [H.trapezoid(tri_def), [((6, 0), (n, n))]]
    for d in range(P):
        for lb, ub in use[d]:
            prog.set_absolute_use("tri", rows, "X", d, lb, ub)
    prog.set_trapezoid_def("tri", rows, "Y", 0, tri_def)
    prog.set_absolute_def("tri", rows, "Y", 1, (6, 0), (n, n))
    prog.apply_kernel("tri", rows, Y, X)
    w.apply_abs(O.K_NONE, rowsw, [(Yw, [[], []], defs), (Xw, use, [[], []])])
    got, ref = O.msgs_by_pair(LibAdapter(h).msgs()), O.msgs_by_pair(w.msgs())
    assert got.keys() == ref.keys() and ref
    for key in ref:
        np.testing.assert_array_equal(got[key], ref[key])
    np.testing.assert_array_equal(h.owner_map(Y), w.owner_map(Yw))
    h.close()


@pytest.mark.parametrize("src,msg", [
    ("#pragma hdarray use(Q,(0,0))\n__kernel void k(__global float *A) {}", "names no array"),
    ("#pragma hdarray use(A,(0,x))\n__kernel void k(__global float *A) {}", "bad offset"),
    ("#pragma hdarray use(A,(0,0))\nint x = 1;", "must precede a kernel"),
    ("#pragma hdarray use(A,(0,0))\n", "without a kernel"),
    ("#pragma hdarray partition(p, (8,8), dev:0, (0,4),(0,8), dev:2, (4,4),(0,8))", "devices must be"),
    ("#pragma hdarray frobnicate(A)\n__kernel void k(__global float *A) {}", "unrecognised"),
])
def test_pragma_errors(src, msg):
    with pytest.raises(F.PragmaError, match=msg):
        F.parse(src)


def test_mixed_offset_and_absolute_rejected():
    src = "#pragma hdarray use@(X) def(Y,(0,0))\n__kernel void m(__global float *Y, __global float *X) {}"
    h = H.HDArray(n_gpus=0, n_devices=2)
    prog = F.Program(h, F.parse(src))
    prog.bind("m", H.K_NONE, arrays=["Y", "X"])
    X = h.create(H.F32, (4, 4))
    Y = h.create(H.F32, (4, 4))
    p = h.partition(H.ROW, (4, 4))
    with pytest.raises(ValueError, match="mixing"):
        prog.apply_kernel("m", p, Y, X)
    h.close()


def test_emitted_c_drives_the_c_abi(tmp_path):
    """The frontend's C output (P:L372 task 3) compiles against include/hdarray.h and,
    linked with libhdarray.so in a plan-only context, plans the expected halo: the
    second Jacobi call moves row 7 (device 0 -> 1) and row 8 (1 -> 0), columns [1,15)."""
    import os
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("needs gcc")
    src = JACOBI_CU + r"""
#pragma hdarray partition(work, (16,16), dev:0, (1,7),(1,14), dev:1, (8,7),(1,14))
"""
    gen = F.emit_c(F.parse(src))
    (tmp_path / "hdam.h").write_text(gen)
    (tmp_path / "main.c").write_text(r'''
#include <stdio.h>
#include "hdam.h"
int main(void) {
  hda_ctx_t* ctx; hda_array_t A, B; hda_part_t w;
  const int64_t shape[2] = {16, 16};
  if (hda_init(&ctx, 0, NULL, 2)) return 1;
  if (hda_create(ctx, HDA_F64, 2, shape, NULL, &A) || hda_create(ctx, HDA_F64, 2, shape, NULL, &B)) return 2;
  if (hdam_partition_work(ctx, &w)) return 3;
  hda_access_t acc[2];
  hda_array_t ab[2] = {A, B}, ba[2] = {B, A};
  hdam_jacobi_step_access(acc, ab);
  if (hda_apply(ctx, HDA_K_JACOBI5, w, acc, hdam_jacobi_step_n_arrays(), NULL, 0)) return 4;
  hdam_jacobi_step_access(acc, ba);
  if (hda_apply(ctx, HDA_K_JACOBI5, w, acc, 2, NULL, 0)) return 5;
  hda_msg_t m[8]; int32_t n = 0;
  if (hda_last_plan(ctx, m, 8, &n)) return 6;
  for (int i = 0; i < n; i++)
    printf("%d %d %d %lld %lld %lld %lld\n", m[i].array, m[i].src, m[i].dst, (long long)m[i].lb[0],
           (long long)m[i].ub[0], (long long)m[i].lb[1], (long long)m[i].ub[1]);
  return hda_finalize(ctx);
}
''')
    libdir = os.path.dirname(H.lib()._name)
    inc = os.path.join(os.path.dirname(libdir), "include")
    exe = str(tmp_path / "main")
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-I", inc, "-I", str(tmp_path),
                    str(tmp_path / "main.c"), "-o", exe, "-L", libdir, "-lhdarray",
                    "-Wl,-rpath," + libdir], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, (r.returncode, r.stderr)
    rows = sorted(tuple(int(v) for v in line.split()) for line in r.stdout.split("\n") if line.strip())
    assert rows == [(0, 0, 1, 7, 8, 1, 15), (0, 1, 0, 8, 9, 1, 15)]
