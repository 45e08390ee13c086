"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/hdarray.h declares; plan-only contexts work without a GPU."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "hdarray.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hda_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for n in ("hda_create", "hda_partition", "hda_apply", "hda_sync", "hda_read", "hda_write",
              "hda_partition_manual", "hda_init", "hda_finalize"):
        assert n in names


def test_library_exports_every_declared_symbol():
    import paper_1809_05657_b200 as H
    H.lib()
    out = subprocess.run(["nm", "-D", "--defined-only", H.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (hda_[a-z_0-9]+)$", out, flags=re.M))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    assert set(H.EXPORTS) == set(declared_functions())


def test_library_is_sm100a():
    import paper_1809_05657_b200 as H
    H.lib()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", H.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_plan_only_context_and_errors():
    import paper_1809_05657_b200 as H
    h = H.HDArray(n_gpus=0, n_devices=4)
    assert h.plan_only
    X = h.create(H.F64, (8, 8))
    p = h.partition(H.ROW, (8, 8))
    with pytest.raises(H.HDAError) as e:
        h.partition(H.COL, (8,))
    assert e.value.code == H.EUNSUPPORTED
    with pytest.raises(H.HDAError) as e:
        h.partition_manual((8, 8), [[0, 0], [2, 0], [5, 0], [6, 0]], [[4, 8], [5, 8], [6, 8], [8, 8]])
    assert e.value.code == H.EOVERLAP
    with pytest.raises(H.HDAError) as e:
        h.apply(H.K_NONE, p, [(X, [], [(0, 0), (1, 0)])])
    assert e.value.code == H.ERACE
    with pytest.raises(H.HDAError) as e:
        h.apply(H.K_JACOBI5, p, [(X, [], [(0, 0)]), (X, [(0, 1)], [])])
    assert e.value.code in (H.EINVAL, H.ERANGE)
    h.apply(H.K_NONE, p, [(X, [(0, 1)], [])])
    assert h.stats()["n_apply"] == 1
    with pytest.raises(H.HDAError) as e:
        h.stream(0)
    h.close()


def test_prepared_call_equals_apply():
    import paper_1809_05657_b200 as H
    J = [(0, -1), (0, 1), (-1, 0), (1, 0)]
    plans = []
    for prepared in (False, True):
        h = H.HDArray(n_gpus=0, n_devices=3)
        A, B = h.create(H.F64, (20, 16)), h.create(H.F64, (20, 16))
        data = h.partition(H.ROW, (20, 16))
        work = h.partition(H.ROW, (20, 16), (1, 1), (19, 15))
        h.write(A, data, None)
        h.write(B, data, None)
        fwd = [(A, [], [(0, 0)]), (B, J, [])]
        bwd = [(B, [], [(0, 0)]), (A, J, [])]
        if prepared:
            calls = [h.prepare(H.K_JACOBI5, work, fwd), h.prepare(H.K_JACOBI5, work, bwd)]
        seq = []
        for s in range(6):
            if prepared:
                calls[s % 2]()
            else:
                h.apply(H.K_JACOBI5, work, fwd if s % 2 == 0 else bwd)
            seq.append(h.last_plan())
        plans.append(seq)
        h.close()
    assert plans[0] == plans[1] and any(plans[0])
