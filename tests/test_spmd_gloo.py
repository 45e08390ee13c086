"""SPMD host logic with world_size 2 over gloo (CPU): every rank runs the replicated
tracker ("each process maintains coherent local copies of the four sets for
all processes") and must derive the same plan as every other rank and as a
single-process context; each rank drives only its own device."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _program(h, H):
    J = [(0, -1), (0, 1), (-1, 0), (1, 0)]
    A = h.create(H.F64, (20, 12))
    B = h.create(H.F64, (20, 12))
    data = h.partition(H.ROW, (20, 12))
    work = h.partition(H.ROW, (20, 12), (1, 1), (19, 11))
    col = h.partition(H.COL, (20, 12))
    h.write(A, data, None)
    h.write(B, data, None)
    plans = []
    for s in range(3):
        h.apply(H.K_JACOBI5, work, [(A, [], [(0, 0)]), (B, J, [])])
        plans.append(h.last_plan())
        h.apply(H.K_COPY, work, [(B, [], [(0, 0)]), (A, [(0, 0)], [])])
        plans.append(h.last_plan())
    h.apply(H.K_SCALE, col, [(B, [(0, 0)], [(0, 0)])], [2.0])  # ROW -> COL repartition
    plans.append(h.last_plan())
    return plans, h.owner_map(B).tolist(), h.stats()["plan_hits"]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1809_05657_b200 as H
    h = H.HDArray.spmd(world, rank, gpu_id=-1)
    local = [h.L.hda_is_local is not None]
    import ctypes
    flags = []
    for d in range(world):
        v = ctypes.c_int32()
        h.L.hda_is_local(h.h, d, ctypes.byref(v))
        flags.append(v.value)
    res = _program(h, H)
    allres = [None] * world
    dist.all_gather_object(allres, res)
    q.put((rank, flags, allres))
    dist.destroy_process_group()
    del local


@pytest.mark.parametrize("world", [2, 4])
def test_spmd_replicated_tracker_gloo(world):
    import paper_1809_05657_b200 as H
    H.lib()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    single = H.HDArray(n_gpus=0, n_devices=world)
    ref = _program(single, H)
    for rank, flags, allres in out:
        assert flags == [1 if d == rank else 0 for d in range(world)]
        for r in allres:
            assert r[0] == ref[0]  # identical plans on every rank
            assert r[1] == ref[1]  # identical owner maps
    assert any(len(p) for p in ref[0])
