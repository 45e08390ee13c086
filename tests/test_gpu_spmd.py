"""SPMD mode on >= 2 GPUs: one process per GPU (the bench's torchrun layout), peer
replicas mapped with CUDA IPC, device-side sync words.  Each rank compares its own
replica with the oracle after every call (bit-exact), for halo exchange (ROW Jacobi,
BLOCK 9-point with corners), a ROW<->COL repartition and the 2MM chain with its
all-gathers fused into the product."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

J = [(0, -1), (0, 1), (-1, 0), (1, 0)]
N9 = [(i, j) for i in (-1, 0, 1) for j in (-1, 0, 1) if i or j]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, env1, gate):
    try:
        os.environ["HDA_TIMEOUT_MS"] = "20000"  # a protocol deadlock fails in seconds
        os.environ["HDA_CE_BYTES"] = "262144"  # 2MM's 512 KiB row blocks on the copy engine (gated product)
        os.environ["HDA_GEMM_GATE"] = gate  # 1: gated inside the kernel; 2 (default): split launches
        if rank == 1:  # rank 1 only: an asymmetric slow reader opens the WAR window
            os.environ.update(env1)
        import torch
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        gpu = rank % torch.cuda.device_count()  # 8 ranks on 4 GPUs: two processes per GPU
        torch.cuda.set_device(gpu)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle as O
        import paper_1809_05657_b200 as H
        import synth
        h = H.HDArray.spmd(world, rank, gpu)
        h.set_transport(int(os.environ.get("HDA_TEST_TRANSPORT", "2")))
        w = O.Oracle(world)
        shape = (130, 262)
        u0 = synth.uniform(5, shape)
        bad = []

        def check(tag, arrs):
            for a in arrs:
                if h.read_replica(a, rank).tobytes() != w.replica(a, rank).tobytes():
                    bad.append((tag, a))
                if not (h.owner_map(a) == w.owner_map(a)).all():
                    bad.append((tag, "owner", a))

        for be in (h, w):
            X = be.create(H.F64, shape, u0)
            Y = be.create(H.F64, shape, u0)
            rowp = be.partition(H.ROW, shape, (1, 1), (shape[0] - 1, shape[1] - 1))
            blk = be.partition(H.BLOCK, shape, (1, 1), (shape[0] - 1, shape[1] - 1))
            colp = be.partition(H.COL, shape)
            full = be.partition(H.ROW, shape)
        for it in range(4):
            for be in (h, w):
                be.apply(H.K_JACOBI5, rowp, [(Y, [], [(0, 0)]), (X, J, [])])
                be.apply(H.K_STENCIL9, blk, [(X, [], [(0, 0)]), (Y, N9, [])])
            check(f"it{it}", [X, Y])
        for be in (h, w):
            be.apply(H.K_SCALE, colp, [(X, [(0, 0)], [(0, 0)])], [2.0])
            be.apply(H.K_SCALE, full, [(X, [(0, 0)], [(0, 0)])], [0.5])
        check("repart", [X])
        # WAR: rank 1 pulls X's top-right block from rank 0 (COPY on COL), then rank 0
        # rescales its own rows of X in place — needing nothing from rank 1, only its ACK
        for it in range(3):
            for be in (h, w):
                be.write(X, full, u0 + it)
                be.apply(H.K_COPY, colp, [(Y, [], [(0, 0)]), (X, [(0, 0)], [])])
                be.apply(H.K_SCALE, full, [(X, [(0, 0)], [(0, 0)])], [2.0])
            check(f"war{it}", [X, Y])
        # bulk ROW<->COL blocks (>= 1 MiB) through the copy engine under AUTO
        big = (1024, 2048)
        v = synth.uniform(8, big, "f32")
        for be in (h, w):
            Z = be.create(H.F32, big)
            rp = be.partition(H.ROW, big)
            cp = be.partition(H.COL, big)
            be.write(Z, rp, v)
            for it in range(3):
                be.apply(H.K_SCALE, cp, [(Z, [(0, 0)], [(0, 0)])], [2.0])
                be.apply(H.K_SCALE, rp, [(Z, [(0, 0)], [(0, 0)])], [0.5])
        check("bulk", [Z])
        # GPU-filling in-place SCALE kernels whose WAR waits depend on the peer's bulk
        # copy-engine pulls: waiting inside every CTA starved the copies (deadlock,
        # found in the configs[3] bench); the wait now runs in one CTA first
        big2 = (4096, 4096)
        v2 = synth.uniform(9, big2, "f32")
        for be in (h, w):
            Z2 = be.create(H.F32, big2)
            rp2 = be.partition(H.ROW, big2)
            cp2 = be.partition(H.COL, big2)
            be.write(Z2, rp2, v2)  # finite values: SCALE of a NaN payload is not bit-defined
            for it in range(2):
                be.apply(H.K_SCALE, cp2, [(Z2, [(0, 0)], [(0, 0)])], [2.0])
                be.apply(H.K_SCALE, rp2, [(Z2, [(0, 0)], [(0, 0)])], [0.5])
        check("bulk-gpu-filling", [Z2])
        # 2MM under ROW: the B and D all-gathers fused into the product — the
        # GEMM starts on its own rows and waits per k-block for the copy-engine blocks
        # (stream-written arrival flags, no SM time on the comm stream); integer inputs
        # keep E exact in any k order
        n2, S = 1024, H.STAR
        Ab, Bb, Cb = (synth.int_bf16(70 + i, (n2, n2), -1, 1) for i in range(3))
        g0 = h.stats()["gated_products"]
        for be in (h, w):
            GA, GB, GC, GD = (be.create(H.BF16, (n2, n2)) for _ in range(4))
            GE = be.create(H.F32, (n2, n2))
            gp = be.partition(H.ROW, (n2, n2))
            for Xg, v in ((GA, Ab), (GB, Bb), (GC, Cb)):
                be.write(Xg, gp, v)
            for it in range(2):
                be.apply(H.K_GEMM, gp, [(GD, [], [(0, 0)]), (GA, [(0, S)], []), (GB, [(S, 0)], [])], [1.0, 0.0])
                be.apply(H.K_GEMM, gp, [(GE, [], [(0, 0)]), (GC, [(0, S)], []), (GD, [(S, 0)], [])], [1.0, 0.0])
        check("2mm-gated", [GB, GD, GE])
        # gated: B once, D twice (this rank's device); split: the two fp32 E products only
        # (the bf16 D products join); at 8 ranks the 128-row shares are below the
        # CTA-pair kernel's 256 rows, so the products join the copies instead
        if world <= 4 and h.stats()["gated_products"] - g0 != {"1": 3, "2": 2}[gate]:
            bad.append(("gated", h.stats()["gated_products"] - g0))
        # Reduce over NVLink sync words: every rank gets the oracle's value
        ints = np.arange(np.prod(shape), dtype=np.float64).reshape(shape) % 97
        for be in (h, w):
            be.write(X, full, ints)
        for op in (H.SUM, H.MAX, H.MIN, H.SUM, H.MIN, H.MAX):  # back to back, distinct partials
            g, o = h.reduce(X, colp, op), w.reduce(X, colp, op)
            if g != o:
                bad.append(("reduce", op, g, o))
        got = h.read(X, full)
        ref = w.read(X, full)
        lb, ub = h.region(full, rank, 2)
        if got[lb[0]:ub[0]].tobytes() != ref[lb[0]:ub[0]].tobytes():
            bad.append(("read",))
        st = h.stats()
        h.close()
        dist.destroy_process_group()
        q.put((rank, bad, st["msgs_total"], st["plan_hits"]))
    except Exception as e:  # report instead of hanging the parent
        import traceback
        q.put((rank, ["exception", traceback.format_exc()], 0, 0))


def _run(world, env1, gate="1"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q, env1, gate)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for rank, bad, msgs, hits in out:
        assert not bad, (rank, bad)
        assert msgs > 0 and hits > 0


# HDA_DEBUG_PULL_DELAY_US makes rank 1's pulls sleep after their RAW waits: a writer
# that overwrote cells without waiting for rank 1's ACK would break parity.
# HDA_DEBUG_REDUCE_READ_DELAY_US makes rank 1's host read its reduce partials late: a
# peer's next reduce must not overwrite them (two alternating slot banks).
@pytest.mark.parametrize("env1", [{}, {"HDA_DEBUG_PULL_DELAY_US": "300", "HDA_DEBUG_REDUCE_READ_DELAY_US": "50000"},
                                  {"HDA_DEBUG_PULL_DELAY_US": "300", "HDA_HALO_MODE": "1"}],
                         ids=["plain", "slow-reader", "slow-reader-fused"])
def test_spmd_two_gpus(env1):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    _run(2, env1)


def test_spmd_two_gpus_split_product():
    """The default split product (HDA_GEMM_GATE=2) across processes: the 2MM E products
    run their resident rows beside the copy-engine all-gather of D and the arrived rows
    after it; everything else as in the plain two-GPU run."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    _run(2, {}, gate="2")


def test_spmd_four_gpus():
    """4 ranks: ROW halos with two neighbours, BLOCK 2x2 with corners, a 4-way
    repartition all-to-all and reductions, every replica against the oracle."""
    import torch
    if torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    _run(4, {})


def test_spmd_eight_ranks():
    """8 ranks (the N=8 layout; two processes per GPU on a 4-GPU box, CUDA IPC within a
    GPU too): ROW halos, BLOCK 4x2 with corners, an 8-way repartition all-to-all, the 2MM
    all-gathers and reductions, every replica against the oracle."""
    import torch
    if torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    _run(8, {})
