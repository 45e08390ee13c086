"""Debug: the bench's repartition sequence under SPMD (torchrun), syncing after every
call so a protocol deadlock shows up as HDA_ETIMEOUT at the call that caused it.
    HDA_TIMEOUT_MS=3000 torchrun --nproc-per-node 2 tools/dbg_spmd_rep.py [n] [backend]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1809_05657_b200 as H  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
backend = sys.argv[2] if len(sys.argv) > 2 else "nccl"
rank, ws, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
if backend == "nccl":
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
else:
    dist.init_process_group("gloo")
h = H.HDArray.spmd(ws, rank, local)
check = os.environ.get("CHECK", "0") == "1"
if check:
    import oracle as O
    w = O.Oracle(ws)
h.set_transport(int(os.environ.get("XPORT", "2")))
h.set_overlap(os.environ.get("OVERLAP", "1") == "1")
bes = (h, w) if check else (h,)
for be in bes:
    X = be.create(H.F32, (n, n))
    rowp = be.partition(H.ROW, (n, n))
    colp = be.partition(H.COL, (n, n))
alpha = float(os.environ.get("ALPHA", "1.0"))


def on_all(fn):
    return lambda: [fn(be) for be in bes]


steps = [("stamp", on_all(lambda be: be.apply(H.K_STAMP, rowp, [(X, [], [(0, 0)])], [4242.0])))]
for i in range(4):
    steps.append((f"scale-col{i}", on_all(lambda be: be.apply(H.K_SCALE, colp, [(X, [(0, 0)], [(0, 0)])], [alpha]))))
    steps.append((f"scale-row{i}", on_all(lambda be: be.apply(H.K_SCALE, rowp, [(X, [(0, 0)], [(0, 0)])],
                                                            [1.0 / alpha]))))
for name, fn in steps:
    t0 = time.time()
    try:
        fn()
        h.sync()
        if check:
            g, o = h.read_replica(X, rank), w.replica(X, rank)
            if g.tobytes() != o.tobytes():
                bad = g.view("u4") != o.view("u4")
                rr, cc = bad.nonzero()
                print(f"rank {rank} {name}: REPLICA MISMATCH {bad.sum()} cells rows {rr.min()}..{rr.max()} "
                      f"cols {cc.min()}..{cc.max()} e.g. got {g[rr[0], cc[0]]} want {o[rr[0], cc[0]]}", flush=True)
        print(f"rank {rank} {name}: ok {time.time() - t0:.3f}s msgs={h.stats()['last_msgs']}", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"rank {rank} {name}: FAILED after {time.time() - t0:.3f}s: {e}", flush=True)
        break
    if os.environ.get("BARRIER", "0") == "1":
        dist.barrier()
h.close()
dist.destroy_process_group()
