#!/usr/bin/env python
"""Benchmark of the HDArray hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload jacobi2d|...] [--impl reference]

N > 1 is launched by the driver with torchrun, one rank per GPU; every rank runs
the paper's SPMD model (hda_init_spmd, replicated tracker, CUDA-IPC peer replicas).

One STEP = one pass of the whole hot path for one call: tracker (plan-cache hit in
steady state) -> halo exchange (pack/transfer/unpack over NVLink) -> stencil kernel
-> commit, i.e. one hda_apply sweep (ping-pong X->Y, Y->X) of configs[1]
(8192^2 fp64 Jacobi, ROW partition of the interior).  value = interior points of the
whole array x K / (max over ranks of the device-timed region).

Only the CPU-baseline legs (cpu_baseline, --impl reference) execute oracle/.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "stencil GPoints/s and halo/repartition GB/s at 1/2/4/8 B200 vs roofline"
J = [(0, -1), (0, 1), (-1, 0), (1, 0)]
NVLINK_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md); 900 nominal


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.p = None
        self.lines = []

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.p = None

    def _read(self):
        for line in self.p.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ----------------------------------------------------------------------------- CPU legs
def oracle_sample(seconds_target=15.0, rows=1026, cols=8192, max_sweeps=400):
    """The oracle as it stands (plain C, one thread): P=1 Jacobi sweeps on a row slab of
    configs[1] (8192 columns), with per-element last-writer maps and checked reads."""
    import oracle as O
    import synth
    w = O.Oracle(1)
    u = synth.uniform(synth.SEED0 + 1, (rows, cols))
    X = w.create(O.F64, (rows, cols), u)
    Y = w.create(O.F64, (rows, cols), u)
    part = w.partition(O.ROW, (rows, cols), (1, 1), (rows - 1, cols - 1))
    pts = (rows - 2) * (cols - 2)
    t0 = time.perf_counter()
    s = 0
    while s < max_sweeps:
        src, dst = (X, Y) if s % 2 == 0 else (Y, X)
        w.apply(O.K_JACOBI5, part, [(dst, [], [(0, 0)]), (src, J, [])])
        s += 1
        if time.perf_counter() - t0 > seconds_target:
            break
    dt = time.perf_counter() - t0
    return {"value": pts * s / dt / 1e9, "unit": "GPoints/s", "cores": 1, "kind": "oracle",
            "sample": f"oracle P=1 Jacobi on a {rows}x{cols} slab of configs[1], {s} sweeps, {dt:.1f} s"}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle as O
    import synth
    O.build()
    rows, cols = 258, 8192  # bounded sample of configs[1] per step
    w = O.Oracle(1)
    u = synth.uniform(synth.SEED0 + 1, (rows, cols))
    X = w.create(O.F64, (rows, cols), u)
    Y = w.create(O.F64, (rows, cols), u)
    part = w.partition(O.ROW, (rows, cols), (1, 1), (rows - 1, cols - 1))
    pts = (rows - 2) * (cols - 2)
    for s in range(args.warmup):
        w.apply(O.K_JACOBI5, part, [(Y if s % 2 == 0 else X, [], [(0, 0)]), (X if s % 2 == 0 else Y, J, [])])
    t0 = time.perf_counter()
    for s in range(args.steps):
        src, dst = (X, Y) if s % 2 == 0 else (Y, X)
        w.apply(O.K_JACOBI5, part, [(dst, [], [(0, 0)]), (src, J, [])])
    dt = time.perf_counter() - t0
    v = pts * args.steps / dt / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GPoints/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "configs[1] 8192^2 fp64 Jacobi (bounded sample: 258x8192 slab per step)"},
            "cpu_baseline": {"value": v, "unit": "GPoints/s", "cores": 1, "kind": "oracle",
                             "sample": f"oracle P=1 Jacobi sweep of a {rows}x{cols} slab per step"},
            "e2e": {"value": v, "unit": "GPoints/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="hdarray")
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--e2e-sweeps", type=int, default=100)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--transport", type=int, default=0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_1809_05657_b200 as H
    import synth

    ws, rank, local = dist_env()
    if ws != args.gpus:
        args.gpus = ws
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    hbm_peak, peak_src = peaks()

    n = args.n
    P = ws
    if ws > 1:
        h = H.HDArray.spmd(P, rank, local)
    else:
        h = H.HDArray(n_gpus=1, n_devices=1, gpu_ids=[local])
    h.set_transport(args.transport)
    a_mode, b_mode = 37, 61
    u0 = synth.eigenmode2d(n, n, a_mode, b_mode)
    X = h.create(H.F64, (n, n), u0)
    Y = h.create(H.F64, (n, n), u0)
    work = h.partition(H.ROW, (n, n), (1, 1), (n - 1, n - 1))
    data = h.partition(H.ROW, (n, n))
    my_lb, my_ub = h.region(work, rank, 2)
    my_pts = (my_ub[0] - my_lb[0]) * (my_ub[1] - my_lb[1])
    total_pts = (n - 2) * (n - 2)
    stream = torch.cuda.ExternalStream(h.stream(rank))
    sweeps_done = [0]
    state = {"src": X, "dst": Y}

    def step():
        h.apply(H.K_JACOBI5, work, [(state["dst"], [], [(0, 0)]), (state["src"], J, [])])
        state["src"], state["dst"] = state["dst"], state["src"]
        sweeps_done[0] += 1

    def barrier():
        h.sync()
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()

    def max_over_ranks(x):
        if ws == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if ws == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    # L2 policy: inputs larger than L2 => back-to-back steps; otherwise flush between steps
    l2_bytes = torch.cuda.get_device_properties(local).L2_cache_size
    work_set = 2 * (my_ub[0] - my_lb[0] + 2) * n * 8
    flush = work_set < 2 * l2_bytes
    flush_buf = torch.empty(int(2 * l2_bytes), dtype=torch.uint8, device="cuda") if flush else None

    for _ in range(args.warmup):
        step()
    barrier()
    h.reset_stats()

    # ---- timed region (device-timed on the library's stream, max over ranks)
    clk = Clocks(local)
    clk.start()
    time.sleep(0.2)
    launches0 = h.stats()["kernel_launches"]
    if not flush:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        barrier()
        ms = ev0.elapsed_time(ev1)
    else:
        ms = 0.0
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        barrier()
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush_buf.zero_()
            if ws > 1:
                torch.cuda.synchronize()
                dist.barrier()
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        barrier()
        ms = sum(a.elapsed_time(b) for a, b in evs)
    launches = h.stats()["kernel_launches"] - launches0
    clocks = clk.stop()
    st = h.stats()
    ms = max_over_ranks(ms)
    value = total_pts * args.steps / (ms * 1e-3) / 1e9

    # ---- per-kernel timing pass (CUDA events bracketing each launch on its stream)
    h.set_kernel_timing(True)
    h.reset_stats()
    kt_steps = min(args.steps, 200)
    for _ in range(kt_steps):
        step()
    barrier()
    k_ms, k_n = h.kernel_time(H.K_JACOBI5)
    x_ms, x_n = h.exchange_time()
    st_kt = h.stats()
    h.set_kernel_timing(False)
    k_avg = k_ms / max(k_n, 1)
    achieved = my_pts * 16 / (k_avg * 1e-3) / 1e9  # algorithmic bytes: 8 B read + 8 B write per point
    achieved = min(achieved, sum_over_ranks(achieved) / ws) if ws > 1 else achieved
    halo_bytes = st_kt["bytes_total"] / max(kt_steps, 1)
    x_avg = x_ms / max(x_n, 1)

    # ---- parity against the closed form (eigenmode) on this rank's rows
    lam = (np.cos(a_mode * np.pi / (n - 1)) + np.cos(b_mode * np.pi / (n - 1))) / 2
    got = h.read(state["src"], data)
    d_lb, d_ub = h.region(data, rank, 2)
    rows = slice(max(my_lb[0], d_lb[0]), min(my_ub[0], d_ub[0]))
    ref = lam ** sweeps_done[0] * u0[rows]
    err = float(np.max(np.abs(got[rows] - ref)) / np.max(np.abs(ref)))
    err = max_over_ranks(err)

    # ---- end to end through the C-ABI with host buffers: write (pinned H2D) ->
    # e2e_sweeps sweeps -> read (D2H) per job
    host_in = torch.from_numpy(u0).pin_memory()
    host_out = torch.empty((n, n), dtype=torch.float64).pin_memory()
    jobs = 2
    e2e_times = []
    for j in range(jobs + 1):
        barrier()
        t0 = time.perf_counter()
        h.write_ptr(X, data, host_in.data_ptr())
        state["src"], state["dst"] = X, Y
        for _ in range(args.e2e_sweeps):
            step()
        h.read_ptr(state["src"], data, host_out.data_ptr())
        barrier()
        if j:
            e2e_times.append(time.perf_counter() - t0)
    e2e_s = max_over_ranks(min(e2e_times))
    my_rows = my_ub[0] - my_lb[0] + (1 if rank == 0 else 0) + (1 if rank == ws - 1 else 0)
    e2e = {"value": total_pts * args.e2e_sweeps / e2e_s / 1e9, "unit": "GPoints/s",
           "h2d_bytes_per_step": int(sum_over_ranks(my_rows * n * 8)),
           "d2h_bytes_per_step": int(sum_over_ranks(my_rows * n * 8)),
           "step": f"one configs[1] job: hda_write X -> {args.e2e_sweeps} sweeps -> hda_read (host wall clock)"}

    launches = int(sum_over_ranks(launches))
    if rank == 0:
        cpu = None
        if ws == 1 and not args.no_cpu_baseline:
            cpu = oracle_sample()
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            try:
                traffic = json.load(open(tp)).get(f"jacobi5_f64_n{n}_P{ws}")
            except Exception:
                traffic = None
        line = {
            "metric": METRIC, "value": value, "unit": "GPoints/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "configs[1]: 8192x8192 fp64 Jacobi (P:L459), ROW partition of the interior, "
                                   "ping-pong sweeps through hda_apply", "n": n, "global_points": total_pts,
                       "parallelism": f"spmd{ws}" if ws > 1 else "single",
                       "transport": ["fused", "staged"][args.transport],
                       "l2": ("L2 flushed between timed steps" if flush else
                              f"inputs larger than L2 (per-GPU working set {work_set / 2**20:.0f} MiB)")},
            "roofline": {"bound": "hbm", "kernel": "stencil2d_kernel<double,JACOBI5>",
                         "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                         "traffic": traffic, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": my_pts * 16, "avg_launch_ms": k_avg},
            "exchange": {"halo_bytes_per_step": halo_bytes, "exchange_ms_per_step": x_avg if x_n else 0.0,
                         "halo_GBps_per_gpu": (halo_bytes / ws / (x_avg * 1e-3) / 1e9) if x_n else None,
                         "nvlink_peak_GBps": NVLINK_GBS},
            "parity": {"closed_form_normwise_err": err, "tol": 1e-12, "pass": err < 1e-12},
            "tracker": {"plan_hits": st["plan_hits"], "plan_misses": st["plan_misses"],
                        "tracker_us_per_call": st["tracker_us"] / max(st["n_apply"], 1)},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    h.close()
    if ws > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
