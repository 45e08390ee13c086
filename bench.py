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

import synth

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


def _env_int(name, default):
    """The library's kernel switches (read once per process by libhdarray), for naming
    the kernel a roofline line describes."""
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


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


def jacobi_workload(n):
    return (f"configs[1]: {n}x{n} fp64 Jacobi (P:L459), ROW partition of the interior, "
            "ping-pong sweeps through hda_apply")


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    if args.workload != "jacobi2d":
        print(json.dumps({"impl": "reference", "unavailable": "the oracle arm times the default jacobi2d workload "
                                                              "only"}), flush=True)
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
            "config": {"workload": jacobi_workload(8192), "n": 8192,
                       "parallelism": f"spmd{ws}" if ws > 1 else "single"},
            "cpu_baseline": {"value": v, "unit": "GPoints/s", "cores": 1, "kind": "oracle",
                             "sample": f"oracle (plain C, one thread, rank 0 only) P=1 Jacobi sweep of a {rows}x{cols} "
                                       "slab of configs[1] per step; value = slab points / time"},
            "e2e": {"value": v, "unit": "GPoints/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- workloads
N9 = [(i, j) for i in (-1, 0, 1) for j in (-1, 0, 1) if i or j]
N7 = [(0, 0, -1), (0, 0, 1), (0, -1, 0), (0, 1, 0), (-1, 0, 0), (1, 0, 0)]


class Stencil:
    """configs[1] (jacobi2d), configs[2] (stencil9) and the 3-D half of configs[4]
    (stencil7): ping-pong sweeps over the interior, eigenmode inputs (closed-form parity)."""

    def __init__(self, kind, H, h, rank, ws, n=None):
        self.kind, self.H, self.h, self.rank, self.ws = kind, H, h, rank, ws
        if kind == "jacobi2d":
            self.n = n or 8192
            self.shape, self.dt, self.es = (self.n, self.n), H.F64, 8
            self.K, self.uses, self.part_kind = H.K_JACOBI5, J, H.ROW
            self.modes = (37, 61)
            self.workload = jacobi_workload(self.n)
            self.kname = ("stencil2d_tma_kernel<double,0> (TMA ring)" if _env_int("HDA_TMA", 0) == 2
                          else "stencil2d_kernel<double,JACOBI5>")
        elif kind == "stencil9":
            self.n = n or 16384
            self.shape, self.dt, self.es = (self.n, self.n), H.F64, 8
            self.K, self.uses, self.part_kind = H.K_STENCIL9, N9, H.BLOCK
            self.modes = (3, 4)
            self.workload = (f"configs[2]: {self.n}x{self.n} fp64 9-point stencil (R12), BLOCK partition of the "
                             "interior with corner halos, ping-pong sweeps")
            self.kname = ("stencil2d_tma_kernel<double,1> (TMA ring)" if _env_int("HDA_TMA", 0) >= 1
                          else "stencil2d_kernel<double,STENCIL9>")
        else:
            self.n = n or 1024
            self.shape, self.dt, self.es = (self.n,) * 3, H.F32, 4
            self.K, self.uses, self.part_kind = H.K_STENCIL7_3D, N7, H.ROW
            self.modes = (5, 7, 9)
            self.workload = (f"configs[4] (3-D half): {self.n}^3 fp32 7-point stencil (R13), slab (ROW) partition "
                             "of the interior, ping-pong sweeps")
            self.kname = "stencil7_kernel<float>"
        self.dtype_name = "f64" if self.es == 8 else "f32"
        nd = len(self.shape)
        self.zero = [(0,) * nd]
        self.u0 = self.initial()
        self.X = h.create(self.dt, self.shape, self.u0)
        self.Y = h.create(self.dt, self.shape, self.u0)
        self.work = h.partition(self.part_kind, self.shape, (1,) * nd, tuple(s - 1 for s in self.shape))
        self.data = h.partition(H.ROW, self.shape)
        self.lb, self.ub = h.region(self.work, rank, nd)
        self.my_pts = int(np.prod(np.subtract(self.ub, self.lb)))
        self.units = int(np.prod([s - 2 for s in self.shape]))  # interior points per step
        self.alg_per_launch = self.my_pts * 2 * self.es
        self.src, self.dst, self.sweeps = self.X, self.Y, 0
        self.calls = [h.prepare(self.K, self.work, [(d, [], self.zero), (s, self.uses, [])])
                      for s, d in ((self.X, self.Y), (self.Y, self.X))]
        self.metric_unit = "GPoints/s"
        self.bound = "hbm"
        self.working_set = 2 * int(np.prod(np.subtract(self.ub, self.lb) + 2)) * self.es

    def initial(self):
        if len(self.shape) == 2:
            return synth.eigenmode2d(self.shape[0], self.shape[1], *self.modes)
        n = self.n
        a, b, c = self.modes
        sz = np.sin(a * np.pi * np.arange(n) / (n - 1))
        sy = np.sin(b * np.pi * np.arange(n) / (n - 1))
        sx = np.sin(c * np.pi * np.arange(n) / (n - 1))
        for v in (sz, sy, sx):
            v[0] = v[-1] = 0.0
        u = np.empty(self.shape, np.float32)
        yx = np.outer(sy, sx)
        for z in range(n):
            u[z] = (sz[z] * yx).astype(np.float32)
        return u

    def lam(self):
        th = [m * np.pi / (s - 1) for m, s in zip(self.modes, self.shape)]
        if self.kind == "jacobi2d":
            return (np.cos(th[0]) + np.cos(th[1])) / 2
        if self.kind == "stencil9":
            return (8 * (np.cos(th[0]) + np.cos(th[1])) + 4 * np.cos(th[0]) * np.cos(th[1])) / 20
        return sum(np.cos(t) for t in th) / 3

    def step(self):
        self.calls[0 if self.src == self.X else 1]()
        self.src, self.dst = self.dst, self.src
        self.sweeps += 1

    def reset_input(self):
        self.src, self.dst = self.X, self.Y

    def parity(self):
        got = self.h.read(self.src, self.data)
        d_lb, d_ub = self.h.region(self.data, self.rank, len(self.shape))
        r0, r1 = max(self.lb[0], d_lb[0]), min(self.ub[0], d_ub[0])
        ref = self.lam() ** self.sweeps * self.u0[r0:r1].astype(np.float64)
        err = float(np.max(np.abs(got[r0:r1].astype(np.float64) - ref)) / max(np.max(np.abs(ref)), 1e-300))
        tol = 1e-12 if self.es == 8 else 1e-4
        return {"closed_form_normwise_err": err, "tol": tol, "sweeps": self.sweeps}


class Repartition:
    """configs[3]: 32768^2 fp32, K1 = SCALE under ROW, K2 = SCALE under COL; every
    switch is a full P(P-1)-block redistribution (all-to-all over NVLink)."""

    def __init__(self, H, h, rank, ws, n=None):
        self.H, self.h, self.rank, self.ws = H, h, rank, ws
        self.n = n or 32768
        self.shape = (self.n, self.n)
        self.X = h.create(H.F32, self.shape)
        self.rowp = h.partition(H.ROW, self.shape)
        self.colp = h.partition(H.COL, self.shape)
        self.seed = 4242
        h.apply(H.K_STAMP, self.rowp, [(self.X, [], [(0, 0)])], [float(self.seed)])  # device-side init
        self.kind = "repartition"
        self.workload = (f"configs[3]: repartition ROW<->COL of a {self.n}x{self.n} fp32 array between two "
                         "SCALE kernels (alpha=1), all-to-all over NVLink")
        self.kname = "copy_runs_kernel (fused NVLink pull)"
        self.dtype_name = "f32"
        self.metric_unit = "GB/s"
        self.bound = "nvlink" if ws > 1 else "hbm"
        self.calls = 0
        self.prepared = [h.prepare(H.K_SCALE, p, [(self.X, [(0, 0)], [(0, 0)])], [1.0])
                         for p in (self.colp, self.rowp)]
        P = ws
        blk = (self.n // P) * (self.n // P) * 4
        self.units = P * (P - 1) * blk  # bytes moved by all ranks per call (one redistribution)
        self.alg_per_launch = (P - 1) * blk  # bytes pulled by this rank per call
        self.my_pts = 0
        self.working_set = self.n * self.n * 4

    def step(self):
        self.prepared[self.calls % 2]()
        self.calls += 1

    def e2e_setup(self, torch):
        self.hX = torch.empty(self.shape, dtype=torch.float32).pin_memory()
        self.hX.numpy()[:] = 1.0
        self.hY = torch.empty(self.shape, dtype=torch.float32).pin_memory()
        self.e2e_units = 2 * self.units  # two redistributions per job
        lb, ub = self.h.region(self.rowp, self.rank, 2)
        b = (ub[0] - lb[0]) * (ub[1] - lb[1]) * 4
        self.e2e_bytes = (b, b)
        self.e2e_desc = ("one job: hda_write X by rows -> SCALE by columns -> SCALE by rows -> hda_read X "
                         "(host wall clock, pinned)")

    def e2e_job(self):
        self.h.write_ptr(self.X, self.rowp, self.hX.data_ptr())
        self.prepared[0]()
        self.prepared[1]()
        self.h.read_ptr(self.X, self.rowp, self.hY.data_ptr())

    def reset_input(self):
        pass

    def parity(self):
        # raw bits of a sampled block of this rank's rows against splitmix64 (STAMP is
        # splitmix64(seed*phi + c)); SCALE by 1.0 keeps every non-NaN value bit-exact
        got = self.h.read(self.X, self.rowp)
        lb, ub = self.h.region(self.rowp, self.rank, 2)
        r = lb[0]
        c = np.arange(self.n, dtype=np.int64) + r * self.n
        exp = synth.splitmix64_stream(self.seed, int(c[0]), self.n)
        e32 = (exp & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.float32)
        g = got[r]
        ok = (g.view(np.uint32) == e32.view(np.uint32)) | (np.isnan(g) & np.isnan(e32))
        return {"raw_bits_row_match": bool(ok.all()), "row": int(r)}


class Gemm:
    """configs[4] (product half): C = A @ B, 16384^2 bf16 in, fp32 C, ROW partition;
    call 1 all-gathers B, steady-state calls move nothing."""

    def __init__(self, H, h, rank, ws, n=None):
        self.H, self.h, self.rank, self.ws = H, h, rank, ws
        self.n = n or 16384
        n = self.n
        S = H.STAR
        self.Ab = synth.int_bf16(51, (n, n))
        self.Bb = synth.int_bf16(52, (n, n))
        self.A = h.create(H.BF16, (n, n))
        self.B = h.create(H.BF16, (n, n))
        self.C = h.create(H.F32, (n, n))
        self.part = h.partition(H.ROW, (n, n))
        h.write(self.A, self.part, self.Ab)
        h.write(self.B, self.part, self.Bb)
        self.acc = [(self.C, [], [(0, 0)]), (self.A, [(0, S)], []), (self.B, [(S, 0)], [])]
        self.kind = "gemm"
        self.workload = f"configs[4] (product half): {n}^2 bf16 GEMM, fp32 accumulate and C, ROW partition, B use=all"
        self.kname = ("gemm2_kernel<float> (tcgen05 cta_group::2)" if _env_int("HDA_GEMM_2SM", 1)
                      else "gemm_kernel<float> (tcgen05)")
        self.dtype_name = "bf16"
        self.metric_unit = "TFLOP/s"
        self.bound = "tensor"
        lb, ub = h.region(self.part, rank, 2)
        self.my_rows = ub[0] - lb[0]
        self.units = 2 * n ** 3 / 1e3  # GFLOP... scaled below
        self.alg_per_launch = 2.0 * self.my_rows * n * n
        self.my_pts = 0
        self.working_set = 3 * n * n * 2

    def step(self):
        self.h.apply(self.H.K_GEMM, self.part, self.acc, [1.0, 0.0])

    def reset_input(self):
        pass

    # end to end: pinned H2D of A and B, the product (incl. B's all-gather), D2H of C
    def e2e_setup(self, torch):
        self.hA = torch.from_numpy(self.Ab.view(np.int16)).pin_memory()
        self.hB = torch.from_numpy(self.Bb.view(np.int16)).pin_memory()
        self.hC = torch.empty((self.n, self.n), dtype=torch.float32).pin_memory()
        self.e2e_units = 2.0 * self.n ** 3
        rows = self.my_rows
        self.e2e_bytes = (2 * rows * self.n * 2, rows * self.n * 4)
        self.e2e_desc = "one job: hda_write A, B -> C = A @ B (B all-gathered) -> hda_read C (host wall clock, pinned)"

    def e2e_job(self):
        self.h.write_ptr(self.A, self.part, self.hA.data_ptr())
        self.h.write_ptr(self.B, self.part, self.hB.data_ptr())
        self.step()
        self.h.read_ptr(self.C, self.part, self.hC.data_ptr())

    def parity(self):
        got = self.h.read(self.C, self.part)
        lb, ub = self.h.region(self.part, self.rank, 2)
        rng = np.random.default_rng(7)
        ii = rng.integers(lb[0], ub[0], 64)
        jj = rng.integers(0, self.n, 64)
        A = synth.bf16_to_f32(self.Ab[ii]).astype(np.int64)
        exact = np.einsum("sk,ks->s", A, synth.bf16_to_f32(self.Bb[:, jj]).astype(np.int64))
        return {"integer_exact_samples": bool((got[ii, jj].astype(np.int64) == exact).all()), "samples": 64}


class TwoMM:
    """the 2MM chain D = A x B ; E = C x D (16384^2 bf16
    inputs, D bf16, E fp32) under a ROW or COL partition.  ROW re-gathers D every
    iteration (B once); COL moves A and C once and nothing afterwards (Table 3's
    1262.5 vs 25 GiB, P9).  One step = both products."""

    def __init__(self, H, h, rank, ws, n=None, part="row"):
        self.H, self.h, self.rank, self.ws = H, h, rank, ws
        self.n = n or 16384
        n = self.n
        S = H.STAR
        self.Ab, self.Bb, self.Cb = (synth.int_bf16(60 + i, (n, n), -1, 1) for i in range(3))
        self.A, self.B, self.C = (h.create(H.BF16, (n, n)) for _ in range(3))
        self.D = h.create(H.BF16, (n, n))
        self.E = h.create(H.F32, (n, n))
        self.part_name = part
        self.part = h.partition(H.ROW if part == "row" else H.COL, (n, n))
        for X, v in ((self.A, self.Ab), (self.B, self.Bb), (self.C, self.Cb)):
            h.write(X, self.part, v)
        self.acc1 = [(self.D, [], [(0, 0)]), (self.A, [(0, S)], []), (self.B, [(S, 0)], [])]
        self.acc2 = [(self.E, [], [(0, 0)]), (self.C, [(0, S)], []), (self.D, [(S, 0)], [])]
        self.kind = "2mm"
        self.workload = (f"SURVEY 8(f)-1 2MM chain (P:L425): D=AxB, E=CxD, {n}^2 bf16 in, D bf16, E fp32, "
                         f"{part.upper()} partition")
        self.kname = ("gemm2_kernel (tcgen05 cta_group::2), two products per step" if _env_int("HDA_GEMM_2SM", 1)
                      else "gemm_kernel (tcgen05), two products per step")
        self.dtype_name = "bf16"
        self.metric_unit = "TFLOP/s"
        self.flops_per_step = 4.0 * n ** 3
        self.bound = "tensor"
        lb, ub = h.region(self.part, rank, 2)
        self.lb, self.ub = lb, ub
        self.alg_per_launch = 2.0 * (ub[0] - lb[0]) * (ub[1] - lb[1]) * n
        self.my_pts = 0
        self.working_set = 6 * n * n * 2

    def step(self):
        self.h.apply(self.H.K_GEMM, self.part, self.acc1, [1.0, 0.0])
        self.h.apply(self.H.K_GEMM, self.part, self.acc2, [1.0, 0.0])

    def reset_input(self):
        pass

    def e2e_setup(self, torch):
        self.hin = [torch.from_numpy(v.view(np.int16)).pin_memory() for v in (self.Ab, self.Bb, self.Cb)]
        self.hE = torch.empty((self.n, self.n), dtype=torch.float32).pin_memory()
        self.e2e_units = self.flops_per_step
        cells = (self.ub[0] - self.lb[0]) * (self.ub[1] - self.lb[1])
        self.e2e_bytes = (3 * cells * 2, cells * 4)
        self.e2e_desc = "one job: hda_write A, B, C -> D = A @ B, E = C @ D -> hda_read E (host wall clock, pinned)"

    def e2e_job(self):
        for X, hx in zip((self.A, self.B, self.C), self.hin):
            self.h.write_ptr(X, self.part, hx.data_ptr())
        self.step()
        self.h.read_ptr(self.E, self.part, self.hE.data_ptr())

    def parity(self):
        """D sampled against the exact integer product rounded to bf16 (RNE); E sampled
        against the exact int64 product of C with the GPU's D (every partial sum is an
        integer below 2^24, so fp32 accumulation is exact in any order)."""
        D = self.h.read_replica(self.D, self.rank)
        E = self.h.read_replica(self.E, self.rank)
        rng = np.random.default_rng(11)
        ii = rng.integers(self.lb[0], self.ub[0], 64)
        jj = rng.integers(self.lb[1], self.ub[1], 64)
        A = synth.bf16_to_f32(self.Ab[ii]).astype(np.int64)
        exact = np.einsum("sk,ks->s", A, synth.bf16_to_f32(self.Bb[:, jj]).astype(np.int64))
        bits = exact.astype(np.float32).view(np.uint32)
        rne = ((bits + np.uint32(0x7FFF) + ((bits >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)).astype(np.uint16)
        d_ok = bool((D[ii, jj] == rne).all())
        Dv = synth.bf16_to_f32(D[:, jj]).astype(np.int64)
        e_exact = np.einsum("sk,ks->s", synth.bf16_to_f32(self.Cb[ii]).astype(np.int64), Dv)
        e_ok = bool((E[ii, jj].astype(np.int64) == e_exact).all())
        return {"D_bf16_rne_exact_samples": d_ok, "E_integer_exact_samples": e_ok, "samples": 64}


# ----------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=None)
    ap.add_argument("--impl", default="hdarray")
    ap.add_argument("--workload", default="jacobi2d",
                    choices=["jacobi2d", "stencil9", "stencil7", "repartition", "gemm", "2mm"])
    ap.add_argument("--part", default="row", choices=["row", "col"], help="2mm: ROW or COL partition")
    ap.add_argument("--size", "--n", dest="n", type=int, default=None,
                    help="problem edge (use --size under torchrun: its parser takes --n as its own prefix)")
    ap.add_argument("--watchdog", type=float, default=0.0,
                    help="dump every thread's Python stack and exit after this many seconds (debugging hangs)")
    ap.add_argument("--e2e-sweeps", type=int, default=100)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--transport", type=int, default=2, help="0 fused SM pull, 1 staged, 2 auto (default)")
    ap.add_argument("--no-overlap", action="store_true")
    ap.add_argument("--trace", type=int, default=0, help="trace N steps after the timed region")
    args = ap.parse_args()
    if args.watchdog > 0:
        import faulthandler
        faulthandler.dump_traceback_later(args.watchdog, exit=True)
    defaults = {"jacobi2d": (1000, 20), "stencil9": (200, 10), "stencil7": (100, 5), "repartition": (40, 4),
                "gemm": (20, 3), "2mm": (10, 3)}[args.workload]
    args.steps = args.steps or defaults[0]
    args.warmup = max(args.warmup if args.warmup is not None else defaults[1], 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_1809_05657_b200 as H

    ws, rank, local = dist_env()
    args.gpus = ws
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    hbm_peak, peak_src = peaks()
    if ws > 1:
        h = H.HDArray.spmd(ws, rank, local)
    else:
        h = H.HDArray(n_gpus=1, n_devices=1, gpu_ids=[local])
    h.set_transport(args.transport)
    h.set_overlap(not args.no_overlap)
    if args.workload in ("jacobi2d", "stencil9", "stencil7"):
        wl = Stencil(args.workload, H, h, rank, ws, args.n)
    elif args.workload == "repartition":
        wl = Repartition(H, h, rank, ws, args.n)
    elif args.workload == "2mm":
        wl = TwoMM(H, h, rank, ws, args.n, args.part)
    else:
        wl = Gemm(H, h, rank, ws, args.n)
    stream = torch.cuda.ExternalStream(h.stream(rank))

    def barrier():
        h.sync()
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()

    def reduce(x, op):
        if ws == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=op)
        return float(t.item())

    MAX = dist.ReduceOp.MAX if ws > 1 else None
    SUM = dist.ReduceOp.SUM if ws > 1 else None

    # L2 policy: inputs larger than L2 => back-to-back steps; otherwise flush between steps
    l2_bytes = torch.cuda.get_device_properties(local).L2_cache_size
    flush = wl.working_set < 2 * l2_bytes
    flush_buf = torch.empty(int(2 * l2_bytes), dtype=torch.uint8, device="cuda") if flush else None
    # after writing the flush buffer, READ a second one of 2x L2: the flush's dirty lines
    # are written back here, outside the timed step, instead of inside the next kernel
    flush_rd = torch.zeros(int(2 * l2_bytes) // 8, dtype=torch.int64, device="cuda") if flush else None

    for _ in range(args.warmup):
        wl.step()
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
        th0 = time.perf_counter()
        for _ in range(args.steps):
            wl.step()
        host_us = (time.perf_counter() - th0) / args.steps * 1e6
        ev1.record(stream)
        barrier()
        ms = ev0.elapsed_time(ev1)
    else:
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        host_us = None
        barrier()
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush_buf.zero_()
                flush_rd.max()
            if ws > 1:
                torch.cuda.synchronize()
                dist.barrier()
            # ~100 us of device sleep before the start event: the host issues the step
            # (tens of us) while the GPU sleeps, so the event pair brackets the device's
            # step as in the back-to-back mode, not the host's issue latency after an idle
            with torch.cuda.stream(stream):
                torch.cuda._sleep(200000)
            evs[i][0].record(stream)
            wl.step()
            evs[i][1].record(stream)
        barrier()
        ms = sum(a.elapsed_time(b) for a, b in evs)
    launches = h.stats()["kernel_launches"] - launches0
    clocks = clk.stop()
    st = h.stats()
    ms = reduce(ms, MAX)
    if wl.metric_unit == "GPoints/s":
        value = wl.units * args.steps / (ms * 1e-3) / 1e9
    elif wl.metric_unit == "GB/s":
        value = wl.units * args.steps / (ms * 1e-3) / 1e9
    else:
        value = getattr(wl, "flops_per_step", 2.0 * wl.n ** 3) * args.steps / (ms * 1e-3) / 1e12

    # ---- per-kernel timing pass (CUDA events bracketing each launch on its stream)
    h.set_kernel_timing(True)
    h.reset_stats()
    kt_steps = min(args.steps, 200)
    for _ in range(kt_steps):
        wl.step()
    barrier()
    kid = {"jacobi2d": H.K_JACOBI5, "stencil9": H.K_STENCIL9, "stencil7": H.K_STENCIL7_3D,
           "repartition": H.K_SCALE, "gemm": H.K_GEMM, "2mm": H.K_GEMM}[args.workload]
    k_ms, k_n = h.kernel_time(kid)
    x_ms, x_n = h.exchange_time()
    st_kt = h.stats()
    h.set_kernel_timing(False)
    k_avg = k_ms / max(k_n, 1)
    x_avg = x_ms / max(x_n, 1)
    halo_bytes = st_kt["bytes_total"] / max(kt_steps, 1)
    if wl.bound == "hbm" and args.workload != "repartition":
        achieved = wl.alg_per_launch / (k_avg * 1e-3) / 1e9
        roof = {"bound": "hbm", "kernel": wl.kname, "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": wl.alg_per_launch, "avg_launch_ms": k_avg}
    elif args.workload == "repartition":
        if ws > 1:
            achieved = wl.alg_per_launch / (x_avg * 1e-3) / 1e9  # bytes received per GPU / pull time
            roof = {"bound": "nvlink", "kernel": wl.kname, "achieved": achieved, "peak": NVLINK_GBS,
                    "unit": "GB/s", "frac": achieved / NVLINK_GBS, "scale_kernel_ms": k_avg,
                    "peak_source": "measured peer copy per direction (B200_PROFILING.md); 900 nominal",
                    "algorithmic_bytes_per_launch": wl.alg_per_launch, "avg_launch_ms": x_avg}
        else:
            scale_bytes = wl.n * wl.n * 4 * 2
            achieved = scale_bytes / (k_avg * 1e-3) / 1e9
            roof = {"bound": "hbm", "kernel": "scale_kernel<float>", "achieved": achieved, "peak": hbm_peak,
                    "unit": "GB/s", "frac": achieved / hbm_peak, "peak_source": peak_src,
                    "algorithmic_bytes_per_launch": scale_bytes, "avg_launch_ms": k_avg}
    else:
        burst, sustained = 1642.9, 1399.6
        try:
            mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
            burst, sustained = float(mp["bf16_tflops"]), float(mp["bf16_tflops_sustained"])
        except Exception:
            pass
        # the denominator is the measured cuBLAS burst figure (MEASURED_PEAKS.json, an 8192^3
        # torch.matmul); the CTA-pair kernel at 16384^3 can exceed it (frac > 1), so the
        # ratio to the nominal dense peak (2.25 PFLOP/s) rides along
        achieved = wl.alg_per_launch / (k_avg * 1e-3) / 1e12
        roof = {"bound": "tensor", "kernel": wl.kname, "achieved": achieved, "peak": burst, "unit": "TFLOP/s",
                "frac": achieved / burst, "frac_of_sustained": achieved / sustained,
                "frac_of_nominal_dense_2250": achieved / 2250.0,
                "peak_source": "measured cuBLAS bf16 burst (MEASURED_PEAKS.json); sustained 1399.6",
                "algorithmic_flops_per_launch": wl.alg_per_launch, "avg_launch_ms": k_avg}
    if ws > 1:
        roof["achieved_min_over_ranks"] = -reduce(-roof["achieved"], MAX)
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    roof["traffic"] = None
    if os.path.exists(tp):
        try:
            roof["traffic"] = json.load(open(tp)).get(f"{args.workload}_n{wl.n}_P{ws}")
        except Exception:
            pass

    # Stencils: take the roofline from the timed region itself (CUDA events on the
    # kernel's stream, max over ranks).  At N=1 a step is exactly one launch; at N>1 the
    # dominant (interior) launch runs concurrently with the pull and the boundary part,
    # so the per-GPU step time is its duration with the exchange included (conservative);
    # the event-bracketed pass, which serialises those parts, is kept for reference.
    if isinstance(wl, Stencil) and (ws > 1 or launches == args.steps):
        roof["avg_launch_ms_bracketed"] = roof["avg_launch_ms"]
        roof["avg_launch_ms"] = ms / args.steps
        roof["achieved"] = wl.alg_per_launch / (roof["avg_launch_ms"] * 1e-3) / 1e9
        roof["frac"] = roof["achieved"] / roof["peak"]
        roof["timing"] = ("timed region (one launch per step)" if ws == 1 else
                          "timed region (per-GPU step incl. the overlapped exchange)")
        if ws > 1:
            roof["achieved_min_over_ranks"] = roof["achieved"]  # ms is already the max over ranks
    if args.trace:
        barrier()
        h.set_trace(True)
        for _ in range(args.trace):
            wl.step()
        barrier()
        tr = h.trace()
        h.set_trace(False)
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        with open(os.path.join(ROOT, "gpurun_out", f"trace_{args.workload}_n{ws}_r{rank}.json"), "w") as f:
            json.dump(tr.tolist(), f)

    par = wl.parity()

    # context for the tensor roofline: cuBLAS (torch.matmul) on the same shape, same GPU
    cublas = None
    if isinstance(wl, (Gemm, TwoMM)) and ws == 1:
        a = torch.randn(wl.n, wl.n, device="cuda", dtype=torch.bfloat16)
        b = torch.randn(wl.n, wl.n, device="cuda", dtype=torch.bfloat16)
        for _ in range(3):
            torch.matmul(a, b)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        reps = 10
        for _ in range(reps):
            torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        cublas = 2.0 * wl.n ** 3 * reps / (e0.elapsed_time(e1) * 1e-3) / 1e12
        roof["cublas_same_shape_tflops"] = cublas
        del a, b

    # ---- end to end through the C-ABI with host buffers (stencils: write (pinned H2D)
    # -> e2e_sweeps sweeps -> read (D2H) per job)
    e2e = None
    if not args.no_e2e and isinstance(wl, Stencil):
        host_in = torch.from_numpy(np.ascontiguousarray(wl.u0)).pin_memory()
        host_out = torch.empty(wl.shape, dtype=host_in.dtype).pin_memory()
        times = []
        for j in range(3):
            barrier()
            t0 = time.perf_counter()
            h.write_ptr(wl.X, wl.data, host_in.data_ptr())
            wl.reset_input()
            for _ in range(args.e2e_sweeps):
                wl.step()
            h.read_ptr(wl.src, wl.data, host_out.data_ptr())
            barrier()
            if j:
                times.append(time.perf_counter() - t0)
        e2e_s = reduce(min(times), MAX)
        d_lb, d_ub = h.region(wl.data, rank, len(wl.shape))
        my_bytes = int(np.prod(np.subtract(d_ub, d_lb))) * wl.es
        e2e = {"value": wl.units * args.e2e_sweeps / e2e_s / 1e9, "unit": "GPoints/s",
               "h2d_bytes_per_step": int(reduce(my_bytes, SUM)), "d2h_bytes_per_step": int(reduce(my_bytes, SUM)),
               "step": f"one job: hda_write -> {args.e2e_sweeps} sweeps -> hda_read (host wall clock, pinned)"}

    elif not args.no_e2e and hasattr(wl, "e2e_job"):
        wl.e2e_setup(torch)
        times = []
        for j in range(3):
            barrier()
            t0 = time.perf_counter()
            wl.e2e_job()
            barrier()
            if j:
                times.append(time.perf_counter() - t0)
        e2e_s = reduce(min(times), MAX)
        scale = 1e12 if wl.metric_unit == "TFLOP/s" else 1e9
        e2e = {"value": wl.e2e_units / e2e_s / scale, "unit": wl.metric_unit,
               "h2d_bytes_per_step": int(reduce(wl.e2e_bytes[0], SUM)),
               "d2h_bytes_per_step": int(reduce(wl.e2e_bytes[1], SUM)), "step": wl.e2e_desc}

    launches = int(reduce(launches, SUM))
    if rank == 0:
        cpu = None
        if ws == 1 and not args.no_cpu_baseline and args.workload == "jacobi2d":
            cpu = oracle_sample()
        line = {
            "metric": METRIC, "value": value, "unit": wl.metric_unit, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": wl.dtype_name, "data": "synthetic",
            "config": {"workload": wl.workload, "n": wl.n, "parallelism": f"spmd{ws}" if ws > 1 else "single",
                       "transport": ["fused", "staged", "auto"][args.transport], "overlap": not args.no_overlap,
                       "l2": ("L2 flushed between timed steps (write a 2x-L2 buffer, then read another; each step is "
                              "queued behind a 100 us device sleep so its events bracket device time)" if flush else
                              f"inputs larger than L2 (per-GPU working set {wl.working_set / 2**20:.0f} MiB)")},
            **({"note": "one device: a repartition moves nothing (value 0); the roofline is the SCALE kernel's"}
               if args.workload == "repartition" and ws == 1 else {}),
            "roofline": roof,
            "exchange": {"bytes_per_step": halo_bytes, "exchange_ms_per_step": x_avg if x_n else 0.0,
                         "GBps_per_gpu": (halo_bytes / ws / (x_avg * 1e-3) / 1e9) if x_n else None,
                         "nvlink_peak_GBps": NVLINK_GBS},
            "parity": par,
            "tracker": {"plan_hits": st["plan_hits"], "plan_misses": st["plan_misses"],
                        "tracker_us_per_call": st["tracker_us"] / max(st["n_apply"], 1),
                        "host_issue_us_per_step": host_us},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    h.close()
    if ws > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
