#!/usr/bin/env python
"""Benchmark of the ARRABIT-MPM hot path on B200 (BASELINE.json metric:
"filtered SpMM HBM GB/s vs 8 TB/s peak; eigpairs/sec at 1/2/4/8 B200").

One STEP = one full fixed-parameter eig_solve (every §8(a) row: interval,
fused Chebyshev filter degrees + MPM normalisation, block-Krylov augmentation,
DMMA Gram/projection products, small eig, residuals) of the N=1 workload
BASELINE.json's metric is quoted on: configs[1] = cfg2, the 2-D 5-point
Laplacian 300x300 (n=90,000), k=200, d=20, p=1, tol=1e-10, X0 ~ N(0,1) seed 1.
value = eigenpairs/s = k * steps * N / (max-over-ranks device time).
The filter's HBM GB/s (the metric's first half) is the `roofline` object.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
N>1 (torchrun): each rank solves its own replica (no data-path collective).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402
from synth import configs  # noqa: E402

METRIC = "eigpairs/s (full ARRABIT-MPM solve to tol=1e-10); filtered SpMM HBM GB/s in roofline"
UNIT = "eigpairs/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def oracle_counts(cid):
    p = os.path.join(ROOT, "tests", "golden", f"oracle_cfg{cid}_counts.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def filter_bytes_per_degree(n, nnz, w, d):
    """Algorithmic bytes of one filter-degree launch: A once
    (12 nnz + 8(n+1)), read Y_j, read Y_{j-1}, write Y_{j+1} (24 n w); the first
    degree has no Y_{j-1} (16 n w).  Averaged over the d launches of a sweep."""
    a = 12 * nnz + 8 * (n + 1)
    return (a + 16 * n * w + (d - 1) * (a + 24 * n * w)) / d


# ------------------------------------------------------------------ oracle arm
def oracle_sample(A, spec, X0):
    """One bounded sample of the workload on the CPU oracle: one MPM sweep
    (d degrees + normalisation) and one ARR + residual pass, from X0."""
    import oracle
    a = oracle.gershgorin_lower(A)
    mu0, _, _ = oracle.rayleigh_ritz(A, X0)
    b = float(mu0[spec.w - 1])
    t0 = time.perf_counter()
    X = oracle.mpm_sweep(A, a, b, spec.d, X0)
    t1 = time.perf_counter()
    mu, Y, _ = oracle.arr(A, X, spec.p)
    oracle.residuals(A, Y[:, :spec.k], mu[:spec.k])
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    A, spec = configs.build_config(args.config)
    X0 = synth.starting_block(spec)
    cnt = oracle_counts(args.config)
    S, O = (cnt["sweeps"], cnt["outer"]) if cnt else (38, 10)
    for _ in range(args.warmup):
        oracle_sample(A, spec, X0)
    sw, ar, wall = [], [], []
    for _ in range(args.steps):
        t = time.perf_counter()
        s, r = oracle_sample(A, spec, X0)
        wall.append(time.perf_counter() - t)
        sw.append(s)
        ar.append(r)
    t_solve = S * statistics.mean(sw) + O * statistics.mean(ar)
    value = spec.k / t_solve
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count()))
    sample = (f"{spec.name}: per step one MPM sweep (d={spec.d}) + one ARR(p={spec.p}) + residuals on the full "
              f"block; extrapolated to the oracle's own full solve ({S} sweeps, {O} ARR steps, "
              f"tests/golden/oracle_cfg{args.config}_counts.json)")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000 * statistics.mean(wall), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": spec.name, "n": A.n, "nnz": A.nnz, "k": spec.k, "d": spec.d, "p": spec.p,
                       "tol": spec.tol},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_1507_06078_b200 as arr

    A, spec = configs.build_config(args.config)
    X0h = synth.starting_block(spec)
    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        Ad = arr.to_device_csr(A, device=dev)
        X0 = torch.from_numpy(X0h).to(dev)
        X = torch.empty_like(X0)
        flush = torch.empty(256 * 2 ** 20 // 8, dtype=torch.float64, device=dev)  # > 126 MB L2
    stream.synchronize()
    ctx = arr.eig_init(Ad, spec.k, spec.p, spec.d, stream=stream, w=spec.w)

    def one_solve():
        X.copy_(X0)
        return ctx.eig_solve(X, tol=spec.tol, maxit=spec.maxit, s_max=spec.s_max)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            ev, res, info = one_solve()
    ctx.eig_set_timing(True)
    launches0 = ctx.launch_count
    sampler = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    sampler.start()
    step_ms = []
    infos = []
    with torch.cuda.stream(stream):
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ev, res, info = one_solve()
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            infos.append((info.converged, info.outer, info.sweeps, info.maxres))
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    launches = ctx.launch_count - launches0
    phase_ms, phase_cnt = ctx.eig_phase_times()
    total_ms = float(sum(step_ms))
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = spec.k * args.steps * world / (total_ms / 1000.0)

    # roofline of the dominant kernel (filter degree)
    peak, peak_src = load_peaks()
    deg_ms = phase_ms[0] / max(1, phase_cnt[0])
    bpl = filter_bytes_per_degree(A.n, A.nnz, spec.w, spec.d)
    achieved = bpl / (deg_ms / 1000.0) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"ncu_traffic_cfg{args.config}.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                traffic = json.load(f).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": "spmm_fused_kernel (one Chebyshev filter degree)",
                "bytes_per_launch": bpl, "avg_launch_us": deg_ms * 1000.0, "launches": int(phase_cnt[0]),
                "peak_source": peak_src,
                "share_of_step": phase_ms[0] / total_ms if world == 1 else None,
                "phase_ms_per_step": {"filter_degrees": phase_ms[0] / args.steps, "arr_project": phase_ms[1] / args.steps,
                                      "arr_basis": phase_ms[3] / args.steps, "arr_H": phase_ms[4] / args.steps,
                                      "arr_small_eig": phase_ms[5] / args.steps,
                                      "residuals": phase_ms[2] / args.steps}}

    # e2e through the host-buffer C-ABI entry (H2D inputs + D2H eigenpairs inside the timed region)
    e2e = None
    if not args.no_e2e:
        rp = torch.from_numpy(A.row_ptr).pin_memory()
        ci = torch.from_numpy(A.col_idx).pin_memory()
        va = torch.from_numpy(A.val).pin_memory()
        x0p = torch.from_numpy(X0h).pin_memory()
        evec = torch.empty((A.n, spec.k), dtype=torch.float64).pin_memory()
        e2e_s = []
        for _ in range(max(1, args.steps)):
            torch.cuda.synchronize(dev)
            t = time.perf_counter()
            arr.eig_solve_host(A.n, rp, ci, va, spec.k, spec.p, spec.d, x0p, tol=spec.tol, maxit=spec.maxit,
                               s_max=spec.s_max, evec=evec, stream=stream)
            e2e_s.append(time.perf_counter() - t)
        tot = float(sum(e2e_s))
        if world > 1:
            t = torch.tensor([tot], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tot = float(t.item())
        e2e = {"value": spec.k * len(e2e_s) * world / tot, "unit": UNIT,
               "h2d_bytes_per_step": int(8 * (A.n + 1) + 12 * A.nnz + 8 * A.n * spec.w),
               "d2h_bytes_per_step": int(16 * spec.k + 8 * A.n * spec.k),
               "api": "eig_solve_host (C-ABI, pinned host buffers, device alloc + copies inside)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cnt = oracle_counts(args.config)
        S, O = (cnt["sweeps"], cnt["outer"]) if cnt else (infos[-1][2], infos[-1][1])
        ts, ta = oracle_sample(A, spec, X0h)
        cpu = {"value": spec.k / (S * ts + O * ta), "unit": UNIT,
               "cores": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count())), "kind": "oracle",
               "sample": f"one MPM sweep ({ts:.2f} s) + one ARR+residuals ({ta:.2f} s) of {spec.name}, "
                         f"extrapolated to {S} sweeps / {O} ARR steps "
                         f"({'oracle full-solve counts, tests/golden' if cnt else 'GPU solve counts'})"}

    if rank == 0:
        conv, outer, sweeps, maxres = infos[-1]
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": spec.name, "n": A.n, "nnz": A.nnz, "k": spec.k, "w": spec.w, "d": spec.d,
                           "p": spec.p, "tol": spec.tol, "step": "one full eig_solve from X0",
                           "l2": "flushed between timed steps (256 MiB write), outside the events",
                           "parallelism": "1 GPU" if world == 1 else f"{world} independent replicas (no collective)",
                           "converged": bool(conv), "outer": outer, "sweeps": sweeps, "maxres": maxres},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
                "clocks": clocks}
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
