#!/usr/bin/env python
"""Benchmark of the ARRABIT-MPM hot path on B200 (BASELINE.json metric:
"filtered SpMM HBM GB/s vs 8 TB/s peak; eigpairs/sec at 1/2/4/8 B200").

One STEP = one full fixed-parameter eig_solve (every §8(a) row: interval,
fused Chebyshev filter degrees + MPM normalisation, block-Krylov augmentation,
DMMA Gram/projection products, small eig, residuals) of the workload the
metric's "1/2/4/8 B200" is quoted on: BASELINE.json configs[2] = cfg3, the 3-D
7-point Laplacian 100^3 + diag(U[0,1)) (n = 1e6), k = 500 (w = 550), d = 20, p = 2,
tol = 1e-10, seed 2 (--config selects another).  The 3-D grids run the stencil-aware
filter path (eig_set_stencil; DIA + TMA-staged 2.5-D kernel), others the CSR kernels.
value = eigenpairs/s = k * steps / (max-over-ranks device time).
`roofline` is the dominant kernel of the timed steps (largest share of device time:
at cfg3 the FP64 DMMA Gram, vs the measured DGEMM peak); `roofline.kernels` holds the
other classes, among them the filter's HBM GB/s (the metric's first half).  A shorter
cfg2 solve (BASELINE.json configs[1]) is reported beside it as `secondary`.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
N>1 (torchrun): the config is row-partitioned over the ranks (z-slabs / balanced
blocks; halo or all-gather exchange before every SpMM and Gram allreduce over NCCL
inside libarrabit; strong scaling; on the grids every rank declares its z-slab and runs
the stencil kernel with the neighbouring planes as ghost planes); --replicas runs
independent copies instead.
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
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--spmm", default="auto", choices=["auto", "csr", "stencil"],
                    help="filter kernels: auto = the stencil path for 3-D grids, CSR otherwise")
    ap.add_argument("--no-secondary", action="store_true", help="skip the secondary cfg2 solve")
    ap.add_argument("--replicas", action="store_true", help="N>1: independent replicas instead of a partition")
    ap.add_argument("--partition", default="rows", choices=["rows", "column"],
                    help="N>1: rows = row partition (halo / all-gather before every SpMM); column = the column split "
                         "(eig_init_colsplit: A replicated, column-local filter, ARR on a row partition)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--filter", default="cheb", choices=["cheb", "interp"],
                    help="cheb: T_d (default); interp: the paper's interpolant psi_d (Section 5)")
    ap.add_argument("--adapt", type=int, default=0,
                    help="the paper's adaptive options (bit mask: 1 p, 2 d, 4 continuation + deflation)")
    ap.add_argument("--inner-solver", default="mpm", choices=["mpm", "gn"],
                    help="inner solver of Alg. Arrabit2: mpm (default) or gn (Gauss-Newton)")
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


def filter_bytes_per_degree(n, nnz, w, d, abytes=None):
    """Algorithmic bytes of one filter-degree launch: A once, read Y_j,
    read Y_{j-1}, write Y_{j+1} (24 n w); the first degree has no Y_{j-1} (16 n w).
    A is 12 nnz + 8(n+1) bytes as CSR; on the stencil path `abytes` per row (8 K for the
    K diagonals, 8 for the diagonal of a constant-off-diagonal operator, 0 when every
    coefficient is constant: eig_stencil_abytes).  Averaged over the d launches of a sweep."""
    a = abytes * n if abytes is not None and abytes >= 0 else 12 * nnz + 8 * (n + 1)
    return (a + 16 * n * w + (d - 1) * (a + 24 * n * w)) / d


def stencil_grid(spec):
    """The grid a config's operator is declared on for the stencil path (x fastest);
    a 2-D grid is declared (nx, 1, ny) so that the march runs along y."""
    if spec.kind == "lap1d":
        return (spec.size, 1, 1)
    if spec.kind == "lap2d":
        return (spec.size, 1, spec.size)
    if spec.kind in ("lap3dV", "st27"):
        return (spec.size, spec.size, spec.size)
    return None


def use_stencil(spec, args):
    if args.spmm == "csr" or stencil_grid(spec) is None:
        return False
    return args.spmm == "stencil" or spec.kind in ("lap1d", "lap2d", "lap3dV", "st27")


def config_dict(spec, A, args):
    """The workload (identical in both arms)."""
    return {"workload": spec.name, "n": int(A.n), "nnz": int(A.nnz), "k": spec.k, "w": spec.w, "d": spec.d,
            "p": spec.p, "tol": spec.tol, "seed": spec.seed, "step": "one full eig_solve from X0",
            "filter": {"cheb": "T_d (Eq. cheby-poly)", "interp": "psi_d (paper Section 5)"}[args.filter],
            "adapt": args.adapt, "inner_solver": args.inner_solver,
            "l2": "flushed between timed steps (256 MiB write), outside the events"}


def cpu_info():
    info = {"model": None, "sockets": None, "logical_cpus": os.cpu_count(), "ram_gb": None}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            k, _, v = ln.partition(":")
            if k.strip() == "Model name":
                info["model"] = v.strip()
            elif k.strip() == "Socket(s)":
                info["sockets"] = int(v.strip())
            elif k.strip() == "Core(s) per socket":
                info["cores_per_socket"] = int(v.strip())
    except Exception:
        pass
    try:
        with open("/proc/meminfo") as f:
            kb = int(f.readline().split()[1])
        info["ram_gb"] = round(kb / 2 ** 20, 1)
    except Exception:
        pass
    return info


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


def oracle_filter_sample(A, spec, cols=16):
    """Seconds of one oracle MPM sweep on `cols` columns of the workload."""
    import oracle
    X = synth.gaussian_block_rows(A.n, cols, spec.seed, 0, A.n)
    a = oracle.gershgorin_lower(A)
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    upper = float(np.bincount(rows, weights=np.abs(A.val), minlength=A.n).max())
    t0 = time.perf_counter()
    oracle.mpm_sweep(A, a, a + 0.9 * (upper - a), spec.d, X)
    return time.perf_counter() - t0


def oracle_step_estimate(A, spec, cid):
    """Oracle seconds for one full solve of the workload, from a bounded sample:
    cfg 1-2: one sweep + one ARR of the full block, times the oracle's own counts
    (tests/golden/oracle_cfg<N>_counts.json); larger configs: a 16-column sweep x w/16
    times the sweep count of the oracle's golden solve when there is one (ARR not
    sampled: the oracle's ARR at these widths takes minutes)."""
    cnt = oracle_counts(cid)
    if cid <= 2:
        S, O = (cnt["sweeps"], cnt["outer"]) if cnt else (38, 10)
        ts, ta = oracle_sample(A, spec, configs.starting_block(spec))
        smp = (f"{spec.name}: one MPM sweep (d={spec.d}, {ts:.2f} s) + one ARR(p={spec.p}) + residuals "
               f"({ta:.2f} s) on the full block, extrapolated to the oracle's own full solve ({S} sweeps, {O} ARR)")
        return S * ts + O * ta, smp
    gold = oracle_golden(cid)
    import oracle
    # the golden solve's sweep count when it ran under the current sweeps rule (R6);
    # else the count of the GPU solve under the same rule (profiles/r02: cfg3 18, cfg5 56)
    same_rule = bool(gold) and float(gold.get("range_digits", 8.0)) == float(oracle.RANGE_DIGITS)
    gpu_counts = {3: 18, 5: 56}
    S = gold["sweeps"] if same_rule else gpu_counts.get(cid, 24)
    src = ("the oracle golden solve" if same_rule else
           "the GPU solve's count under the same sweeps rule" if cid in gpu_counts else "assumed")
    ts = oracle_filter_sample(A, spec) * spec.w / 16
    smp = (f"{spec.name}: one MPM sweep of 16 of the {spec.w} columns ({ts * 16 / spec.w:.2f} s) x w/16, "
           f"extrapolated to {S} sweeps ({src}); ARR not sampled")
    return S * ts, smp


def oracle_golden(cid):
    p = os.path.join(ROOT, "tests", "golden", f"oracle_cfg{cid}_eigs.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return None


def single_thread_leg(cid):
    """The same oracle sample with OMP / BLAS threads pinned to 1 (a subprocess, since
    the thread count is fixed when the libraries load)."""
    env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1")
    code = ("import sys, json; sys.path.insert(0, %r); import bench; from synth import configs; "
            "A, spec = configs.build_config(%d); t, s = bench.oracle_step_estimate(A, spec, %d); "
            "print(json.dumps({'seconds': t, 'sample': s}))") % (ROOT, cid, cid)
    try:
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
        return json.loads(out.stdout.strip().splitlines()[-1])
    except Exception as exc:  # noqa: BLE001
        return {"error": str(exc)[:200]}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    A, spec = configs.build_config(args.config)
    for _ in range(args.warmup):
        oracle_step_estimate(A, spec, args.config)
    est, wall = [], []
    smp = ""
    for _ in range(args.steps):
        t = time.perf_counter()
        e, smp = oracle_step_estimate(A, spec, args.config)
        wall.append(time.perf_counter() - t)
        est.append(e)
    value = spec.k / statistics.mean(est)
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count()))
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000 * statistics.mean(wall), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference", "parallelism": f"CPU oracle, {cores} host threads",
            "config": config_dict(spec, A, args),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": smp,
                             "cpu": cpu_info()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def _partition_spec(spec):
    """How a config is row-partitioned over ranks: z-slabs of
    whole grid planes for the stencils, nnz-balanced row blocks otherwise."""
    if spec.kind in ("lap3dV", "st27"):
        return ("planes", spec.size, spec.size ** 2)
    if spec.kind == "lap2d":
        return ("planes", spec.size, spec.size)
    return ("balanced",)


def solve_run(arr, torch, spec, A, Aloc, X0, X, flush, stream, dev, args, steps, warmup, plan=None, comm=None,
              world=1, dist=None):
    """Create a context, run warm-up + timed solves; return measurements."""
    partitioned = plan is not None
    if isinstance(plan, arr.partition.ColSplitPlan):
        ctx = arr.eig_init_colsplit(Ad_of(arr, A, dev, stream), Ad_of(arr, plan.rows, dev, stream), plan, spec.k,
                                    spec.p, spec.d, spec.w, comm, stream=stream)
        partitioned = False  # the column context has the whole A: the stencil path applies
    else:
        ctx = arr.eig_init(Ad_of(arr, Aloc, dev, stream), spec.k, spec.p, spec.d, stream=stream, w=spec.w, comm=comm,
                           plan=plan)
    nrows = X.shape[0]
    ctx_lean = ctx.workspace_bytes < 8 * nrows * spec.w * (spec.p + 2)
    if args.filter != "cheb":
        ctx.eig_set_filter(args.filter)
    path = "csr"
    if not partitioned and use_stencil(spec, args):
        ctx.eig_set_stencil(*stencil_grid(spec))
        path = f"stencil ({ctx.stencil_points}-point, A {ctx.stencil_abytes} B/row)"
    elif partitioned and use_stencil(spec, args) and _partition_spec(spec)[0] == "planes":
        # z-slab of whole grid planes: the stencil kernel with the neighbouring planes as ghost
        # planes (interior planes during the halo exchange, then the slab's first / last plane)
        ps_ = _partition_spec(spec)
        slab = ((ps_[2] // ps_[1], ps_[1], plan.n_own // ps_[2]) if spec.kind != "lap2d"
                else (ps_[2], 1, plan.n_own // ps_[2]))
        ctx.eig_set_stencil(*slab)
        path = f"stencil on z-slabs ({ctx.stencil_points}-point, A {ctx.stencil_abytes} B/row, slab {slab})"
    elif not partitioned and spec.kind in ("lap3dV", "st27"):
        from paper_1507_06078_b200 import schedule
        by, tile = {"lap3dV": (10, 16), "st27": (8, 32)}[spec.kind]
        ctx.eig_set_schedule(*schedule.yband_3d(spec.size, spec.size, spec.size, by, tile))
        path = f"csr, y-band order by={by}, {tile}-row tiles"

    def one_solve():
        return ctx.eig_solve(X, tol=spec.tol, maxit=spec.maxit, s_max=spec.s_max, adapt=args.adapt,
                             inner_solver=args.inner_solver)

    with torch.cuda.stream(stream):
        for _ in range(warmup):
            X.copy_(X0, non_blocking=True)
            one_solve()
    ctx.eig_set_timing(True)
    launches0 = ctx.launch_count
    sampler = ClockSampler(dev.index)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    sampler.start()
    step_ms, infos = [], []
    with torch.cuda.stream(stream):
        for _ in range(steps):
            X.copy_(X0, non_blocking=True)  # X <- X0 (outside the events)
            flush.zero_()  # L2 flush between timed steps (outside the events)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ev, res, info = one_solve()
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            infos.append(info)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    launches = ctx.launch_count - launches0
    phase_ms, phase_cnt = ctx.eig_phase_times()
    kern_ms, kern_flops, kern_cnt = ctx.eig_kernel_times()  # the DMMA Gram / GEMM kernels alone
    # the kernel the filter degrees launch (one more filter_step, outside the timed region)
    with torch.cuda.stream(stream):
        ctx.eig_set_interval(infos[-1].a, infos[-1].b)
        ctx.filter_step(X, normalize=True)
    kernel = ctx.last_spmm_kernel
    return dict(ctx=ctx, step_ms=step_ms, infos=infos, clocks=clocks, launches=launches, phase_ms=phase_ms,
                phase_cnt=phase_cnt, kern_ms=kern_ms, kern_flops=kern_flops, kern_cnt=kern_cnt, kernel=kernel, path=path, lean=ctx_lean, stencil_K=ctx.stencil_points,
                stencil_abytes=ctx.stencil_abytes if ctx.stencil_points else None,
                eigenvalues=ev)


_AD = {}


def Ad_of(arr, Aloc, dev, stream):
    key = id(Aloc)
    if key not in _AD:
        import torch
        with torch.cuda.stream(stream):
            _AD[key] = arr.to_device_csr(Aloc, device=dev)
        stream.synchronize()
    return _AD[key]


def load_fp64_peak():
    """The FP64 tensor (DMMA) peak: cuBLAS DGEMM 8192^3 measured on this pool's B200
    (profiles/peaks_fp64.json; the sustained figure for kernels timed inside a long step)."""
    pp = os.path.join(ROOT, "profiles", "peaks_fp64.json")
    try:
        with open(pp) as f:
            pk = json.load(f)
        return float(pk["fp64_dgemm_tflops_sustained"]), "profiles/peaks_fp64.json (cuBLAS DGEMM 8192^3, back to back, measured)"
    except Exception:
        return None, None


def _traffic(cid, family):
    tp = os.path.join(ROOT, "profiles", f"ncu_traffic_{family}_cfg{cid}.json" if family in ("gram", "gemm")
                      else f"ncu_traffic_cfg{cid}.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                tj = json.load(f)
            return tj, tj.get("dram_bytes_per_launch"), tj.get("source")
        except Exception:
            pass
    return None, None, None


def roofline_of(r, spec, nrow, nnz, args, steps, cid=None, w=None):
    """The roofline of the DOMINANT kernel of the timed steps (largest share of the step's
    device time, per-launch CUDA events on the context stream) plus the other two kernel
    classes of the path: the filter degree (HBM-bound; BJ's metric), the DMMA Gram and the
    DMMA GEMM (FP64-tensor-bound)."""
    cid = args.config if cid is None else cid
    peak, peak_src = load_peaks()
    w = spec.w if w is None else w  # the filtered width on this rank (the column split filters w_r columns)
    deg_ms = r["phase_ms"][0] / max(1, r["phase_cnt"][0])
    bpl = filter_bytes_per_degree(nrow, nnz, w, spec.d, r["stencil_abytes"])
    if args.filter == "interp":  # Clenshaw steps also read X (the a_k X term): + 8 n w per degree
        bpl += 8 * nrow * w
    achieved = bpl / (deg_ms / 1000.0) / 1e9
    tj, traffic, traffic_src = _traffic(cid, "filter")
    if tj is not None and not (tj.get("kernel_family", "") and tj["kernel_family"] in r["kernel"]):
        traffic, traffic_src = None, None
    pm, st = r["phase_ms"], sum(r["step_ms"])
    filt = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "traffic_source": traffic_src, "kernel": r["kernel"],
            "bytes_per_launch": bpl, "bytes_model": (
                {None: "12 nnz + 8(n+1)", 0: "0 (all coefficients constant)", 8: "8 n (diagonal; constant off-diagonals)"}.get(
                    r["stencil_abytes"], "8 K n (K diagonals)") + " + 24 n w (16 n w on a sweep's first degree)"),
            "avg_launch_us": deg_ms * 1000.0, "launches": int(r["phase_cnt"][0]), "peak_source": peak_src,
            "frac_of_8TBs": achieved / 8000.0, "share_of_step": pm[0] / st}
    pk64, pk64_src = load_fp64_peak()
    dmma = {}
    for i, (name, kern) in enumerate((("dmma_gram", "gram_kernel_pv (FP64 DMMA m8n8k4, X^T Y split over rows)"),
                                      ("dmma_gemm", "gemm_kernel_ca (FP64 DMMA m8n8k4, X B)"))):
        ms, fl, cnt = float(r["kern_ms"][i]), float(r["kern_flops"][i]), int(r["kern_cnt"][i])
        if cnt == 0 or ms <= 0:
            continue
        ach = fl / (ms / 1e3) / 1e12
        o = {"bound": "tensor", "achieved": ach, "peak": pk64, "unit": "TFLOP/s",
             "frac": ach / pk64 if pk64 else None, "traffic": None, "kernel": kern,
             "flops_per_launch": fl / cnt, "flops_model": "2 n m1 m2 (symmetric Gram n m (m+1); upper-triangular B "
             "2 n sum_c min(c+1, m1)), summed over the step's launches of every shape",
             "avg_launch_us": ms * 1e3 / cnt, "launches": cnt, "peak_source": pk64_src, "share_of_step": ms / st}
        tj, tr, ts = _traffic(cid, name[5:])  # profiles/ncu_traffic_{gram,gemm}_cfg<N>.json
        if tj is not None:
            o["traffic"], o["traffic_source"] = tr, ts
            o["traffic_note"] = "mean DRAM bytes per launch over the launches of one ARR (ncu --set full)"
        dmma[name] = o
    kinds = {"filter": filt, **dmma}
    dom = max(kinds, key=lambda k: kinds[k]["share_of_step"])
    out = dict(kinds[dom])
    out["dominant"] = dom
    out["dominant_by"] = "largest share of the timed steps' device time (CUDA events per launch on the context stream)"
    out["kernels"] = {k: v for k, v in kinds.items() if k != dom}
    out["phase_ms_per_step"] = {"filter_degrees": pm[0] / steps, "arr_project": pm[1] / steps,
                                "arr_basis": pm[3] / steps, "arr_H": pm[4] / steps, "arr_small_eig": pm[5] / steps,
                                "residuals": pm[2] / steps}
    return out


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
    from paper_1507_06078_b200 import partition as pt

    A, spec = configs.build_config(args.config)
    partitioned = world > 1 and not args.replicas
    plan = comm = None
    colsplit = partitioned and args.partition == "column"
    c0, c1 = 0, spec.w
    if colsplit:
        plan = pt.colsplit_plan(A, spec.w, world, rank)
        Aloc = A
        c0, c1 = plan.col_range
        r0, r1, nrows = 0, A.n, A.n
    elif partitioned:
        ps = _partition_spec(spec)
        bounds = pt.bounds_planes(ps[1], ps[2], world) if ps[0] == "planes" else pt.bounds_balanced(A.row_ptr, world)
        # 3-D grids: each rank's interior tiles in y-band order (the row order the CSR kernels
        # run on one GPU without the stencil path; results unchanged)
        yband = (spec.size, spec.size, {"lap3dV": 10, "st27": 8}[spec.kind]) if spec.kind in ("lap3dV", "st27") else None
        plan = pt.local_plan(A, bounds, rank, yband=yband)
        Aloc = plan
        r0, r1 = plan.row_begin, plan.row_begin + plan.n_own
        nrows = plan.n_rows_block
    else:
        Aloc = A
        r0, r1, nrows = 0, A.n, A.n

    def host_X0():
        X = np.zeros((nrows, spec.w))
        X[:r1 - r0, :spec.k] = synth.gaussian_block_rows(A.n, spec.k, spec.seed, r0, r1)
        if spec.q:
            X[:r1 - r0, spec.k:] = synth.gaussian_block_rows(A.n, spec.q, spec.seed, r0, r1, stream=2)
        return np.ascontiguousarray(X[:, c0:c1]) if colsplit else X

    X0h = host_X0()
    stream = torch.cuda.Stream(device=dev)
    # X0 stays on the device unless the solve's blocks would not fit next to it (cfg5 on
    # one GPU: X + the (p+1)-block basis is ~151 GB); then it is re-uploaded from pinned
    # host memory before each step, outside the timed region
    blk = 8 * nrows * (c1 - c0)
    x0_on_host = blk * (spec.p + 4) > 0.9 * torch.cuda.get_device_properties(dev).total_memory
    # the solve's block X with 128-byte rows (leading dimension rounded up to 16 doubles, the
    # layout eig_solve_host and the library's own blocks use: TMA boxes and 16-byte vectors
    # start on sector boundaries)
    ldp = (X0h.shape[1] + 15) // 16 * 16

    def padded(rows, cols):
        return torch.empty((rows, ldp), dtype=torch.float64, device=dev)[:, :cols]

    with torch.cuda.stream(stream):
        if x0_on_host:
            X0 = torch.from_numpy(X0h).pin_memory()
            X = padded(*X0.shape)
        else:
            X0 = padded(*X0h.shape)
            X0.copy_(torch.from_numpy(X0h).to(dev))
            X = padded(*X0.shape)
        flush = torch.empty(256 * 2 ** 20 // 8, dtype=torch.float64, device=dev)  # > 126 MB L2
    stream.synchronize()
    if partitioned:
        comm = arr.Comm.from_torch_distributed()
    r = solve_run(arr, torch, spec, A, Aloc, X0, X, flush, stream, dev, args, args.steps, args.warmup, plan=plan,
                  comm=comm, world=world, dist=dist)
    ctx = r["ctx"]
    total_ms = float(sum(r["step_ms"]))
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    # eigenpairs/s: each replica (or the one partitioned job) finds k pairs per step
    jobs = 1 if partitioned else world
    value = spec.k * args.steps * jobs / (total_ms / 1000.0)
    nnz_loc = int(Aloc.nnz) if (not partitioned or colsplit) else plan.nnz
    roofline = roofline_of(r, spec, r1 - r0, nnz_loc, args, args.steps, w=c1 - c0)

    # the DMMA Gram kernel of A4 (X^T Y, n x w by n x w, 2 n w^2 flops) timed alone on this block
    dense = None
    try:
        if colsplit:
            raise RuntimeError("gram is not exported on a column-split context")
        G = torch.empty((spec.w, spec.w), dtype=torch.float64, device=dev)
        nrow = r1 - r0
        with torch.cuda.stream(stream):
            Y2 = X0 if not x0_on_host else X  # second operand (X^T X when X0 is on the host)
            for _ in range(3):
                ctx.gram(Y2[:nrow], X[:nrow], G)
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 10
            ev0.record(stream)
            for _ in range(reps):
                ctx.gram(Y2[:nrow], X[:nrow], G)
            ev1.record(stream)
            ev1.synchronize()
        gms = ev0.elapsed_time(ev1) / reps
        fl = 2.0 * nrow * spec.w * spec.w * (0.5 if x0_on_host else 1.0)  # symmetric Gram: upper half
        pk = None
        pp = os.path.join(ROOT, "profiles", "peaks_fp64.json")
        if os.path.exists(pp):
            with open(pp) as f:
                pk = json.load(f).get("fp64_dgemm_tflops_burst")
        dense = {"bound": "tensor (FP64 DMMA)", "kernel": "gram_kernel + gram_reduce_kernel (X^T Y, n x w)",
                 "achieved": fl / (gms / 1e3) / 1e12, "unit": "TFLOP/s", "peak": pk,
                 "frac": (fl / (gms / 1e3) / 1e12 / pk) if pk else None,
                 "peak_source": "profiles/peaks_fp64.json (cuBLAS DGEMM 8192^3, measured)" if pk else None,
                 "avg_launch_us": gms * 1e3, "flops_per_launch": fl}
    except Exception as e:  # noqa: BLE001
        dense = {"error": str(e)}
    roofline["gram_timed_alone"] = dense
    if spec.kind == "zipf":
        roofline["gather_model_bytes_per_launch"] = (12 * nnz_loc + 8 * (r1 - r0 + 1) + 8 * nnz_loc * spec.w
                                                     + 16 * (r1 - r0) * spec.w)
    ctx.close()
    Y2 = G = None  # the dense-Gram measurement held X (or X0)
    del X, X0, Y2, G
    _AD.clear()
    torch.cuda.empty_cache()

    # secondary: the BASELINE.json configs[1] workload (cfg2), a short solve on one GPU
    secondary = None
    if world == 1 and not args.no_secondary and args.config != 2:
        try:
            A2, spec2 = configs.build_config(2)
            with torch.cuda.stream(stream):
                x02 = torch.from_numpy(configs.starting_block(spec2)).to(dev)
                ld2 = (x02.shape[1] + 15) // 16 * 16  # 128-byte rows, as for the main workload
                X02 = torch.empty((x02.shape[0], ld2), dtype=torch.float64, device=dev)[:, :x02.shape[1]]
                X02.copy_(x02)
                X2 = torch.empty((x02.shape[0], ld2), dtype=torch.float64, device=dev)[:, :x02.shape[1]]
                del x02
            args2 = argparse.Namespace(**vars(args))
            args2.config = 2
            r2 = solve_run(arr, torch, spec2, A2, A2, X02, X2, flush, stream, dev, args2, 3, 2)
            tot2 = float(sum(r2["step_ms"]))
            i2 = r2["infos"][-1]
            secondary = {"workload": spec2.name, "value": spec2.k * 3 / (tot2 / 1e3), "unit": UNIT,
                         "ms_per_step": tot2 / 3, "steps": 3, "warmup": 2, "spmm_path": r2["path"],
                         "converged": bool(i2.converged), "outer": i2.outer, "sweeps": i2.sweeps,
                         "maxres": i2.maxres, "roofline": roofline_of(r2, spec2, A2.n, A2.nnz, args2, 3),
                         "clocks": r2["clocks"]}
            r2["ctx"].close()
            del X2, X02
            _AD.clear()
            torch.cuda.empty_cache()
        except Exception as exc:  # noqa: BLE001
            secondary = {"error": str(exc)[:200]}

    # e2e through the public API with HOST buffers: H2D of the CSR + X0 and D2H of the
    # eigenpairs inside the timed region (one GPU: the eig_solve_host C-ABI call;
    # partitioned: each rank uploads its local CSR + X0 rows, eig_init_dist, eig_solve)
    e2e = None
    if not args.no_e2e and colsplit:
        e2e = {"value": None, "unit": UNIT, "error": "no host-buffer entry for the column split"}
    elif not args.no_e2e and (args.filter != "cheb" or args.adapt or args.inner_solver != "mpm"):
        e2e = {"value": None, "unit": UNIT, "error": "the host-buffer entry eig_solve_host runs the fixed-parameter T_d solve only"}
    elif not args.no_e2e:
        try:
            xp = torch.from_numpy(X0h).pin_memory()
            evec = torch.empty((r1 - r0, spec.k), dtype=torch.float64).pin_memory()
            rp = torch.from_numpy(np.ascontiguousarray(Aloc.row_ptr)).pin_memory()
            ci = torch.from_numpy(np.ascontiguousarray(Aloc.col_idx)).pin_memory()
            va = torch.from_numpy(np.ascontiguousarray(Aloc.val)).pin_memory()
            grid = stencil_grid(spec) if (not partitioned and use_stencil(spec, args)) else None
            e2e_s = []
            for _ in range(max(1, args.steps)):
                if world > 1:
                    dist.barrier()
                torch.cuda.synchronize(dev)
                t = time.perf_counter()
                if not partitioned:
                    arr.eig_solve_host(A.n, rp, ci, va, spec.k, spec.p, spec.d, xp, tol=spec.tol, maxit=spec.maxit,
                                       s_max=spec.s_max, evec=evec, stream=stream, grid=grid)
                else:
                    with torch.cuda.stream(stream):
                        Ad2 = arr.DeviceCSR(plan.n_own, rp.to(dev, non_blocking=True), ci.to(dev, non_blocking=True),
                                            va.to(dev, non_blocking=True))
                        Xd = xp.to(dev, non_blocking=True)
                        c2 = arr.eig_init(Ad2, spec.k, spec.p, spec.d, stream=stream, w=spec.w, comm=comm, plan=plan)
                        c2.eig_solve(Xd, tol=spec.tol, maxit=spec.maxit, s_max=spec.s_max)
                        evec.copy_(Xd[:r1 - r0, :spec.k], non_blocking=True)
                        stream.synchronize()
                        c2.close()
                        del Ad2, Xd
                e2e_s.append(time.perf_counter() - t)
            tot = float(sum(e2e_s))
            if world > 1:
                t = torch.tensor([tot], dtype=torch.float64, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                tot = float(t.item())
            e2e = {"value": spec.k * len(e2e_s) * jobs / tot, "unit": UNIT,
                   "h2d_bytes_per_step": int(8 * (r1 - r0 + 1) + 12 * nnz_loc + 8 * nrows * spec.w),
                   "d2h_bytes_per_step": int(16 * spec.k + 8 * (r1 - r0) * spec.k),
                   "step_ms": [round(1e3 * x, 3) for x in e2e_s],
                   "api": ("eig_solve_host (C-ABI, pinned host buffers, device alloc + copies inside"
                           + (", stencil grid declared" if grid else "") + ")" if not partitioned
                           else "per rank: H2D of local CSR + X0 rows, eig_init_dist + eig_solve, D2H of the local "
                                "eigenvector rows (bytes of rank 0)")}
        except Exception as exc:  # noqa: BLE001  (e.g. ARR_ENOMEM: the host-buffer call needs its own copies)
            e2e = {"value": None, "unit": UNIT, "error": str(exc)[:200]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ts, smp = oracle_step_estimate(A, spec, args.config)
        one = single_thread_leg(args.config)
        cpu = {"value": spec.k / ts, "unit": UNIT, "cores": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count())),
               "kind": "oracle", "sample": smp, "cpu": cpu_info(),
               "single_thread": ({"value": spec.k / one["seconds"], "unit": UNIT, "cores": 1,
                                  "sample": one["sample"] + " (OMP/BLAS threads = 1)"} if "seconds" in one else one)}

    if rank == 0:
        info = r["infos"][-1]
        par = ("1 GPU" if world == 1 else
               (f"column split over {world} GPUs (A replicated, column-local filter, ARR on a balanced row "
                f"partition; NCCL all-to-all transposes + halo/all-gather + allreduce)" if colsplit else
                f"row partition over {world} GPUs ({_partition_spec(spec)[0]}; SpMM path: {r['path']}" + ("; CSR interior tiles in y-band order" if spec.kind in ("lap3dV", "st27") else "") + "), NCCL halo/all-gather + allreduce"
                if partitioned else f"{world} independent replicas (no collective)"))
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
                "scaling": "strong" if partitioned else "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "parallelism": par,
                "config": config_dict(spec, A, args),
                "run": {"spmm_path": r["path"], "context": "lean (no scratch block)" if r["lean"] else "standard",
                        "converged": bool(info.converged), "outer": info.outer, "sweeps": info.sweeps,
                        "maxres": info.maxres, "locked": info.locked, "p_final": info.p_final,
                        "d_final": info.d_final, "step_ms": [round(x, 3) for x in r["step_ms"]]},
                "roofline": roofline, "secondary": secondary, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(r["launches"]), "clocks": r["clocks"]}
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
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
