"""Stencil path on z-slabs at cfg3's full size, on ONE GPU: G ranks of an in-process group
(one host thread and stream each, as tests/test_gpu_dist.py), each declaring its slab with
eig_set_stencil.  Checks the un-normalised filter bitwise against the one-GPU stencil path
and reports the wall time of one filter_step of all G ranks running together next to the
one-GPU time (same total work on the same GPU: the cost of the slab decomposition, i.e.
ghost planes, the three launches per degree and the exchange copies).  Not a bench line."""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1507_06078_b200 as arr  # noqa: E402
from paper_1507_06078_b200 import partition as pt  # noqa: E402
from synth import configs  # noqa: E402


def run_ranks(G, fn):
    out, err = [None] * G, [None] * G

    def body(r):
        try:
            torch.cuda.set_device(0)
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            err[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(G)]
    [t.start() for t in th]
    [t.join() for t in th]
    for e in err:
        if e is not None:
            raise e
    return out


def main():
    cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    A, spec = configs.build_config(cid)
    N = spec.size
    w, d = spec.w, spec.d
    ld = (w + 15) // 16 * 16
    X0 = np.random.default_rng(7).standard_normal((A.n, w))
    c1 = arr.eig_init(arr.to_device_csr(A), spec.k, 0, d, w=w)
    c1.eig_set_stencil(N, N, N)
    a = c1.eig_gershgorin_lower()
    b = a + 0.9 * (float(np.abs(A.val).max()) * 8 - a)
    c1.eig_set_interval(a, b)
    Xb = torch.zeros((A.n, ld), dtype=torch.float64, device="cuda")
    X1 = Xb[:, :w]
    X1.copy_(torch.from_numpy(X0))
    c1.filter_step(X1, normalize=False)
    ref = X1.cpu().numpy()
    ts = []
    for _ in range(3):
        X1.copy_(torch.from_numpy(X0))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        c1.filter_step(X1, normalize=False)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"cfg{cid} one GPU: filter_step (d = {d}) {min(ts) * 1e3:.1f} ms, kernel {c1.last_spmm_kernel}", flush=True)
    c1.close()
    del Xb, X1
    for G in (2, 4, 8):
        ps = pt.plans(A, pt.bounds_planes(N, N * N, G))
        comms = arr.Comm.local_group(G)
        bar = threading.Barrier(G)
        wall = [0.0] * G

        def work(r):
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                Ad = arr.to_device_csr(ps[r])
            s.synchronize()
            ctx = arr.eig_init(Ad, spec.k, 0, d, stream=s, w=w, comm=comms[r], plan=ps[r])
            with torch.cuda.stream(s):
                ctx.eig_set_stencil(N, N, ps[r].n_own // (N * N))
                ctx.eig_set_interval(a, b)
                blk = torch.from_numpy(pt.scatter_rows(X0, ps[r], ld)).cuda()
                Xr = blk[:, :w]
                ctx.filter_step(Xr, normalize=False)
                raw = Xr[:ps[r].n_own].cpu().numpy()
                kern = ctx.last_spmm_kernel
                best = 1e9
                for _ in range(3):
                    Xr.copy_(torch.from_numpy(pt.scatter_rows(X0, ps[r], ld)).cuda()[:, :w])
                    s.synchronize()
                    bar.wait()
                    t0 = time.perf_counter()
                    ctx.filter_step(Xr, normalize=False)
                    s.synchronize()
                    bar.wait()
                    best = min(best, time.perf_counter() - t0)
                wall[r] = best
            ctx.close()
            return raw, kern

        res = run_ranks(G, work)
        for c in comms:
            c.close()
        raw = np.vstack([x[0] for x in res])
        ok = np.array_equal(raw, ref)
        print(f"cfg{cid} G = {G} slabs on one GPU: bitwise equal {ok}; filter_step of all ranks together "
              f"{max(wall) * 1e3:.1f} ms; kernels {sorted(set(x[1] for x in res))}", flush=True)
        assert ok


if __name__ == "__main__":
    main()
