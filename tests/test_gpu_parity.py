"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the
same seeded inputs.  Tolerances (BASELINE.json north_star):
filter step rel. Frobenius <= 1e-12; eigenvalues rel. <= 1e-10; every
residual <= tol; SpMM / Gram / GEMM / residuals <= 1e-13 .. 1e-12 relative."""
import numpy as np
import pytest
import torch

import oracle
import synth
from synth import configs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def arr():
    import paper_1507_06078_b200 as m
    return m


def dev_block(X, ld=None):
    n, w = X.shape
    ld = w if ld is None else ld
    buf = torch.zeros((n, ld), dtype=torch.float64, device="cuda")
    buf[:, :w] = torch.from_numpy(np.ascontiguousarray(X))
    return buf[:, :w]


def host(Xd):
    return Xd.cpu().numpy()


def relF(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


SMALL = {
    "lap1d": lambda: synth.laplacian_1d(1000),
    "lap2d": lambda: synth.laplacian_2d(37, 41),
    "lap3dV": lambda: synth.laplacian_3d_potential(13, 2),
    "zipf": lambda: synth.zipf_random(5000, 3),
    "st27": lambda: synth.stencil27_3d(11),
}


# ---------------------------------------------------------------- SpMM (A3)
@pytest.mark.parametrize("kind", list(SMALL))
@pytest.mark.parametrize("w,ld", [(1, 1), (7, 8), (20, 20), (33, 34), (200, 202), (513, 514), (1000, 1000)])
def test_spmm_vs_oracle(arr, kind, w, ld):
    A = SMALL[kind]()
    X = synth.gaussian_block(A.n, w, 11)
    ref = oracle.spmm(A, X)
    Ad = arr.to_device_csr(A)
    ctx = arr.eig_init(Ad, k=4, p=1, d=3)
    Xd = dev_block(X, ld)
    Yd = dev_block(np.zeros_like(X), ld)
    ctx.spmm(Xd, Yd, alpha=0.5, shift=1.25)
    assert relF(host(Yd), 0.5 * (ref - 1.25 * X)) <= 1e-13


# ---------------------------------------------------------------- filter (A1/A2)
@pytest.mark.parametrize("kind", list(SMALL))
@pytest.mark.parametrize("d", [1, 2, 7, 20])
def test_filter_step_vs_oracle(arr, kind, d):
    A = SMALL[kind]()
    w = 24
    X = synth.gaussian_block(A.n, w, 5)
    a = oracle.gershgorin_lower(A)
    b = a + 0.8 * (A.val.max() * 2 - a)
    ref = oracle.cheb_filter(A, a, b, d, X)
    ctx = arr.eig_init(arr.to_device_csr(A), k=w, p=1, d=d)
    ctx.eig_set_interval(a, b)
    Xd = dev_block(X)
    ctx.filter_step(Xd, normalize=False)
    assert relF(host(Xd), ref) <= 1e-12
    # normalised (MPM sweep) + the pre-normalisation norms
    Xd = dev_block(X)
    nrm = torch.empty(w, dtype=torch.float64, device="cuda")
    ctx.filter_step(Xd, normalize=True, colnorm=nrm)
    refn = oracle.mpm_sweep(A, a, b, d, X)
    assert relF(host(Xd), refn) <= 1e-12
    assert np.allclose(nrm.cpu().numpy(), np.linalg.norm(ref, axis=0), rtol=1e-12, atol=0)
    assert np.max(np.abs(np.linalg.norm(host(Xd), axis=0) - 1)) < 1e-14


def test_filter_diagonal_closed_form(arr):
    rng = np.random.default_rng(0)
    diag = rng.uniform(-0.5, 4.0, 3001)
    A = synth.diagonal(diag)
    X = rng.standard_normal((3001, 10))
    ctx = arr.eig_init(arr.to_device_csr(A), k=10, p=0, d=30)
    ctx.eig_set_interval(0.0, 3.0)
    Xd = dev_block(X)
    ctx.filter_step(Xd, normalize=False)
    t = (diag - 1.5) / 1.5
    f = np.where(np.abs(t) <= 1, np.cos(30 * np.arccos(np.clip(t, -1, 1))),
                 np.sign(t) ** 30 * np.cosh(30 * np.arccosh(np.maximum(np.abs(t), 1))))
    assert relF(host(Xd), f[:, None] * X) <= 1e-12


def test_filter_is_deterministic_and_column_independent(arr):
    A = synth.laplacian_2d(60)
    X = synth.gaussian_block(A.n, 40, 3)
    ctx = arr.eig_init(arr.to_device_csr(A), k=40, p=1, d=9)
    ctx.eig_set_interval(0.0, 7.5)
    outs = []
    for _ in range(2):
        Xd = dev_block(X)
        ctx.filter_step(Xd, normalize=True)
        outs.append(host(Xd))
    assert np.array_equal(outs[0], outs[1])
    ctx2 = arr.eig_init(arr.to_device_csr(A), k=40, p=1, d=9)
    ctx2.eig_set_interval(0.0, 7.5)
    Xd = dev_block(X)
    ctx2.filter_step(Xd, normalize=False)
    full = host(Xd)
    ctx3 = arr.eig_init(arr.to_device_csr(A), k=8, p=1, d=9)
    ctx3.eig_set_interval(0.0, 7.5)
    Xs = dev_block(X[:, 8:16])
    ctx3.filter_step(Xs, normalize=False)
    # per-row arithmetic does not depend on the block width: bitwise
    assert np.array_equal(full[:, 8:16], host(Xs))


def test_filter_errors(arr):
    A = synth.laplacian_1d(100)
    ctx = arr.eig_init(arr.to_device_csr(A), k=4, p=1, d=3)
    Xd = dev_block(np.ones((100, 4)))
    with pytest.raises(arr.ArrError):
        ctx.filter_step(Xd)  # no interval yet
    with pytest.raises(arr.ArrError):
        ctx.eig_set_interval(1.0, 1.0)
    # a zero column -> ARR_ENUMERIC
    ctx.eig_set_interval(0.0, 3.0)
    X = np.ones((100, 4))
    X[:, 2] = 0
    with pytest.raises(arr.ArrError) as e:
        ctx.filter_step(dev_block(X), normalize=True)
    assert e.value.status == 7
    # (p+1)k >= n rejected at init
    with pytest.raises(arr.ArrError):
        arr.eig_init(arr.to_device_csr(A), k=50, p=1, d=3)


def test_gershgorin(arr):
    for A in (synth.laplacian_2d(30), synth.laplacian_3d_potential(9, 2), synth.zipf_random(3000, 1)):
        ctx = arr.eig_init(arr.to_device_csr(A), k=4, p=1, d=3)
        assert ctx.eig_gershgorin_lower() == pytest.approx(oracle.gershgorin_lower(A), abs=1e-12 * A.val.max())


# ---------------------------------------------------------------- dense (A4)
@pytest.mark.parametrize("n,m1,m2", [(1000, 20, 20), (4097, 65, 130), (90000, 200, 200), (33, 7, 3), (20000, 400, 200)])
def test_gram_gemm_vs_numpy(arr, n, m1, m2):
    rng = np.random.default_rng(n + m1)
    X = rng.standard_normal((n, m1))
    Y = rng.standard_normal((n, m2))
    B = rng.standard_normal((m1, m2))
    C = rng.standard_normal((n, m2))
    A = synth.laplacian_1d(n)
    ctx = arr.eig_init(arr.to_device_csr(A), k=2, p=1, d=1)
    G = torch.zeros((m1, m2), dtype=torch.float64, device="cuda")
    ctx.gram(dev_block(X), dev_block(Y), G)
    ref = X.T @ Y
    assert np.max(np.abs(G.cpu().numpy() - ref)) <= 1e-13 * np.sqrt(n) * 4
    Gs = torch.zeros((m1, m1), dtype=torch.float64, device="cuda")
    Xd = dev_block(X)
    ctx.gram(Xd, Xd, Gs)
    gs = Gs.cpu().numpy()
    assert np.array_equal(gs, gs.T)
    assert np.max(np.abs(gs - X.T @ X)) <= 1e-13 * n * 4
    Out = dev_block(np.zeros((n, m2)))
    Bd = torch.from_numpy(B).cuda()
    Cd = dev_block(C)
    ctx.gemm(Xd, Bd, Out, alpha=-0.5, beta=2.0, Cin=Cd)
    assert relF(host(Out), -0.5 * X @ B + 2.0 * C) <= 1e-14 * np.sqrt(m1) * 4


def test_orthonormalize(arr):
    A = synth.laplacian_2d(100)
    X = synth.gaussian_block(A.n, 64, 2)
    X = X @ np.diag(np.logspace(0, 6, 64))  # column dynamic range 1e6
    ctx = arr.eig_init(arr.to_device_csr(A), k=64, p=1, d=3)
    Xd = dev_block(X)
    r = ctx.orthonormalize(Xd)
    U = host(Xd)
    assert r == 64
    assert np.linalg.norm(U.T @ U - np.eye(64)) < 1e-13
    # same span
    assert np.linalg.norm(X - U @ (U.T @ X)) < 1e-11 * np.linalg.norm(X)
    # an exactly dependent column: rank deficit reported, output still orthonormal
    X2 = synth.gaussian_block(A.n, 64, 3)
    X2[:, 10] = X2[:, 3]
    Xd = dev_block(X2)
    r = ctx.orthonormalize(Xd)
    U = host(Xd)
    assert r == 63
    assert np.linalg.norm(U.T @ U - np.eye(64)) < 1e-12
    assert np.linalg.norm(X2 - U @ (U.T @ X2)) < 1e-11 * np.linalg.norm(X2)


# ---------------------------------------------------------------- ARR (A4)
@pytest.mark.parametrize("kind", ["lap2d", "lap3dV", "zipf", "st27"])
@pytest.mark.parametrize("p", [0, 1, 2])
def test_arr_project_vs_oracle(arr, kind, p):
    A = SMALL[kind]()
    w = 16
    X = synth.gaussian_block(A.n, w, 9)
    a = oracle.gershgorin_lower(A)
    b = a + 0.7 * (2 * np.abs(A.val).max() - a)
    X = oracle.mpm_sweep(A, a, b, 4, X)  # a realistic, well-conditioned filtered block
    mu_o, Y_o, r_o = oracle.arr(A, X, p)
    ctx = arr.eig_init(arr.to_device_csr(A), k=w, p=2, d=4)
    Xd = dev_block(X)
    Yd = dev_block(np.zeros_like(X))
    ritz, rank = ctx.arr_project(Xd, Yd, p=p)
    m = (p + 1) * w
    assert r_o == m and rank == m
    scale = np.abs(A.val).max() * 2
    assert np.max(np.abs(ritz - mu_o[:m])) <= 1e-12 * scale
    Y = host(Yd)
    assert np.linalg.norm(Y.T @ Y - np.eye(w)) < 1e-12
    # same Ritz vectors up to sign within non-degenerate clusters: compare projectors
    res_g = ctx.residuals(Yd, ritz[:w])
    res_o = oracle.residuals(A, Y_o, mu_o[:w])
    assert np.max(np.abs(res_g - res_o)) <= 1e-10 * max(1.0, res_o.max())


def test_arr_exact_eigenvectors(arr):
    n, k = 2000, 20
    A = synth.laplacian_1d(n)
    j = np.arange(1, n + 1)
    lam = 2 - 2 * np.cos(j * np.pi / (n + 1))
    top = np.argsort(-lam)[:k]
    V = np.sin(np.outer(j, j[top]) * np.pi / (n + 1))
    V /= np.linalg.norm(V, axis=0)
    ctx = arr.eig_init(arr.to_device_csr(A), k=k, p=1, d=10)
    Xd = dev_block(V @ np.random.default_rng(0).standard_normal((k, k)))
    Yd = dev_block(np.zeros((n, k)))
    ritz, _ = ctx.arr_project(Xd, Yd)
    assert np.max(np.abs(ritz[:k] - lam[top]) / lam[top]) < 1e-13
    assert np.max(ctx.residuals(Yd, ritz[:k])) < 1e-12


def test_arr_exact_eigenvectors_p2(arr):
    """p = 2 on an exactly invariant X: the augmentation blocks U_1, U_2 are orthonormalised
    rounding noise (no Krylov information), the case where the block-tridiagonal H of
    reading R22 leans hardest on U_2 being orthogonal to U_0 and U_1.  The k wanted Ritz
    pairs must still be the exact eigenpairs."""
    n, k = 2000, 20
    A = synth.laplacian_1d(n)
    j = np.arange(1, n + 1)
    lam = 2 - 2 * np.cos(j * np.pi / (n + 1))
    top = np.argsort(-lam)[:k]
    V = np.sin(np.outer(j, j[top]) * np.pi / (n + 1))
    V /= np.linalg.norm(V, axis=0)
    ctx = arr.eig_init(arr.to_device_csr(A), k=k, p=2, d=10)
    Xd = dev_block(V @ np.random.default_rng(0).standard_normal((k, k)))
    Yd = dev_block(np.zeros((n, k)))
    ritz, _ = ctx.arr_project(Xd, Yd)
    assert np.max(np.abs(ritz[:k] - lam[top]) / lam[top]) < 1e-13
    assert np.max(ctx.residuals(Yd, ritz[:k])) < 1e-12
    # every Ritz value of the 3k-dimensional space lies in the spectrum's range (a true
    # Rayleigh quotient of an orthonormal basis)
    assert ritz.min() > -1e-12 and ritz.max() < 4 + 1e-12


# ---------------------------------------------------------------- residuals (A6)
def test_residuals_vs_oracle(arr):
    A = synth.zipf_random(6000, 7)
    Y = synth.gaussian_block(A.n, 30, 1)
    mu = np.linspace(-3, 40, 30)
    ctx = arr.eig_init(arr.to_device_csr(A), k=30, p=1, d=3)
    res = ctx.residuals(dev_block(Y), mu)
    ref = oracle.residuals(A, Y, mu)
    assert np.max(np.abs(res - ref) / ref) < 1e-12


# ---------------------------------------------------------------- full solve
def _closed_lap1d(n):
    return np.sort(2 - 2 * np.cos(np.arange(1, n + 1) * np.pi / (n + 1)))[::-1]


def test_solve_cfg1_vs_closed_form_and_oracle(arr):
    A, spec = configs.build_config(1)
    X0 = synth.starting_block(spec)
    ctx = arr.eig_init(arr.to_device_csr(A), spec.k, spec.p, spec.d, w=spec.w)
    Xd = dev_block(X0)
    ev, res, info = ctx.eig_solve(Xd, tol=spec.tol)
    assert info.converged == 1
    assert np.all(res <= spec.tol)
    lam = _closed_lap1d(A.n)[:spec.k]
    assert np.max(np.abs(ev - lam) / lam) < 1e-10
    orc = oracle.solve(A, spec.k, spec.d, spec.p, X0, tol=spec.tol)
    assert np.max(np.abs(ev - orc.mu) / np.abs(orc.mu)) < 1e-10
    # residual certificate recomputed by the oracle from the GPU's pairs
    cert = oracle.residuals(A, host(Xd)[:, :spec.k], ev)
    assert np.all(cert <= 1.01 * spec.tol)


@pytest.mark.parametrize("kind", ["lap2d", "lap3dV", "zipf", "st27"])
def test_solve_small_analogs_vs_oracle(arr, kind):
    spec = configs.SMALL_ANALOGS[kind]
    A, _ = configs.build_config(spec)
    X0 = synth.starting_block(spec)
    ctx = arr.eig_init(arr.to_device_csr(A), spec.k, spec.p, spec.d, w=spec.w)
    Xd = dev_block(X0)
    ev, res, info = ctx.eig_solve(Xd, tol=spec.tol)
    assert info.converged == 1 and np.all(res <= spec.tol)
    lam = np.sort(np.linalg.eigvalsh(A.to_dense()))[::-1][:spec.k]
    assert np.max(np.abs(ev - lam) / np.maximum(1, np.abs(lam))) < 1e-10
    orc = oracle.solve(A, spec.k, spec.d, spec.p, X0, tol=spec.tol)
    assert np.max(np.abs(ev - orc.mu) / np.maximum(1, np.abs(orc.mu))) < 1e-10


def test_solve_cfg2_closed_form(arr):
    A, spec = configs.build_config(2)
    X0 = synth.starting_block(spec)
    ctx = arr.eig_init(arr.to_device_csr(A), spec.k, spec.p, spec.d, w=spec.w)
    Xd = dev_block(X0)
    ev, res, info = ctx.eig_solve(Xd, tol=spec.tol)
    assert info.converged == 1 and np.all(res <= spec.tol)
    N = 300
    c = 2 * np.cos(np.arange(1, N + 1) * np.pi / (N + 1))
    lam = np.sort((4 - c[:, None] - c[None, :]).ravel())[::-1][:spec.k]
    assert np.max(np.abs(ev - lam) / lam) < 1e-10
    assert ev.sum() == pytest.approx(1596.924226909574, rel=1e-12)  # SURVEY §8c-5 closed form
    cert = oracle.residuals(A, host(Xd)[:, :spec.k], ev)
    assert np.all(cert <= 1.01 * spec.tol)


def test_solve_host_entry(arr):
    spec = configs.SMALL_ANALOGS["lap2d"]
    A, _ = configs.build_config(spec)
    X0 = synth.starting_block(spec)
    evec = np.empty((A.n, spec.k))
    ev, res, info = arr.eig_solve_host(A.n, A.row_ptr, A.col_idx, A.val, spec.k, spec.p, spec.d, X0,
                                       tol=spec.tol, evec=evec)
    assert info.converged == 1
    cert = oracle.residuals(A, evec, ev)
    assert np.all(cert <= 1.01 * spec.tol)


@pytest.mark.parametrize("kind", ["lap2d", "st27"])
def test_lean_context_is_bitwise_identical(arr, kind, monkeypatch):
    """A context without the scratch block (lean: the spare basis block and the
    output block serve as scratch, DESIGN.md §5 Memory) computes exactly the
    same solve: only buffer locations change, never the arithmetic."""
    spec = configs.SMALL_ANALOGS[kind]
    A, _ = configs.build_config(spec)
    X0 = synth.starting_block(spec)
    out = []
    for lean in (False, True):
        if lean:
            monkeypatch.setenv("ARRABIT_LEAN", "1")
        ctx = arr.eig_init(arr.to_device_csr(A), spec.k, spec.p, spec.d, w=spec.w)
        Xd = dev_block(X0)
        ev, res, info = ctx.eig_solve(Xd, tol=spec.tol)
        out.append((ev, res, info.outer, host(Xd)))
        if lean:
            Y = torch.empty_like(Xd)
            with pytest.raises(arr.ArrError):
                ctx.arr_project(Xd, Y)  # lean: the Ritz vectors must overwrite X
        ctx.close()
    assert out[0][2] == out[1][2]
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
    assert np.array_equal(out[0][3], out[1][3])


def test_cfg2_full_filter_and_arr_vs_oracle(arr):
    """The bench workload (configs[1] = cfg2, n = 90,000, w = 220) in the launch
    configuration eig_solve uses: one MPM sweep (d = 20) against the oracle's
    element by element (rel. Frobenius <= 1e-12, BASELINE north star), then one ARR
    (p = 1) on the filtered block against the oracle's paper-literal ARR (pivoted QR
    of [X, AX]; same span, different orthonormalisation, R8): the leading w
    Ritz values agree to 1e-11 relative."""
    A, spec = configs.build_config(2)
    X0 = synth.starting_block(spec)
    ctx = arr.eig_init(arr.to_device_csr(A), spec.k, spec.p, spec.d, w=spec.w)
    a = ctx.eig_gershgorin_lower()
    mu0, _, _ = oracle.rayleigh_ritz(A, X0)
    b = float(mu0[spec.w - 1])
    ctx.eig_set_interval(a, b)
    Xd = torch.from_numpy(X0).cuda()
    ctx.filter_step(Xd, normalize=True)
    ref = oracle.mpm_sweep(A, a, b, spec.d, X0)
    assert relF(host(Xd), ref) <= 1e-12
    Y = torch.empty_like(Xd)
    ritz, rank = ctx.arr_project(Xd, Y)
    mu, _, _ = oracle.arr(A, ref, spec.p)
    w = spec.w
    assert np.max(np.abs(ritz[:w] - mu[:w]) / np.abs(mu[:w])) <= 1e-11
    res = ctx.residuals(Y[:, :spec.k], ritz[:spec.k])
    res_o = oracle.residuals(A, host(Y)[:, :spec.k], ritz[:spec.k])
    assert np.max(np.abs(res - res_o)) <= 1e-12 * max(1.0, res_o.max())


@pytest.mark.parametrize("kind", list(SMALL))
@pytest.mark.parametrize("d", [1, 2, 7, 20])
def test_interp_filter_step_vs_oracle(arr, kind, d):
    """The paper's interpolant filter rho_d (eig_set_filter 'interp') against the
    oracle's Clenshaw evaluation (oracle.poly_filter), before and after normalisation."""
    A = SMALL[kind]()
    w = 24
    X0 = synth.gaussian_block(A.n, w, 13)
    ctx = arr.eig_init(arr.to_device_csr(A), w, 1, d)
    ctx.eig_set_filter("interp")
    a = ctx.eig_gershgorin_lower()
    b = a + 0.6 * (2 * float(np.abs(A.val).max()) * 2 - a)
    ctx.eig_set_interval(a, b)
    coef = oracle.interp_coeffs(d)
    ref = oracle.poly_filter(A, a, b, coef, X0)
    Xd = dev_block(X0, ld=w + 2)
    ctx.filter_step(Xd, normalize=False)
    assert relF(host(Xd), ref) <= 1e-12
    Xd = dev_block(X0)
    ctx.filter_step(Xd, normalize=True)
    assert relF(host(Xd), oracle.poly_sweep(A, a, b, coef, X0)) <= 1e-12


@pytest.mark.parametrize("kind", ["lap2d", "st27", "zipf"])
def test_solve_with_interp_filter(arr, kind):
    spec = configs.SMALL_ANALOGS[kind]
    A, _ = configs.build_config(spec)
    X0 = synth.starting_block(spec)
    ctx = arr.eig_init(arr.to_device_csr(A), spec.k, spec.p, spec.d, w=spec.w)
    ctx.eig_set_filter("interp")
    Xd = dev_block(X0)
    ev, res, info = ctx.eig_solve(Xd, tol=spec.tol)
    assert info.converged == 1 and np.all(res <= spec.tol)
    lam = np.sort(np.linalg.eigvalsh(A.to_dense()))[::-1][:spec.k]
    assert np.max(np.abs(ev - lam) / np.maximum(1, np.abs(lam))) < 1e-10


@pytest.mark.parametrize("kind", ["lap2d", "zipf"])
def test_smallest_mode_solve(arr, kind):
    """k algebraically smallest eigenpairs (eig_set_mode 'smallest': the method on
    -A, the paper's second mode, Table 6): eigenvalues of A ascending, equal to
    the dense spectrum; the oracle's solve on -A gives the same values; residual
    certificates recomputed by the oracle with A itself."""
    spec = configs.SMALL_ANALOGS[kind]
    A, _ = configs.build_config(spec)
    X0 = synth.starting_block(spec)
    ctx = arr.eig_init(arr.to_device_csr(A), spec.k, spec.p, spec.d, w=spec.w)
    ctx.eig_set_mode("smallest")
    Xd = dev_block(X0)
    ev, res, info = ctx.eig_solve(Xd, tol=spec.tol)
    assert info.converged == 1 and np.all(res <= spec.tol)
    lam = np.sort(np.linalg.eigvalsh(A.to_dense()))[:spec.k]
    assert np.all(np.diff(ev) >= 0)
    assert np.max(np.abs(ev - lam) / np.maximum(1, np.abs(lam))) < 1e-10
    negA = synth.CSR(A.n, A.row_ptr, A.col_idx, -A.val, name="negA")
    orc = oracle.solve(negA, spec.k, spec.d, spec.p, X0, tol=spec.tol)
    assert np.max(np.abs(ev + orc.mu) / np.maximum(1, np.abs(ev))) < 1e-10
    cert = oracle.residuals(A, host(Xd)[:, :spec.k], ev)
    assert np.all(cert <= 1.01 * spec.tol)


def test_smallest_mode_bipartite_symmetry(arr):
    """2-D Dirichlet Laplacian (diagonal 4, bipartite): the spectrum is symmetric about
    4, so the k smallest are 8 - (the k largest)."""
    spec = configs.SMALL_ANALOGS["lap2d"]
    A, _ = configs.build_config(spec)
    X0 = synth.starting_block(spec)
    out = {}
    for mode in ("largest", "smallest"):
        ctx = arr.eig_init(arr.to_device_csr(A), spec.k, spec.p, spec.d, w=spec.w)
        ctx.eig_set_mode(mode)
        ev, _, info = ctx.eig_solve(dev_block(X0), tol=spec.tol)
        assert info.converged == 1
        out[mode] = ev
    np.testing.assert_allclose(out["smallest"], 8.0 - out["largest"], rtol=0, atol=1e-10 * 8)


def test_paper_exit_rules(arr):
    """The paper's extra stop rules, opt-in: (ii) stops a solve whose
    tolerance is out of reach once max res stalls for three outer iterations; (iii),
    when it fires, leaves max res < 10 tol."""
    spec = configs.SMALL_ANALOGS["lap2d"]
    A, _ = configs.build_config(spec)
    X0 = synth.starting_block(spec)
    ctx = arr.eig_init(arr.to_device_csr(A), spec.k, spec.p, spec.d, w=spec.w)
    ev, res, info = ctx.eig_solve(dev_block(X0), tol=1e-18, maxit=200, exits=1)
    assert info.exit_rule == 2 and info.outer < 200 and info.converged == 0
    ev2, res2, info2 = ctx.eig_solve(dev_block(X0), tol=1e-10, maxit=200, exits=2)
    assert info2.exit_rule in (1, 3)
    assert res2.max() < 10 * 1e-10
    ev3, res3, info3 = ctx.eig_solve(dev_block(X0), tol=1e-10, maxit=200, exits=0)
    assert info3.exit_rule == 1 and info3.outer >= info2.outer


@pytest.mark.parametrize("kind", ["lap2d", "lap3dV"])
def test_solve_with_paper_rcond_inner_rule(arr, kind):
    """The paper's inner stop rule (rcond(X^T X) every 5 sweeps) instead of
    the dynamic-range rule: the solve still reaches the dense eigenvalues."""
    spec = configs.SMALL_ANALOGS[kind]
    A, _ = configs.build_config(spec)
    X0 = synth.starting_block(spec)
    ctx = arr.eig_init(arr.to_device_csr(A), spec.k, spec.p, spec.d, w=spec.w)
    ev, res, info = ctx.eig_solve(dev_block(X0), tol=spec.tol, maxit=100, inner="rcond")
    assert info.converged == 1 and info.sweeps % 5 == 0
    lam = np.sort(np.linalg.eigvalsh(A.to_dense()))[::-1][:spec.k]
    assert np.max(np.abs(ev - lam) / np.maximum(1, np.abs(lam))) < 1e-10


@pytest.mark.parametrize("kind,adapt", [("lap2d", 1), ("lap2d", 2), ("lap3dV", 3), ("zipf", 3)])
def test_solve_with_adaptive_p_and_d(arr, kind, adapt):
    """The paper's adaptive augmentation depth (Eq. block) and degree (Eqs. hat-d,
    degree): the solve reaches the dense eigenvalues; p stays within
    [1, p_max] and d within [3, d_max]; the context's degree is restored."""
    spec = configs.SMALL_ANALOGS[kind]
    A, _ = configs.build_config(spec)
    X0 = synth.starting_block(spec)
    ctx = arr.eig_init(arr.to_device_csr(A), spec.k, spec.p, spec.d, w=spec.w)
    ev, res, info = ctx.eig_solve(dev_block(X0), tol=spec.tol, maxit=200, adapt=adapt)
    assert info.converged == 1
    lam = np.sort(np.linalg.eigvalsh(A.to_dense()))[::-1][:spec.k]
    assert np.max(np.abs(ev - lam) / np.maximum(1, np.abs(lam))) < 1e-10
    if adapt & 1:
        assert 1 <= info.p_final <= spec.p
    else:
        assert info.p_final == spec.p
    if adapt & 2:
        assert 3 <= info.d_final <= spec.d
    ev2, _, info2 = ctx.eig_solve(dev_block(X0), tol=spec.tol)  # fixed parameters afterwards
    assert info2.d_final == spec.d and info2.p_final == spec.p


@pytest.mark.parametrize("kind", ["lap2d", "lap3dV", "st27", "zipf"])
def test_solve_with_continuation_and_deflation(arr, kind):
    """Alg. Arrabit2's continuation and deflation (locking), adapt bit 4:
    the solve reaches the dense eigenvalues, every returned pair (locked or not) meets
    tol by the oracle's own residual recomputation, and the pairs come out ordered."""
    spec = configs.SMALL_ANALOGS[kind]
    A, _ = configs.build_config(spec)
    X0 = synth.starting_block(spec)
    ctx = arr.eig_init(arr.to_device_csr(A), spec.k, spec.p, spec.d, w=spec.w)
    Xd = dev_block(X0)
    ev, res, info = ctx.eig_solve(Xd, tol=spec.tol, maxit=200, adapt=4)
    assert info.converged == 1 and 0 <= info.locked < spec.k, (
        info.outer, info.maxres, info.locked, info.exit_rule, info.a, info.b)
    lam = np.sort(np.linalg.eigvalsh(A.to_dense()))[::-1][:spec.k]
    assert np.max(np.abs(ev - lam) / np.maximum(1, np.abs(lam))) < 1e-10
    assert np.all(np.diff(ev) <= 1e-12 * np.abs(ev).max())
    cert = oracle.residuals(A, host(Xd)[:, :spec.k], ev)
    assert np.all(cert <= 1.01 * spec.tol)


@pytest.mark.parametrize("kind", ["lap2d", "lap3dV", "zipf"])
def test_solve_with_gn_inner_solver(arr, kind):
    """Alg. Arrabit2 with the Gauss-Newton inner solver: the solve
    reaches the dense eigenvalues; residual certificates by the oracle."""
    spec = configs.SMALL_ANALOGS[kind]
    A, _ = configs.build_config(spec)
    X0 = synth.starting_block(spec)
    ctx = arr.eig_init(arr.to_device_csr(A), spec.k, spec.p, spec.d, w=spec.w)
    Xd = dev_block(X0)
    ev, res, info = ctx.eig_solve(Xd, tol=spec.tol, maxit=200, inner_solver="gn")
    assert info.converged == 1
    lam = np.sort(np.linalg.eigvalsh(A.to_dense()))[::-1][:spec.k]
    assert np.max(np.abs(ev - lam) / np.maximum(1, np.abs(lam))) < 1e-10
    cert = oracle.residuals(A, host(Xd)[:, :spec.k], ev)
    assert np.all(cert <= 1.01 * spec.tol)


def test_phase_and_kernel_times(arr):
    """eig_set_timing / eig_phase_times / eig_kernel_times: the d filter launches of a sweep
    are counted; the DMMA Gram and GEMM launches report their ALGORITHMIC flops (2 n m1 m2,
    a symmetric Gram n m (m + 1), an upper-triangular B 2 n sum_c min(c + 1, m1)) and
    positive device times; a Gram of known shape adds exactly its flops."""
    A = synth.laplacian_2d(60)
    k, p, d = 24, 1, 7
    ctx = arr.eig_init(arr.to_device_csr(A), k, p, d)
    X = torch.from_numpy(synth.gaussian_block(A.n, k, 3)).cuda()
    ctx.eig_set_interval(ctx.eig_gershgorin_lower(), 6.0)
    ctx.eig_set_timing(True)
    ctx.filter_step(X, normalize=True)
    Y = torch.empty_like(X)
    ctx.arr_project(X, Y)
    ms, cnt = ctx.eig_phase_times()
    assert cnt[0] == d and ms[0] > 0 and cnt[1] == 1 and ms[1] > 0
    kms, kfl, kcnt = ctx.eig_kernel_times()
    assert kcnt[0] > 0 and kcnt[1] > 0 and (kms > 0).all()
    G = torch.empty((k, 8), dtype=torch.float64, device="cuda")
    ctx.eig_set_timing(True)  # zeroes the totals
    ctx.gram(X, X[:, :8], G)
    ms2, fl2, c2 = ctx.eig_kernel_times()
    assert c2[0] == 1 and c2[1] == 0 and fl2[0] == 2.0 * A.n * k * 8
    Gs = torch.empty((k, k), dtype=torch.float64, device="cuda")
    ctx.gram(X, X, Gs)  # symmetric: the upper triangle's n k (k + 1)
    ms3, fl3, c3 = ctx.eig_kernel_times()
    assert c3[0] == 2 and fl3[0] - fl2[0] == float(A.n) * k * (k + 1)
    ctx.close()
