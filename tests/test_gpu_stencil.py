"""The stencil-aware filter path (eig_set_stencil, csrc/stencil_kernels.cu): the same
fused degree as the CSR kernels with the same per-row FMA order, so the un-normalised
output is bitwise the CSR kernels' and both match the oracle (Eq. cheby-poly
P:377-383; Alg. Arrabit2 line P:1486).  Covers 1-D / 2-D / 3-D 7-point (+V) / 27-point
operators, ragged patches, several panels and z-chunks, padded leading dimensions, the
interpolant filter's fourth operand and the MPM normalisation."""
import numpy as np
import pytest
import torch

import oracle
import synth

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


def relF(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def _varcoef(A, seed):
    """The same pattern with every off-diagonal value scaled by its own factor in [0.5, 1.5)
    (no constant coefficient: the K-diagonal value mode)."""
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    off = rows != A.col_idx
    val = A.val.copy()
    val[off] *= 0.5 + np.random.default_rng(seed).random(int(off.sum()))
    return synth.CSR(A.n, A.row_ptr.copy(), A.col_idx.copy(), val, A.name + "_var")


# (matrix, declared grid (nx, ny, nz), A bytes per row the stencil path reads)
CASES = {
    "lap1d": (lambda: synth.laplacian_1d(1000), (1000, 1, 1), 0),       # all coefficients constant
    "lap2d_xz": (lambda: synth.laplacian_2d(37, 41), (37, 1, 41), 0),   # march along y
    "lap2d_xy": (lambda: synth.laplacian_2d(37, 41), (37, 41, 1), 0),   # one plane, y halo
    "lap3dV": (lambda: synth.laplacian_3d_potential(13, 2), (13, 13, 13), 56),    # nx odd: K diagonals
    "lap3dV_even": (lambda: synth.laplacian_3d_potential(14, 2), (14, 14, 14), 8),  # the diagonal only
    "lap3d_var": (lambda: _varcoef(synth.laplacian_3d_potential(12, 2), 3), (12, 12, 12), 56),
    "st27": (lambda: synth.stencil27_3d(11), (11, 11, 11), 0),
    "st27_tall": (lambda: synth.stencil27_3d(6), (6, 6, 6), 0),
    "st27_var": (lambda: _varcoef(synth.stencil27_3d(8), 4), (8, 8, 8), 216),
}


def _pair(arr, A, grid, w, d, ld=None):
    Ad = arr.to_device_csr(A)
    c_csr = arr.eig_init(Ad, k=w, p=0, d=d)
    c_st = arr.eig_init(Ad, k=w, p=0, d=d)
    c_st.eig_set_stencil(*grid)
    assert c_st.stencil_points > 0 and c_csr.stencil_points == 0
    return c_csr, c_st


@pytest.mark.parametrize("kind", list(CASES))
@pytest.mark.parametrize("w,ld", [(2, 2), (24, 26), (98, 98), (282, 282), (550, 552)])
def test_stencil_filter_bitwise_and_oracle(arr, kind, w, ld):
    mk, grid, abytes = CASES[kind]
    A = mk()
    if w >= A.n:
        pytest.skip("block wider than the matrix")
    d = 5
    X = synth.gaussian_block(A.n, w, 7)
    a = oracle.gershgorin_lower(A)
    b = a + 0.7 * (2 * np.abs(A.val).max() * 2 - a)
    c_csr, c_st = _pair(arr, A, grid, w, d)
    assert c_st.stencil_abytes == abytes  # the value mode detected from the coefficients
    out = {}
    for name, ctx in (("csr", c_csr), ("st", c_st)):
        ctx.eig_set_interval(a, b)
        Xd = dev_block(X, ld)
        ctx.filter_step(Xd, normalize=False)
        out[name] = Xd.cpu().numpy()
    diff = np.abs(out["csr"] - out["st"])
    assert np.array_equal(out["csr"], out["st"]), \
        f"stencil path not bitwise equal to the CSR kernels: {np.count_nonzero(diff)} entries, max {diff.max():.3e}"
    if w <= 98:
        ref = oracle.cheb_filter(A, a, b, d, X)
        assert relF(out["st"], ref) <= 1e-12


@pytest.mark.parametrize("kind", ["lap3dV", "lap3dV_even", "lap3d_var", "st27", "lap2d_xz"])
def test_stencil_normalised_and_interp(arr, kind):
    mk, grid, _ = CASES[kind]
    A = mk()
    w, d = 40, 8
    X = synth.gaussian_block(A.n, w, 9)
    a = oracle.gershgorin_lower(A)
    b = a + 0.6 * (2 * np.abs(A.val).max() * 2 - a)
    c_csr, c_st = _pair(arr, A, grid, w, d)
    ref = oracle.mpm_sweep(A, a, b, d, X)
    res = {}
    for name, ctx in (("csr", c_csr), ("st", c_st)):
        ctx.eig_set_interval(a, b)
        Xd = dev_block(X)
        nrm = torch.empty(w, dtype=torch.float64, device="cuda")
        ctx.filter_step(Xd, normalize=True, colnorm=nrm)
        res[name] = Xd.cpu().numpy()
        assert relF(res[name], ref) <= 1e-12
    # column norms are summed in another order by the two paths: equal to rounding
    assert relF(res["st"], res["csr"]) <= 1e-14
    # the paper's interpolant filter (Clenshaw steps with X as the fourth operand)
    coef = oracle.interp_coeffs(d)
    ref = oracle.poly_filter(A, a, b, coef, X)
    outs = {}
    for name, ctx in (("csr", c_csr), ("st", c_st)):
        ctx.eig_set_filter("interp")
        Xd = dev_block(X)
        ctx.filter_step(Xd, normalize=False)
        outs[name] = Xd.cpu().numpy()
    assert np.array_equal(outs["csr"], outs["st"])
    assert relF(outs["st"], ref) <= 1e-12


def test_stencil_rejects_non_stencil(arr):
    A = synth.zipf_random(3000, 3)
    ctx = arr.eig_init(arr.to_device_csr(A), k=8, p=1, d=3)
    with pytest.raises(arr.ArrError):
        ctx.eig_set_stencil(3000, 1, 1)
    A = synth.laplacian_3d_potential(9, 2)
    ctx = arr.eig_init(arr.to_device_csr(A), k=8, p=1, d=3)
    with pytest.raises(arr.ArrError):
        ctx.eig_set_stencil(27, 3, 9)  # right n, wrong grid: neighbours outside the 3x3x3 box
    with pytest.raises(arr.ArrError):
        ctx.eig_set_stencil(9, 9, 10)
    ctx.eig_set_stencil(9, 9, 9)
    assert ctx.stencil_points == 7
    ctx.eig_set_stencil(0, 0, 0)
    assert ctx.stencil_points == 0


@pytest.mark.parametrize("kind", ["lap3dV", "st27"])
def test_stencil_solve_and_arr(arr, kind):
    """Full solves (ARR's augmentation SpMMs also take the stencil path): identical
    eigenvalues and iteration counts to the CSR path, and the oracle's certificates."""
    from synth import configs
    spec = configs.SMALL_ANALOGS[kind]
    A, _ = configs.build_config(spec)
    X0 = configs.starting_block(spec)
    N = spec.size
    outs = {}
    for st in (False, True):
        ctx = arr.eig_init(arr.to_device_csr(A), spec.k, spec.p, spec.d, w=spec.w)
        if st:
            ctx.eig_set_stencil(N, N, N)
        ev, res, info = ctx.eig_solve(torch.from_numpy(X0).cuda(), tol=1e-10)
        assert info.converged
        outs[st] = (ev, info.outer, info.sweeps)
    assert outs[True][1:] == outs[False][1:]
    assert np.max(np.abs(outs[True][0] - outs[False][0]) / np.abs(outs[False][0])) <= 1e-13
    lam = np.sort(np.linalg.eigvalsh(A.to_dense()))[::-1][:spec.k]
    assert np.max(np.abs(outs[True][0] - lam) / np.abs(lam)) <= 1e-10


# ---------------------------------------------------------------- lazy MPM normalisation
@pytest.mark.parametrize("kind", ["lap2d_xz", "lap3dV", "lap3dV_even", "st27", "st27_var"])
@pytest.mark.parametrize("w", [24, 98])
@pytest.mark.parametrize("d", [1, 2, 6])
def test_lazy_normalisation(arr, kind, w, d):
    """filter_step(normalize="lazy") leaves X = p_d(A) X unscaled with its norms pending; the
    next filter_step on the same X folds D = 1/norm into its first two degrees, so its output
    is p_d(A) applied to the NORMALISED block (Survey §8a A2: p_d(A)(X D) = p_d(A) X D).
    Checked against the oracle on both kernel families; any other call in between drops the
    pending scale; d odd normalises eagerly."""
    mk, grid, _ = CASES[kind]
    A = mk()
    X0 = synth.gaussian_block(A.n, w, 7)
    c_csr, c_st = _pair(arr, A, grid, w, d)
    a = c_csr.eig_gershgorin_lower()
    b = a + 0.7 * (float(np.abs(A.val).max()) * 8 - a)
    outs = []
    for ctx in (c_csr, c_st):
        ctx.eig_set_interval(a, b)
        X = dev_block(X0, w + 2)
        ctx.filter_step(X, normalize="lazy")
        Y1 = X.cpu().numpy().copy()
        ctx.filter_step(X, normalize=False)
        outs.append((Y1, X.cpu().numpy().copy()))
    y1 = oracle.cheb_filter(A, a, b, d, X0)
    if d % 2 == 1:  # an odd degree count normalises eagerly (the result sits in the scratch block)
        y1 = oracle.mpm_sweep(A, a, b, d, X0)
    y2 = oracle.cheb_filter(A, a, b, d, oracle.mpm_sweep(A, a, b, d, X0))
    for Y1, Y2 in outs:
        assert relF(Y1, y1) <= 1e-12, "lazy sweep output is the unscaled p_d(A) X"
        assert relF(Y2, y2) <= 1e-12, "the pending scale is folded into the next sweep"
    # the two families reduce the column norms in different orders (different CTA partials),
    # so D, and with it the folded sweep, agree to rounding only
    assert relF(outs[0][1], outs[1][1]) <= 1e-14
    # dropped by any other call: the next sweep filters the unscaled block
    ctx = c_csr
    X = dev_block(X0, w + 2)
    ctx.filter_step(X, normalize="lazy")
    ctx.eig_phase_times()
    ctx.filter_step(X, normalize=False)
    assert relF(X.cpu().numpy(), oracle.cheb_filter(A, a, b, d, y1)) <= 1e-12
    # a lazy sweep followed by an eager one equals two MPM sweeps
    X = dev_block(X0, w + 2)
    ctx.filter_step(X, normalize="lazy")
    ctx.filter_step(X, normalize=True)
    ref = oracle.mpm_sweep(A, a, b, d, oracle.mpm_sweep(A, a, b, d, X0))
    assert relF(X.cpu().numpy(), ref) <= 1e-12
    assert np.max(np.abs(np.linalg.norm(X.cpu().numpy(), axis=0) - 1.0)) <= 1e-14
    for cx in (c_csr, c_st):
        cx.close()
