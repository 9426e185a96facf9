"""The opt-in union-staged SpMM (csrc/spmm_union.cu, ARRABIT_UNION=1): the same fused
filter degree (Eq. cheby-poly), residual pass (Eq. resi) and solve
as the default tiled kernels.  Per-row sums run in CSR order in both, so un-normalised
filter output is bitwise equal; column norms (different CTA partition of the sums of
squares) agree to rounding; both match the oracle."""
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


def _ctx(arr, A, w, p, d, union, monkeypatch, rows=None, k=None):
    monkeypatch.setenv("ARRABIT_UNION", "1" if union else "0")
    monkeypatch.setenv("ARRABIT_UNION_MIN", "0")  # take the union path whatever the reuse
    monkeypatch.setenv("ARRABIT_UNION_VERBOSE", "1")
    if rows:
        monkeypatch.setenv("ARRABIT_UNION_ROWS", str(rows))
    return arr.eig_init(arr.to_device_csr(A), k=k or w, p=p, d=d, w=w)


@pytest.mark.parametrize("kind", ["lap2d", "lap3dV", "st27"])
@pytest.mark.parametrize("rows", [7, 64])
def test_union_filter_bitwise_and_oracle(arr, kind, rows, monkeypatch, capfd):
    spec = configs.SMALL_ANALOGS[kind]
    A, _ = configs.build_config(spec)
    w, d = 22, 7  # w % 16 = 6: a ragged last panel
    X = synth.gaussian_block(A.n, w, 3)
    a = oracle.gershgorin_lower(A)
    b = a + 0.7 * (np.abs(A.val).max() * 8 - a)
    out = {}
    for union in (False, True):
        ctx = _ctx(arr, A, w, 1, d, union, monkeypatch, rows)
        if union:
            assert "-> on" in capfd.readouterr().err  # the plan was built and taken
        ctx.eig_set_interval(a, b)
        Xd = torch.from_numpy(X.copy()).cuda()
        ctx.filter_step(Xd, normalize=False)
        nrm = torch.empty(w, dtype=torch.float64, device="cuda")
        Xn = torch.from_numpy(X.copy()).cuda()
        ctx.filter_step(Xn, normalize=True, colnorm=nrm)
        out[union] = (Xd.cpu().numpy(), Xn.cpu().numpy(), nrm.cpu().numpy())
        ctx.close()
    assert np.array_equal(out[True][0], out[False][0])  # same per-row fma sequence
    assert np.max(np.abs(out[True][2] - out[False][2]) / out[False][2]) <= 1e-14
    ref = oracle.cheb_filter(A, a, b, d, X)
    assert np.linalg.norm(out[True][0] - ref) / np.linalg.norm(ref) <= 1e-12
    refn = ref / oracle.col_norms(ref)
    assert np.linalg.norm(out[True][1] - refn) / np.linalg.norm(refn) <= 1e-12


@pytest.mark.parametrize("kind", ["lap2d", "st27"])
def test_union_solve_and_residuals(arr, kind, monkeypatch, capfd):
    spec = configs.SMALL_ANALOGS[kind]
    A, _ = configs.build_config(spec)
    ctx = _ctx(arr, A, spec.w, spec.p, spec.d, True, monkeypatch, k=spec.k)
    assert "-> on" in capfd.readouterr().err
    Xd = torch.from_numpy(synth.starting_block(spec)).cuda()
    ev, res, info = ctx.eig_solve(Xd, tol=spec.tol, maxit=200)
    assert info.converged == 1
    lam = np.sort(np.linalg.eigvalsh(A.to_dense()))[::-1][:spec.k]
    assert np.max(np.abs(ev - lam) / np.maximum(1, np.abs(lam))) < 1e-10
    Y = Xd[:, :spec.k].cpu().numpy()
    assert np.all(oracle.residuals(A, Y, ev) <= 1.01 * spec.tol)
    # the residual pass itself (shifted SpMM + fused norms) against the oracle
    r = ctx.residuals(Xd[:, :spec.k].contiguous(), ev)
    assert np.allclose(r, oracle.residuals(A, Y, ev), rtol=1e-8, atol=1e-15)
