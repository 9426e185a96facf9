"""ORACLE — test infrastructure only (see oracle/__init__.py).

The oracle's own dense steps, written from textbook definitions so that a reader can
check them by eye (no LAPACK on the oracle path; scipy/numpy LAPACK routines appear
only in tests as independent cross-checks):

* ``qr_pivoted``  Householder QR with column pivoting (Businger & Golub 1965;
  Golub & Van Loan, Alg. 5.4.1): the "orthonormalize Z to obtain U in orth(Z)" step of
  Alg. RR with the rank cut r = #{|R_ii| > n eps |R_11|}.
* ``jacobi_eigh``  cyclic Jacobi for a symmetric matrix (Jacobi 1846; Golub & Van Loan
  §8.5): the "H = V^T Sigma V" step of Alg. RR.  Rotations are applied in
  the round-robin (tournament) ordering, m/2 disjoint (p, q) pairs per round, each
  rotation the classical one that zeroes H_pq.
* ``gram`` / ``gemm``  the tall-skinny products of the CGS2 variant as plain
  row-panel loops around a library matmul step (a matmul is allowed as one step).

Cost notes: qr_pivoted streams the n x m block once per reflector (m * 8 n m bytes);
jacobi_eigh is O(m^3) per sweep with ~6-10 sweeps to fp64 convergence.
"""
from __future__ import annotations

import numpy as np

EPS = np.finfo(np.float64).eps


# --------------------------------------------------------------------------- QR
def _rank1_sub(B: np.ndarray, v: np.ndarray, w: np.ndarray, chunk: int = 8192):
    """B -= v w^T, in row chunks (keeps the outer-product temporary small)."""
    for r0 in range(0, B.shape[0], chunk):
        B[r0:r0 + chunk] -= np.outer(v[r0:r0 + chunk], w)


def _form_q(V: list, betas: list, n: int, t: int, nb: int = 32) -> np.ndarray:
    """Q = H_0 H_1 ... H_{t-1} [I_t; 0] from reflectors v_k (v_k[0] = 1, length n - k),
    applied in compact-WY groups of nb (I - V T V^T, Schreiber & Van Loan) in reverse."""
    Q = np.zeros((n, t))
    Q[np.arange(t), np.arange(t)] = 1.0
    for k0 in range(((t - 1) // nb) * nb, -1, -nb):
        k1 = min(t, k0 + nb)
        b = k1 - k0
        Vp = np.zeros((n - k0, b))
        for j in range(b):
            Vp[j:, j] = V[k0 + j]
        T = np.zeros((b, b))
        for j in range(b):
            T[j, j] = betas[k0 + j]
            if j:
                T[:j, j] = -betas[k0 + j] * (T[:j, :j] @ (Vp[:, :j].T @ Vp[:, j]))
        Q[k0:, k0:] -= Vp @ (T @ (Vp.T @ Q[k0:, k0:]))
    return Q


def qr_pivoted(Z: np.ndarray, want_q: bool = True):
    """Z[:, piv] = Q R, Q n x m with orthonormal columns, R upper triangular with
    |R_00| >= |R_11| >= ... (column pivoting on the largest remaining 2-norm).

    Returns (Q, R, piv).  Householder reflectors H_k = I - beta_k v_k v_k^T with
    v_k[k] = 1 (Golub & Van Loan Alg. 5.1.1), applied to the trailing columns; the
    trailing column norms are downdated (nrm_j^2 -= R_kj^2) and recomputed when they
    have lost more than 99% to cancellation (Golub & Van Loan §5.4.1); Q is
    accumulated from the reflectors in reverse order (compact WY groups)."""
    A = np.array(Z, dtype=np.float64, copy=True)
    n, m = A.shape
    t = min(n, m)
    piv = np.arange(m)
    V = []       # reflector vectors (length n - k)
    betas = []
    nrm2 = np.einsum("ij,ij->j", A, A)
    ref2 = nrm2.copy()
    for k in range(t):
        j = k + int(np.argmax(nrm2[k:]))
        if j != k:
            A[:, [k, j]] = A[:, [j, k]]
            piv[[k, j]] = piv[[j, k]]
            nrm2[[k, j]] = nrm2[[j, k]]
            ref2[[k, j]] = ref2[[j, k]]
        x = A[k:, k].copy()
        alpha = np.sqrt(x @ x)
        if alpha == 0.0:
            V.append(np.zeros(n - k))
            betas.append(0.0)
            continue
        # v = x + sign(x_0) ||x|| e_0, scaled so v_0 = 1; beta = 2 / v^T v
        s = 1.0 if x[0] >= 0 else -1.0
        v = x.copy()
        v[0] = x[0] + s * alpha
        v /= v[0]
        beta = 2.0 / float(v @ v)
        # H_k applied to the trailing columns: A <- A - beta v (v^T A)
        wv = beta * (v @ A[k:, k:])
        _rank1_sub(A[k:, k:], v, wv)
        A[k + 1:, k] = 0.0
        V.append(v)
        betas.append(beta)
        # downdate the trailing norms by the new row of R
        if k + 1 < m:
            nrm2[k + 1:] -= A[k, k + 1:] ** 2
            bad = np.nonzero(nrm2[k + 1:] <= 1e-2 * ref2[k + 1:])[0] + k + 1
            for c in bad:
                nrm2[c] = A[k + 1:, c] @ A[k + 1:, c]
                ref2[c] = nrm2[c]
    R = np.triu(A[:t, :])
    if not want_q:
        return None, R, piv
    return _form_q(V, betas, n, t), R, piv


# --------------------------------------------------------------------------- eig
def _round_robin(m: int):
    """Rounds of disjoint pairs covering every (p, q), p < q, once (circle method)."""
    players = list(range(m)) + ([-1] if m % 2 else [])
    M = len(players)
    rounds = []
    for _ in range(M - 1):
        pairs = [(players[i], players[M - 1 - i]) for i in range(M // 2)]
        pairs = [(min(a, b), max(a, b)) for a, b in pairs if a >= 0 and b >= 0]
        rounds.append((np.array([p for p, _ in pairs], dtype=np.int64),
                       np.array([q for _, q in pairs], dtype=np.int64)))
        players = [players[0]] + [players[-1]] + players[1:-1]
    return rounds


def jacobi_eigh(H: np.ndarray, tol: float = None, max_sweeps: int = 60):
    """Eigen-decomposition of a symmetric H = V diag(lam) V^T by cyclic Jacobi.

    Each rotation in the (p, q) plane is the classical one (Golub & Van Loan §8.5.2):
        theta = (H_qq - H_pp) / (2 H_pq),  t = sign(theta) / (|theta| + sqrt(1 + theta^2)),
        c = 1 / sqrt(1 + t^2),  s = t c,
    so that the rotated H_pq is zero.  A round applies m/2 disjoint rotations at once
    (they commute); a sweep is m-1 rounds.  Stops when the off-diagonal Frobenius norm
    is <= tol * ||H||_F (default eps; Jacobi converges quadratically, so the last sweep
    typically takes it from ~sqrt(eps) to far below).  Returns (lam ascending, V)."""
    A = np.array(H, dtype=np.float64, copy=True)
    m = A.shape[0]
    A = 0.5 * (A + A.T)
    V = np.eye(m)
    if m == 1:
        return A.diagonal().copy(), V
    tol = EPS if tol is None else tol
    fro = np.linalg.norm(A)
    rounds = _round_robin(m)
    for _ in range(max_sweeps):
        off = np.linalg.norm(A - np.diag(A.diagonal()))  # direct: no cancellation
        if off <= tol * fro:
            break
        for P, Q in rounds:
            apq = A[P, Q]
            app = A[P, P]
            aqq = A[Q, Q]
            nz = np.abs(apq) > 0.0
            c = np.ones_like(apq)
            s = np.zeros_like(apq)
            if np.any(nz):
                with np.errstate(over="ignore"):
                    theta = (aqq[nz] - app[nz]) / (2.0 * apq[nz])
                t = np.where(theta >= 0, 1.0, -1.0) / (np.abs(theta) + np.hypot(1.0, theta))
                c[nz] = 1.0 / np.sqrt(1.0 + t * t)
                s[nz] = t * c[nz]
            # A <- J^T A J with J the product of the disjoint rotations:
            # columns p, q first, then rows p, q
            Ap, Aq = A[:, P].copy(), A[:, Q].copy()
            A[:, P] = c * Ap - s * Aq
            A[:, Q] = s * Ap + c * Aq
            Ap, Aq = A[P, :].copy(), A[Q, :].copy()
            A[P, :] = c[:, None] * Ap - s[:, None] * Aq
            A[Q, :] = s[:, None] * Ap + c[:, None] * Aq
            A[P, Q] = 0.0
            A[Q, P] = 0.0
            Vp, Vq = V[:, P].copy(), V[:, Q].copy()
            V[:, P] = c * Vp - s * Vq
            V[:, Q] = s * Vp + c * Vq
    lam = A.diagonal().copy()
    order = np.argsort(lam, kind="stable")
    return lam[order], V[:, order]


# --------------------------------------------------------------------------- tall-skinny products
PANEL = 65536  # rows per panel


def gram(X: np.ndarray, Y: np.ndarray) -> np.ndarray:
    """G = X^T Y summed over row panels in order (each panel one library matmul)."""
    G = np.zeros((X.shape[1], Y.shape[1]))
    for r0 in range(0, X.shape[0], PANEL):
        G += X[r0:r0 + PANEL].T @ Y[r0:r0 + PANEL]
    return G


def gemm(X: np.ndarray, B: np.ndarray) -> np.ndarray:
    """X B, row panel by row panel."""
    out = np.empty((X.shape[0], B.shape[1]))
    for r0 in range(0, X.shape[0], PANEL):
        out[r0:r0 + PANEL] = X[r0:r0 + PANEL] @ B
    return out


def cholesky_upper(G: np.ndarray) -> np.ndarray:
    """G = R^T R, R upper triangular (Cholesky-Banachiewicz, row by row); raises
    FloatingPointError on a non-positive pivot."""
    m = G.shape[0]
    R = np.zeros_like(G)
    for i in range(m):
        d = G[i, i] - R[:i, i] @ R[:i, i]
        if not d > 0.0:
            raise FloatingPointError(f"Cholesky pivot {i} = {d}")
        R[i, i] = np.sqrt(d)
        R[i, i + 1:] = (G[i, i + 1:] - R[:i, i] @ R[:i, i + 1:]) / R[i, i]
    return R


def solve_upper_right(X: np.ndarray, R: np.ndarray) -> np.ndarray:
    """X R^{-1} for upper-triangular R, by forward substitution over columns:
    out[:, j] = (X[:, j] - out[:, :j] R[:j, j]) / R_jj."""
    out = np.empty_like(X)
    for j in range(R.shape[0]):
        out[:, j] = (X[:, j] - out[:, :j] @ R[:j, j]) / R[j, j]
    return out


def qr_blocked(W: np.ndarray, nb: int = 32):
    """W = Q R (thin), unpivoted Householder QR in panels of nb columns with the
    compact WY form H_0 ... H_{b-1} = I - V T V^T (Schreiber & Van Loan 1989; Golub &
    Van Loan §5.2.3): each panel is factored reflector by reflector (Alg. 5.1.1), the
    trailing columns are updated with Q_panel^T = I - V T^T V^T (two matmul steps) and
    Q is accumulated panel by panel in reverse.  Backward stable for any conditioning;
    a rank-deficient W still gets m orthonormal columns."""
    A = np.array(W, dtype=np.float64, copy=True)
    n, m = A.shape
    panels = []
    for k0 in range(0, m, nb):
        k1 = min(m, k0 + nb)
        b = k1 - k0
        Vp = np.zeros((n - k0, b))
        betas = np.zeros(b)
        for j in range(b):
            c = k0 + j
            x = A[c:, c]
            alpha = np.linalg.norm(x)
            if alpha == 0.0:
                continue
            s = 1.0 if x[0] >= 0 else -1.0
            v = x.copy()
            v[0] = x[0] + s * alpha
            v /= v[0]
            beta = 2.0 / float(v @ v)
            A[c:, c:k1] -= beta * np.outer(v, v @ A[c:, c:k1])
            A[c + 1:, c] = 0.0
            Vp[j:, j] = v
            betas[j] = beta
        T = np.zeros((b, b))
        for j in range(b):
            T[j, j] = betas[j]
            if j:
                T[:j, j] = -betas[j] * (T[:j, :j] @ (Vp[:, :j].T @ Vp[:, j]))
        if k1 < m:
            A[k0:, k1:] -= Vp @ (T.T @ (Vp.T @ A[k0:, k1:]))
        panels.append((k0, Vp, T))
    R = np.triu(A[:m, :])
    Q = np.zeros((n, m))
    Q[np.arange(m), np.arange(m)] = 1.0
    for k0, Vp, T in reversed(panels):
        Q[k0:, k0:] -= Vp @ (T @ (Vp.T @ Q[k0:, k0:]))
    return Q, R


def solve_gepp(M: np.ndarray, f: np.ndarray) -> np.ndarray:
    """M a = f by Gaussian elimination with partial pivoting and back substitution
    (Golub & Van Loan Alg. 3.4.1); M square."""
    M = np.array(M, dtype=np.float64, copy=True)
    a = np.array(f, dtype=np.float64, copy=True)
    m = M.shape[0]
    for k in range(m - 1):
        piv = k + int(np.argmax(np.abs(M[k:, k])))
        if piv != k:
            M[[k, piv]] = M[[piv, k]]
            a[[k, piv]] = a[[piv, k]]
        if M[k, k] == 0.0:
            raise FloatingPointError("singular system")
        l = M[k + 1:, k] / M[k, k]
        M[k + 1:, k:] -= np.outer(l, M[k, k:])
        a[k + 1:] -= l * a[k]
    for k in range(m - 1, -1, -1):
        a[k] = (a[k] - M[k, k + 1:] @ a[k + 1:]) / M[k, k]
    return a
