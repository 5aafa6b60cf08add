"""Numpy restatement of the reference solvers on the hot path (TEST INFRASTRUCTURE).

Reference files (/root/reference/pkg/src/multilap/): graphs.py (normalized
Laplacian), krylov.py (thick-restart Lanczos, Lanczos f(A)v / PKSM),
powermean.py (M_p^p operator, eigen-mapping), allencahn.py (multiclass
convexity splitting).  Operators are plain callables v -> A v on numpy
vectors so the same code drives oracle kernel layers and dense test
matrices.  Pinned against reference-generated golden vectors.
"""

import math

import numpy as np


class OracleNumericalError(Exception):
    pass


# ----------------------------------------------------------------- graphs --
class OracleLayer:
    """Weights callable + degrees + shift (graphs.py:147-183)."""

    def __init__(self, matvec, n, shift=0.0, degrees=None):
        self.matvec = matvec
        self.n = n
        self.shift = float(shift)
        if degrees is None:
            degrees = matvec(np.ones(n))                      # graphs.py:176-177
            bad = np.flatnonzero(degrees <= 1e-300)
            if bad.size:
                raise OracleNumericalError(f"node {bad[0]} has zero degree")
        self.degrees = degrees
        self.isd = 1.0 / np.sqrt(degrees)                     # graphs.py:159-165

    def shifted(self, shift):
        return OracleLayer(self.matvec, self.n, shift, self.degrees)


def sym_laplacian(layer, v):
    """(1+delta) v - D^-1/2 W D^-1/2 v (graphs.py:197-201)."""
    v = np.asarray(v, dtype=float)
    return (1.0 + layer.shift) * v - layer.isd * layer.matvec(layer.isd * v)


# ----------------------------------------------------------------- krylov --
def _cgs2(w, V, cols):
    """Two-pass classical Gram-Schmidt (krylov.py:65-71)."""
    B = V[:, :cols]
    h = B.T @ w
    w = w - B @ h
    h2 = B.T @ w
    w -= B @ h2
    return w, h + h2


def symmetry_probe(n, apply, tol=1e-8):
    """krylov.py:27-37 with default_rng(0) probes."""
    rng = np.random.default_rng(0)
    for _ in range(2):
        x = rng.standard_normal(n)
        y = rng.standard_normal(n)
        ax = apply(x)
        ay = apply(y)
        sc = max(np.linalg.norm(ax) * np.linalg.norm(y), 1e-300)
        if abs(ax @ y - x @ ay) > tol * sc:
            raise OracleNumericalError("symmetry probe failed")


def lanczos_top(n, apply, k, tol=1e-8, max_subspace=None, max_restarts=60, seed=0):
    """Thick-restart Lanczos, k largest pairs, descending (krylov.py:74-169).

    Returns (values, vectors, residuals, matvecs, restarts).
    """
    if not 1 <= k < n:
        raise ValueError("need 1 <= k < n")
    symmetry_probe(n, apply)
    if max_subspace is None:
        max_subspace = max(2 * k + 10, 20)
    ms = int(min(max_subspace, n))
    if ms < k + 2:
        ms = min(n, k + 2)
    keep = min(ms - 1, k + max(2, k // 2))
    V = np.empty((n, ms))
    H = np.zeros((ms, ms))
    rng = np.random.default_rng(seed)                         # krylov.py:57-62
    v0 = np.ones(n) + 1e-2 * rng.standard_normal(n)
    V[:, 0] = v0 / np.linalg.norm(v0)
    u = V[:, 0].copy()
    s = 0
    matvecs = 0
    fill = np.random.default_rng(seed + 1)
    beta = 0.0
    for restart in range(max_restarts + 1):
        j = s
        while j < ms:
            V[:, j] = u
            w = apply(u)
            matvecs += 1
            w, h = _cgs2(w, V, j + 1)
            H[: j + 1, j] = h
            H[j, : j + 1] = h
            beta = np.linalg.norm(w)
            j += 1
            if beta <= 1e-13 * max(1.0, np.abs(H[:j, :j]).max()):
                if j >= n:
                    break
                u = fill.standard_normal(n)
                u, _ = _cgs2(u, V, j)
                nu = np.linalg.norm(u)
                if nu <= 1e-13:
                    break
                u /= nu
                beta = 0.0
            else:
                u = w / beta
        sd = j
        theta, S = np.linalg.eigh(H[:sd, :sd])
        order = np.argsort(theta)[::-1]
        theta, S = theta[order], S[:, order]
        scale = max(abs(theta[0]), abs(theta[-1]), 1e-300)
        res = np.abs(beta * S[sd - 1, :])
        if np.all(res[:k] <= tol * scale) or sd >= n:
            return theta[:k], V[:, :sd] @ S[:, :k], res[:k], matvecs, restart
        if restart == max_restarts:
            break
        V[:, :keep] = V[:, :sd] @ S[:, :keep]
        H[:, :] = 0.0
        H[:keep, :keep] = np.diag(theta[:keep])
        s = keep
    raise OracleNumericalError("Lanczos did not converge")


def lanczos_fn(n, apply, v, fn, krylov_dim=50, tol=1e-8, trace=None):
    """y = |v| V_s f(T_s) e_1 with the reference stopping rule (krylov.py:172-216).

    `trace`, if a list, receives the number of Krylov steps taken.
    """
    v = np.asarray(v, dtype=float)
    nv = np.linalg.norm(v)
    if nv == 0.0:
        return np.zeros(n)
    dim = int(min(krylov_dim, n))
    V = np.empty((n, dim))
    al = np.empty(dim)
    be = np.empty(dim)
    V[:, 0] = v / nv
    y_prev = None
    s = 0
    while True:
        w = apply(V[:, s])
        al[s] = V[:, s] @ w
        w, _ = _cgs2(w, V, s + 1)
        beta = np.linalg.norm(w)
        be[s] = beta
        s += 1
        T = np.diag(al[:s])
        if s > 1:
            T += np.diag(be[: s - 1], 1) + np.diag(be[: s - 1], -1)
        lam, Q = np.linalg.eigh(T)
        y = nv * (V[:, :s] @ (Q @ (fn(lam) * Q[0, :])))
        if y_prev is not None and np.linalg.norm(y - y_prev) <= tol * max(np.linalg.norm(y), 1e-300):
            break
        if beta <= 1e-13 * max(1.0, np.abs(al[:s]).max()) or s >= dim:
            break
        y_prev = y
        V[:, s] = w / beta
    if trace is not None:
        trace.append(s)
    return y


def power_fn(p):
    """lambda^p with the PSD / positivity checks (krylov.py:230-242)."""
    def fn(lam):
        if lam.min() < -1e-10:
            raise OracleNumericalError("not PSD")
        lam = np.maximum(lam, 0.0)
        if p < 0 and lam.min() <= 0.0:
            raise OracleNumericalError("zero eigenvalue with negative power")
        return lam ** p
    return fn


def pksm(layer, p, v, krylov_dim=50, tol=1e-8, trace=None):
    """(L_sym + delta)^p v (krylov.py:219-244)."""
    return lanczos_fn(layer.n, lambda x: sym_laplacian(layer, x), v, power_fn(p),
                      krylov_dim=krylov_dim, tol=tol, trace=trace)


# -------------------------------------------------------------- powermean --
def default_shift(p):
    return math.log1p(abs(p)) if p < 0 else 0.0               # powermean.py:27-28


def apply_Lp_power(layers, p, v, krylov_dim=50, tol=1e-8, trace=None):
    """(1/T) sum_t PKSM(layer_t) (powermean.py:80-95), layers already shifted."""
    out = np.zeros(len(v))
    for lay in layers:
        out += pksm(lay, p, v, krylov_dim, tol, trace)
    return out / len(layers)


def apply_one_minus_L1(layers, v):
    """(1/T) sum_t isd_t W_t (isd_t v) (powermean.py:64-77)."""
    out = np.zeros(len(v))
    for lay in layers:
        out += lay.isd * lay.matvec(lay.isd * v)
    return out / len(layers)


def power_mean_eigs(layers, p, k, tol=1e-8, max_subspace=None, max_restarts=60,
                    krylov_dim=50, inner_tol=None, seed=0, delta=None, stats=None):
    """k smallest eigenpairs of M_p, ascending (powermean.py:130-189); p=1 or p<0."""
    n = layers[0].n
    if p == 1:
        work = [lay.shifted(0.0) for lay in layers]
        op = lambda v: apply_one_minus_L1(work, v)
        vals, vecs, _, mv, rs = lanczos_top(n, op, k, tol, max_subspace, max_restarts, seed)
        values = np.maximum(1.0 - vals, 0.0)
    elif p < 0:
        dl = default_shift(p) if delta is None else delta
        work = [lay.shifted(dl) for lay in layers]
        itol = tol if inner_tol is None else inner_tol
        op = lambda v: apply_Lp_power(work, p, v, krylov_dim, itol)
        vals, vecs, _, mv, rs = lanczos_top(n, op, k, tol, max_subspace, max_restarts, seed)
        if vals.min() <= 0.0:
            raise OracleNumericalError("power mean spectrum not positive")
        values = vals ** (1.0 / p)
    else:
        raise ValueError("oracle covers p == 1 and p < 0")
    if stats is not None:
        stats.update(matvecs=mv, restarts=rs)
    return values, vecs


# -------------------------------------------------------------- allencahn --
def simplex_project(U):
    """Row-wise Euclidean projection onto the simplex (allencahn.py:105-124)."""
    U = np.atleast_2d(np.asarray(U, dtype=float))
    n, m = U.shape
    s = -np.sort(-U, axis=1)
    cs = np.cumsum(s, axis=1)
    j = np.arange(1, m + 1)
    ok = s + (1.0 - cs) / j > 0
    rho = m - 1 - np.argmax(ok[:, ::-1], axis=1)
    tau = (1.0 - cs[np.arange(n), rho]) / (rho + 1)
    return np.maximum(U + tau[:, None], 0.0)


def well_force(U):
    """T(U): derivative of the multi-well potential (allencahn.py:127-154)."""
    U = np.asarray(U, dtype=float)
    aU = np.abs(U)
    A = aU.sum(axis=1, keepdims=True) - aU + np.abs(U - 1.0)
    B = 0.25 * A * A
    n, m = B.shape
    left = np.ones_like(B)
    right = np.ones_like(B)
    for q in range(1, m):
        left[:, q] = left[:, q - 1] * B[:, q - 1]
    for q in range(m - 2, -1, -1):
        right[:, q] = right[:, q + 1] * B[:, q + 1]
    wtd = A * left * right
    return 0.5 * wtd.sum(axis=1, keepdims=True) - wtd


def allen_cahn(values, vectors, F, fidelity, epsilon=5e-3, omega0=1000.0, c=None,
               dt=0.01, tolerance=1e-6, max_iter=300):
    """Convexity-splitting iteration in the eigenbasis (allencahn.py:172-223).

    Returns (scores, iterations, converged).
    """
    m = F.shape[1]
    cv = omega0 + 3.0 / epsilon if c is None else c
    denom = 1.0 + cv * dt + epsilon * dt * np.asarray(values)
    U = np.full(F.shape, 1.0 / m)                              # allencahn.py:157-162
    lab = fidelity > 0
    U[lab] = F[lab]
    fid = fidelity[:, None]
    conv = False
    it_done = 0
    for it in range(1, max_iter + 1):
        R = (1.0 + cv * dt) * U - (dt / (2.0 * epsilon)) * well_force(U) - dt * fid * (U - F)
        Vc = (vectors.T @ R) / denom[:, None]
        Un = simplex_project(vectors @ Vc)
        dff = Un - U
        num = np.max(np.einsum("ij,ij->i", dff, dff))
        den = np.max(np.einsum("ij,ij->i", Un, Un))
        if den <= 0 or not np.isfinite(num):
            raise OracleNumericalError("degenerate iterate")
        U = Un
        it_done = it
        if num / den <= tolerance:
            conv = True
            break
    return U, it_done, conv


def predict(scores):
    return np.argmax(np.asarray(scores), axis=1)             # allencahn.py:226-229


def corner_distances(U):
    """A_iq = sum_l |U_il| - |U_iq| + |U_iq - 1| (allencahn.py:127-130)."""
    U = np.asarray(U, dtype=float)
    aU = np.abs(U)
    return aU.sum(axis=1, keepdims=True) - aU + np.abs(U - 1.0)


def gl_energy(U, values, vectors, F, fidelity, epsilon, L_dense=None):
    """Ginzburg-Landau diagnostic energy (allencahn.py:232-252): Dirichlet term in
    the eigenbasis (0.5 eps sum lambda C^2, C = Phi^T U) or with a dense
    Laplacian (0.5 eps sum U * (L U)), double-well sum prod_q A^2/4 / (2 eps),
    fidelity 0.5 sum_i fid_i |F_i - U_i|^2."""
    U = np.asarray(U, dtype=float)
    if L_dense is None:
        C = vectors.T @ U
        dirichlet = 0.5 * epsilon * float(np.sum(np.asarray(values)[:, None] * C * C))
    else:
        dirichlet = 0.5 * epsilon * float(np.sum(U * (np.asarray(L_dense) @ U)))
    A = corner_distances(U)
    well = float(np.sum(np.prod(0.25 * A * A, axis=1))) / (2.0 * epsilon)
    diff = F - U
    fid = 0.5 * float(fidelity @ np.einsum("ij,ij->i", diff, diff))
    return dirichlet + well + fid


def binary_allen_cahn(values, vectors, f, epsilon=5e-3, omega0=1000.0, c=None, dt=0.01, tolerance=1e-6,
                      max_iter=300):
    """Two-class spectral scheme with the (u^2-1)^2/4 well (allencahn.py:261-309).

    Returns (scores, iterations, converged)."""
    f = np.asarray(f, dtype=float)
    cv = omega0 + 3.0 / epsilon if c is None else c
    fid = np.where(f != 0, omega0, 0.0)
    denom = 1.0 + cv * dt + epsilon * dt * np.asarray(values)
    lead = 1.0 + cv * dt + dt / epsilon
    v = vectors.T @ f
    u = vectors @ v
    conv = False
    it_done = 0
    for it in range(1, max_iter + 1):
        rhs = lead * v
        rhs -= (dt / epsilon) * (vectors.T @ (u ** 3))
        rhs -= dt * (vectors.T @ (fid * (u - f)))
        v = rhs / denom
        un = vectors @ v
        num = np.max((un - u) ** 2)
        den = np.max(un ** 2)
        u = un
        it_done = it
        if den <= 0:
            conv = True
            break
        if not np.isfinite(num):
            raise OracleNumericalError("binary iterate degenerated")
        if num / den <= tolerance:
            conv = True
            break
    return u, it_done, conv


def predict_binary(scores):
    return np.where(np.asarray(scores) >= 0, 1, -1)          # allencahn.py:312-314
