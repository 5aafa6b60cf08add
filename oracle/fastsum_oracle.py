"""Numpy restatement of the reference NFFT fast summation (TEST INFRASTRUCTURE).

Reference: /root/reference/pkg/src/multilap/fastsum.py (cited as fastsum.py:L)
and kernels.py.  The arithmetic below follows the reference step for step
(same sample grids, same scipy.fft transforms, same bincount scatter/gather
order) so its outputs agree with the reference to rounding; it is pinned
against golden vectors produced by the reference itself
(tests/golden/, oracle/gen_golden.py).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
use this module.
"""

import math

import numpy as np
import scipy.fft as sfft
from scipy.special import i0

EPS_B_DEFAULT = 1.0 / 16.0  # fastsum.py:47


class OracleError(Exception):
    """Raised where the reference raises ConfigError / NumericalError."""


# ---------------------------------------------------------------- kernels --
def gaussian_radial(sigma, r):
    """K(r) = exp(-(r/sigma)^2)  (kernels.py:46-51)."""
    r = np.asarray(r, dtype=float)
    return np.exp(-((r / sigma) ** 2))


def laplacian_radial(sigma, r):
    """K(r) = exp(-r/sigma)  (kernels.py:46-51)."""
    return np.exp(-np.asarray(r, dtype=float) / sigma)


def radial(family, sigma, r):
    return gaussian_radial(sigma, r) if family == "gaussian" else laplacian_radial(sigma, r)


def radial_derivs(family, sigma, r, order):
    """d^j/dr^j K(r), j=0..order (kernels.py:53-73; Hermite recurrence)."""
    r = float(r)
    if family == "laplacian":
        e = math.exp(-r / sigma)
        return [e * (-1.0 / sigma) ** j for j in range(order + 1)]
    x = r / sigma
    e = math.exp(-x * x)
    out = [e]
    hm1, h = 0.0, 1.0
    for j in range(1, order + 1):
        hm1, h = h, 2.0 * x * h - 2.0 * (j - 1) * hm1
        out.append(((-1.0 / sigma) ** j) * h * e)
    return out


# ------------------------------------------------------ regularized kernel --
def bridge_coefficients(family, sigma, eps_b, p):
    """Two-point Hermite bridge on the shell, tau in [0,1] (fastsum.py:87-116).

    Degree 2p-1; Q^(j)(0) = eps_b^j K^(j)(1/2-eps_b) for j<p, Q(1) = K(1/2),
    Q^(j)(1) = 0 for 1<=j<p.
    """
    if p < 1 or p > 12:
        raise OracleError("p_nfft out of range")
    r0 = 0.5 - eps_b
    nc = 2 * p
    A = np.zeros((nc, nc))
    rhs = np.zeros(nc)
    der = radial_derivs(family, sigma, r0, p - 1)
    for j in range(p):
        A[j, j] = math.factorial(j)
        rhs[j] = der[j] * eps_b ** j
        for a in range(j, nc):
            A[p + j, a] = math.factorial(a) / math.factorial(a - j)
        rhs[p + j] = float(radial(family, sigma, 0.5)) if j == 0 else 0.0
    return np.linalg.solve(A, rhs)


def regularized_profile(family, sigma, eps_b, p, r):
    """K_R(r): kernel inside r0, bridge on the shell, flat past 1/2 (fastsum.py:119-132)."""
    if not 0.0 < eps_b < 0.5:
        raise OracleError("eps_b out of range")
    r0 = 0.5 - eps_b
    coef = bridge_coefficients(family, sigma, eps_b, p)
    r = np.asarray(r, dtype=float)
    tau = np.clip((r - r0) / eps_b, 0.0, 1.0)
    br = np.polynomial.polynomial.polyval(tau, coef)
    return np.where(r <= r0, radial(family, sigma, np.minimum(r, r0)), br)


def fourier_coefficients(family, sigma, d, N, eps_b, p):
    """bhat = N^-d fftn(K_R on the fftfreq(N) grid), FFT order (fastsum.py:135-151)."""
    ax = sfft.fftfreq(N)
    mesh = np.meshgrid(*([ax] * d), indexing="ij")
    rad = np.sqrt(sum(g * g for g in mesh))
    return sfft.fftn(regularized_profile(family, sigma, eps_b, p, rad)) / N ** d


# ------------------------------------------------------------------ window --
def kb_window(t, m, b):
    """Kaiser-Bessel window phi(t) with its three branches (fastsum.py:158-167)."""
    t = np.asarray(t, dtype=float)
    z = m * m - t * t
    pos = z > 0
    s_pos = np.sqrt(np.where(pos, z, 1.0))
    s_neg = np.sqrt(np.where(pos, 1.0, -z))
    with np.errstate(invalid="ignore"):
        val = np.where(pos, np.sinh(b * s_pos) / s_pos, np.sin(b * s_neg) / s_neg)
    return np.where(z == 0.0, b, val) / math.pi


def kb_deconv(freqs, ng, m, b):
    """1/I0(m sqrt(b^2 - (2 pi k/ng)^2)) (fastsum.py:170-176)."""
    w = 2.0 * math.pi * np.asarray(freqs, dtype=float) / ng
    arg = b * b - w * w
    if np.any(arg <= 0):
        raise OracleError("frequency outside passband")
    return 1.0 / i0(m * np.sqrt(arg))


def _embed(arr, axis, N, ng, split):
    """Size-N FFT-order axis -> size-ng axis (fastsum.py:219-253)."""
    h = N // 2
    a = np.moveaxis(arr, axis, 0)
    out = np.zeros((ng,) + a.shape[1:], dtype=arr.dtype)
    out[:h] = a[:h]
    out[ng - h + 1:] = a[h + 1:]
    if split:
        out[ng - h] = 0.5 * a[h]
        out[h] = 0.5 * a[h]
    else:
        out[ng - h] = a[h]
    return np.moveaxis(out, 0, axis)


class OraclePlan:
    """Everything fastsum_apply needs (fastsum.py:183-216, built as in :256-313)."""

    def __init__(self, family, sigma, d, N=64, m=5, eps_b=EPS_B_DEFAULT, p=5, rho=2.0):
        if d not in (1, 2, 3):
            raise OracleError("d must be 1..3")
        if N < 4 or N % 2:
            raise OracleError("N must be even >= 4")
        if m < 2:
            raise OracleError("m must be >= 2")
        ng = int(round(rho * N))
        if ng < N + 2 or ng % 2:
            raise OracleError("bad oversampling")
        self.family, self.sigma, self.d, self.N, self.m = family, sigma, d, N, m
        self.eps_b, self.p, self.rho, self.ng = eps_b, p, rho, ng
        self.ball_scale = 1.0 / math.sqrt(d)                          # fastsum.py:268
        self.sigma_eff = sigma * self.ball_scale                      # kernels.py:75-82
        self.coeffs = fourier_coefficients(family, self.sigma_eff, d, N, eps_b, p)
        self.b = math.pi * (2.0 - N / ng)                             # fastsum.py:272
        self.deconv_axis = kb_deconv(sfft.fftfreq(N) * N, ng, m, self.b)
        cr = self.coeffs.real
        if np.max(np.abs(self.coeffs.imag)) > 1e-12 * max(1.0, np.max(np.abs(cr))):
            raise OracleError("coefficients not real")
        full = cr
        for ax in range(d):
            full = _embed(full, ax, N, ng, True)
        fq = sfft.fftfreq(ng) * ng
        band = np.abs(fq) <= N // 2
        w = np.zeros(ng)
        w[band] = kb_deconv(fq[band], ng, m, self.b) ** 2
        for ax in range(d):
            sh = [1] * d
            sh[ax] = ng
            full = full * w.reshape(sh)
        full = full * float(ng) ** d
        self.fused = np.ascontiguousarray(full[..., : ng // 2 + 1])     # fastsum.py:294
        self.K0 = 1.0


# ----------------------------------------------------------------- binding --
def box_halfwidth(eps_b):
    return 0.25 - 0.5 * eps_b  # fastsum.py:61-63


def check_box(points, eps_b):
    """fastsum.py:66-80."""
    points = np.asarray(points, dtype=float)
    if points.ndim != 2:
        raise OracleError("points must be 2-d")
    if points.size and not np.all(np.isfinite(points)):
        raise OracleError("non-finite points")
    if points.size and np.max(np.abs(points)) > box_halfwidth(eps_b) + 1e-12:
        raise OracleError("points exceed the admissible box")
    return points


class OracleBinding:
    """Tensor-product flat indices / weights / point ids (fastsum.py:333-372)."""

    def __init__(self, plan, x_torus, sort=None):
        x = np.asarray(x_torus, dtype=float)
        n, d = x.shape
        ng, m, b = plan.ng, plan.m, plan.b
        self.n, self.d, self.grid_size = n, d, ng ** d
        offs = np.arange(-m, m + 1)
        flat = np.zeros((n, 1), dtype=np.int32)
        wt = np.ones((n, 1))
        for a in range(d):
            tx = ng * x[:, a, None]
            u = np.floor(tx).astype(np.int64) + offs[None, :]
            wa = kb_window(tx - u, m, b)
            ia = np.mod(u, ng).astype(np.int32)
            flat = (flat[:, :, None] * np.int32(ng) + ia[:, None, :]).reshape(n, -1)
            wt = (wt[:, :, None] * wa[:, None, :]).reshape(n, -1)
        C = flat.shape[1] if n else 1
        self.flat = flat.ravel()
        self.w = wt.ravel()
        self.pid = np.repeat(np.arange(n, dtype=np.int32), C)
        if sort is None:
            sort = self.grid_size > 200_000
        if sort and n > 1:
            o = np.argsort(self.flat, kind="stable")
            self.flat, self.w, self.pid = self.flat[o], self.w[o], self.pid[o]


def bind(plan, points, sort=None):
    """bind_points (fastsum.py:375-386): box check, x * 1/sqrt(d), binding."""
    pts = check_box(points, plan.eps_b)
    if pts.shape[1] != plan.d:
        raise OracleError("dimension mismatch")
    return OracleBinding(plan, pts * plan.ball_scale, sort=sort)


def spread(binding, v):
    """Scatter-add onto the ng^d grid (fastsum.py:389-391)."""
    return np.bincount(binding.flat, weights=binding.w * v[binding.pid], minlength=binding.grid_size)


def gather(binding, grid):
    """Segmented sum back to the points (fastsum.py:400-406), real or complex grid."""
    vals = binding.w * grid[binding.flat]
    if np.iscomplexobj(vals):
        return (np.bincount(binding.pid, weights=vals.real, minlength=binding.n)
                + 1j * np.bincount(binding.pid, weights=vals.imag, minlength=binding.n))
    return np.bincount(binding.pid, weights=vals, minlength=binding.n)


def convolve_grid(plan, grid_flat):
    """rfftn -> * fused -> irfftn (fastsum.py:492-495)."""
    shape = (plan.ng,) * plan.d
    spec = sfft.rfftn(grid_flat.reshape(shape))
    spec *= plan.fused
    return sfft.irfftn(spec, s=shape).ravel()


def fastsum(plan, v, binding=None, points=None):
    """W v with zero diagonal (fastsum.py:475-497)."""
    v = np.asarray(v, dtype=float)
    if binding is None:
        binding = bind(plan, points)
    if v.shape != (binding.n,):
        raise OracleError("v shape")
    if binding.n == 0:
        return np.zeros(0)
    out = gather(binding, convolve_grid(plan, spread(binding, v)))
    return out - plan.K0 * v


def fastsum_chunked(plan, points, v, chunk=200_000):
    """Chunked restatement for n beyond the binding RAM limit.

    Bind/spread per point chunk, sum the grids, one FFT stage, gather per
    chunk.  Equals fastsum() up to summation order.
    """
    pts = check_box(points, plan.eps_b)
    n = pts.shape[0]
    grid = np.zeros(plan.ng ** plan.d)
    for lo in range(0, n, chunk):
        b = OracleBinding(plan, pts[lo:lo + chunk] * plan.ball_scale, sort=False)
        grid += spread(b, v[lo:lo + chunk])
    conv = convolve_grid(plan, grid)
    out = np.empty(n)
    for lo in range(0, n, chunk):
        b = OracleBinding(plan, pts[lo:lo + chunk] * plan.ball_scale, sort=False)
        out[lo:lo + chunk] = gather(b, conv)
    return out - plan.K0 * v


def direct(points, v, family, sigma):
    """Exact dense W v, zero diagonal (fastsum.py:500-553), small n only."""
    x = np.asarray(points, dtype=float)
    v = np.asarray(v, dtype=float)
    out = np.empty(x.shape[0])
    blk = max(16, int(4e6 // max(x.shape[0], 1)))
    for lo in range(0, x.shape[0], blk):
        d2 = np.sum((x[lo:lo + blk, None, :] - x[None, :, :]) ** 2, axis=2)
        K = np.exp(-d2 / sigma ** 2) if family == "gaussian" else np.exp(-np.sqrt(d2) / sigma)
        out[lo:lo + blk] = K @ v
    return out - v


# ------------------------------------------------------ bare transforms ----
def nfft_adjoint(plan, points, v):
    """ghat_l = sum_j v_j e^{-2 pi i l.x_j}, l in I_N FFT order (fastsum.py:418-445)."""
    pts = np.asarray(points, dtype=float)
    b = OracleBinding(plan, pts, sort=False)
    v = np.asarray(v)
    if np.iscomplexobj(v):
        g = spread(b, np.ascontiguousarray(v.real)) + 1j * spread(b, np.ascontiguousarray(v.imag))
    else:
        g = spread(b, v.astype(float))
    gh = sfft.fftn(g.reshape((plan.ng,) * plan.d))
    h = plan.N // 2
    keep = np.r_[0:h, plan.ng - h:plan.ng]
    gh = gh[np.ix_(*([keep] * plan.d))]
    for ax in range(plan.d):
        sh = [1] * plan.d
        sh[ax] = plan.N
        gh = gh * plan.deconv_axis.reshape(sh)
    return gh


def nfft_forward(plan, coeffs, points):
    """f_i = sum_l c_l e^{+2 pi i l.x_i} (fastsum.py:448-468)."""
    c = np.asarray(coeffs, dtype=complex)
    for ax in range(plan.d):
        sh = [1] * plan.d
        sh[ax] = plan.N
        c = c * plan.deconv_axis.reshape(sh)
    full = c
    for ax in range(plan.d):
        full = _embed(full, ax, plan.N, plan.ng, False)
    grid = sfft.ifftn(full) * float(plan.ng) ** plan.d
    b = OracleBinding(plan, np.asarray(points, dtype=float), sort=False)
    return gather(b, grid.ravel())
