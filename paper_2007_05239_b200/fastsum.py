"""NFFT fast kernel summation on B200 -- drop-in for multilap.fastsum.

Public surface (fastsum.py of the reference): build_plan, bind_points,
fastsum_apply, direct_apply, nfft_adjoint, nfft_forward, validate_box,
box_halfwidth, kernel_fourier_coefficients, regularized_radial, FastsumPlan,
PointBinding, DEFAULT_*.

Host side (numpy, one time per plan): the regularized kernel, its Fourier
coefficients, the Kaiser-Bessel deconvolution, the fused weights (all as in
fastsum.py:87-313), plus the device tables: fused weights on the |k| <= N/2
band, the twiddles of the pruned DFT between the active sub-box and the
band, and the window polynomials (see csrc/mlb_window.cuh).  Every apply runs
in libmlb.so (spread -> pruned DFT * fused -> gather); there is no CPU path.
"""

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ConfigError, NumericalError
from .kernels import KernelSpec

DEFAULT_N = 64
DEFAULT_M = 5
DEFAULT_EPS_B = 1.0 / 16.0
DEFAULT_P = 5
DEFAULT_RHO = 2.0
BOX_TOL = 1e-12  # validate_box slack (fastsum.py:73)

_fft_workers = 1


def set_fft_workers(n):
    """Kept for API compatibility (fastsum.py:56-58); the device FFT has no workers."""
    global _fft_workers
    _fft_workers = max(1, int(n))


def box_halfwidth(eps_b):
    return 0.25 - 0.5 * eps_b


def validate_box(points, eps_b):
    """Componentwise box check |x|_inf <= 1/4 - eps_b/2 (fastsum.py:66-80)."""
    points = np.asarray(points, dtype=float)
    if points.ndim != 2:
        raise ConfigError(f"points must be a 2-d array, got shape {points.shape}")
    if points.size and not np.all(np.isfinite(points)):
        raise ConfigError("points contain non-finite values")
    hw = box_halfwidth(eps_b)
    if points.size:
        worst = float(np.max(np.abs(points)))
        if worst > hw + BOX_TOL:
            raise ConfigError(
                f"points exceed the admissible box: max |coord| = {worst:.6g} "
                f"> 1/4 - eps_b/2 = {hw:.6g}")
    return points


# ------------------------------------------------------------ plan math ----
def _bridge(kernel, eps_b, p_deg):
    """Hermite bridge on the shell r in (1/2-eps_b, 1/2] in tau = (r-r0)/eps_b
    (degree 2p-1; value+derivatives match at r0, flat at 1/2; fastsum.py:87-116)."""
    p = int(p_deg)
    if p < 1 or p > 12:
        raise ConfigError(f"p_nfft must be in [1, 12], got {p_deg}")
    r0 = 0.5 - eps_b
    n = 2 * p
    j = np.arange(p)
    a = np.arange(n)
    A = np.zeros((n, n))
    A[j, j] = [math.factorial(int(x)) for x in j]
    for jj in range(p):
        A[p + jj, jj:] = [math.factorial(int(x)) / math.factorial(int(x) - jj) for x in a[jj:]]
    der = kernel.radial_derivatives(r0, p - 1)
    rhs = np.zeros(n)
    rhs[:p] = [der[i] * eps_b ** i for i in range(p)]
    rhs[p] = float(kernel.radial(0.5))
    return np.linalg.solve(A, rhs)


def regularized_radial(kernel, eps_b, p_deg):
    """Radial profile of the regularized kernel K_R (fastsum.py:119-132)."""
    if not 0.0 < eps_b < 0.5:
        raise ConfigError(f"eps_b must lie in (0, 1/2), got {eps_b}")
    r0 = 0.5 - eps_b
    coef = _bridge(kernel, eps_b, p_deg)

    def profile(r):
        r = np.asarray(r, dtype=float)
        tau = np.clip((r - r0) / eps_b, 0.0, 1.0)
        return np.where(r <= r0, kernel.radial(np.minimum(r, r0)),
                        np.polynomial.polynomial.polyval(tau, coef))

    return profile


def kernel_fourier_coefficients(kernel, d, N, eps_b, p_nfft):
    """bhat_l = N^-d sum_k K_R(k/N) e^{-2 pi i l.k/N}, FFT order (fastsum.py:135-151)."""
    if d not in (1, 2, 3):
        raise ConfigError(f"fastsum supports d in {{1, 2, 3}}, got d={d}")
    if N < 4 or N % 2:
        raise ConfigError(f"N must be even and >= 4, got {N}")
    profile = regularized_radial(kernel, eps_b, p_nfft)
    ax = np.fft.fftfreq(N)
    mesh = np.meshgrid(*([ax] * d), indexing="ij")
    rad = np.sqrt(sum(g * g for g in mesh))
    return np.fft.fftn(profile(rad)) / N ** d


def _kb_window_ld(t, m, b):
    """Kaiser-Bessel window in extended precision (fit input only)."""
    t = np.asarray(t, dtype=np.longdouble)
    m, b = np.longdouble(m), np.longdouble(b)
    z = m * m - t * t
    out = np.empty_like(t)
    pos, neg = z > 0, z < 0
    s = np.sqrt(z[pos])
    out[pos] = np.sinh(b * s) / s
    s = np.sqrt(-z[neg])
    out[neg] = np.sin(b * s) / s
    out[z == 0] = b
    return out / np.longdouble(math.pi)


def _kb_window(t, m, b):
    """The reference's float64 window (fastsum.py:158-167), for the fit check."""
    t = np.asarray(t, dtype=float)
    z = m * m - t * t
    inside = z > 0
    s_in = np.sqrt(np.where(inside, z, 1.0))
    s_out = np.sqrt(np.where(inside, 1.0, -z))
    with np.errstate(invalid="ignore"):
        v = np.where(inside, np.sinh(b * s_in) / s_in, np.sin(b * s_out) / s_out)
    return np.where(z == 0.0, b, v) / math.pi


def _kb_deconv(freqs, n_grid, m, b):
    w = 2.0 * math.pi * np.asarray(freqs, dtype=float) / n_grid
    arg = b * b - w * w
    if np.any(arg <= 0):
        raise NumericalError("frequency outside the Kaiser-Bessel passband")
    return 1.0 / np.i0(m * np.sqrt(arg))


def window_polynomials(m, b):
    """Monomial coefficients (in s = 2f-1) of phi(f - o), o = -m..m.

    Chebyshev interpolation of the entire function phi at deg+1 nodes from
    extended-precision samples, converted to the monomial basis; the fit is
    checked against the reference's float64 formula.
    """
    deg = 15 if m <= 3 else 13   # odd: as many even as odd terms (csrc/mlb_window.cuh WinDeg)
    nodes = np.cos(np.pi * (np.arange(deg + 1) + 0.5) / (deg + 1))
    coef = np.empty((2 * m + 1, deg + 1))
    f_chk = np.linspace(0.0, 1.0, 513)
    s_chk = 2 * f_chk - 1
    vmax = float(_kb_window(0.0, m, b))
    worst = 0.0
    for i, o in enumerate(range(-m, m + 1)):
        vals = _kb_window_ld((nodes + 1) / 2 - o, m, b).astype(float)
        cheb = np.polynomial.chebyshev.chebfit(nodes, vals, deg)
        coef[i] = np.polynomial.chebyshev.cheb2poly(cheb)
        approx = np.polynomial.polynomial.polyval(s_chk, coef[i])
        worst = max(worst, float(np.max(np.abs(approx - _kb_window(f_chk - o, m, b)))))
    if worst > 1e-13 * vmax:
        raise NumericalError(f"window polynomial fit error {worst / vmax:.2e} too large")
    return coef, deg


def _embed_axis(arr, axis, N, n_grid, split_nyquist):
    """FFT-order size-N axis into a size-n_grid axis (fastsum.py:219-253)."""
    half = N // 2
    a = np.moveaxis(arr, axis, 0)
    out = np.zeros((n_grid,) + a.shape[1:], dtype=arr.dtype)
    out[:half] = a[:half]
    out[n_grid - half + 1:] = a[half + 1:]
    if split_nyquist:
        out[n_grid - half] = 0.5 * a[half]
        out[half] = 0.5 * a[half]
    else:
        out[n_grid - half] = a[half]
    return np.moveaxis(out, 0, axis)


def _full_fused(coeffs, d, N, n_grid, m, b):
    """fused_weights of the reference (fastsum.py:282-294): b-hat (real part)
    embedded in ng^d with the Nyquist value halved onto +-N/2, times the
    squared KB deconvolution on |k| <= N/2 (0 outside) per axis, times ng^d;
    the rfftn half of the last axis."""
    full = coeffs.real
    for ax in range(d):
        full = _embed_axis(full, ax, N, n_grid, True)
    fq = np.fft.fftfreq(n_grid) * n_grid
    band = np.abs(fq) <= N // 2
    wfull = np.zeros(n_grid)
    wfull[band] = _kb_deconv(fq[band], n_grid, m, b) ** 2
    for ax in range(d):
        sh = [1] * d
        sh[ax] = n_grid
        full = full * wfull.reshape(sh)
    full = full * float(n_grid) ** d
    return np.ascontiguousarray(full[..., : n_grid // 2 + 1])


def _band_weights(coeffs, d, N, n_grid, m, b):
    """The same values as fused_weights on the band only: k = -N/2..N/2 on the
    first d-1 axes, k = 0..N/2 on the last, with the identical per-element
    operation order (Nyquist halving -- exact --, the axis-0, 1, 2 deconvolution
    factors in order, then ng^d): the device tables without the ng^d arrays."""
    h = N // 2
    kf = np.arange(-h, h + 1)
    kh = np.arange(0, h + 1)
    c = coeffs.real
    ks = [kf] * (d - 1) + [kh]
    vals = c[np.ix_(*[np.mod(k, N) for k in ks])]
    for ax, k in enumerate(ks):   # embed: the Nyquist entries carry 0.5 (power of two: exact in any order)
        sh = [1] * d
        sh[ax] = len(k)
        vals = vals * np.where(np.abs(k) == h, 0.5, 1.0).reshape(sh)
    w = _kb_deconv(np.arange(-h, h + 1).astype(float), n_grid, m, b) ** 2     # indexed by k + h
    for ax, k in enumerate(ks):
        sh = [1] * d
        sh[ax] = len(k)
        vals = vals * w[k + h].reshape(sh)
    return vals * float(n_grid) ** d


@dataclass
class FastsumPlan:
    """Plan for fast sums of one kernel in one dimension (fastsum.py:183-216).

    Host fields match the reference; `_device` caches the libmlb plans per
    (device, point-domain) pair.
    """

    kernel: KernelSpec
    d: int
    N: int
    m_nfft: int
    eps_b: float
    p_nfft: int
    rho: float
    n_grid: int
    ball_scale: float
    kernel_eff: KernelSpec
    window: str
    window_shape: float
    coeffs: np.ndarray
    deconv_axis: np.ndarray = field(repr=False)
    _fused: np.ndarray = field(default=None, repr=False, compare=False)
    K0: float = 1.0
    win_coef: np.ndarray = field(default=None, repr=False)
    win_deg: int = 13
    _device: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def fused_weights(self):
        """rfftn-layout fused weights (ng,)*(d-1) x (ng/2+1) (fastsum.py:282-294),
        built on first access: the device path only needs the |k| <= N/2
        band (_band_weights), so plan construction skips the ng^d arrays."""
        if self._fused is None:
            self._fused = _full_fused(self.coeffs, self.d, self.N, self.n_grid, self.m_nfft, self.window_shape)
        return self._fused

    def describe(self):
        return {"kernel": self.kernel.family, "sigma": self.kernel.sigma, "d": self.d, "N": self.N,
                "m_nfft": self.m_nfft, "eps_b": self.eps_b, "p_nfft": self.p_nfft, "rho": self.rho,
                "window": self.window, "ball_scale": self.ball_scale}

    # -- device plan --------------------------------------------------------
    def bin_range(self, domain="box"):
        """floor(ng * x * scale) range over admissible points of the domain."""
        ng = self.n_grid
        if domain == "torus":
            return -ng // 2, ng // 2 - 1
        xmax = box_halfwidth(self.eps_b) + BOX_TOL
        lo = math.floor(ng * ((-xmax) * self.ball_scale))
        hi = math.floor(ng * (xmax * self.ball_scale))
        return int(lo), int(hi)

    def device_tables(self, domain="box"):
        """fused band / twiddles / window coefficients as passed to mlb_plan_create."""
        d, N, m, ng = self.d, self.N, self.m_nfft, self.n_grid
        blo, bhi = self.bin_range(domain)
        L = bhi - blo + 1 + 2 * m
        ulo = blo - m
        kfull = np.arange(-N // 2, N // 2 + 1)
        khalf = np.arange(0, N // 2 + 1)
        idx = [np.mod(kfull, ng)] * (d - 1) + [khalf]
        Fb = _band_weights(self.coeffs, d, N, ng, m, self.window_shape)   # K^(d-1) x Kh, k_last >= 0
        band = Fb / float(ng) ** d
        u = np.arange(ulo, ulo + L)
        ph = np.mod(np.outer(u, kfull), ng).astype(float) * (2.0 * math.pi / ng)
        tw = np.empty((L, N + 1, 2))
        tw[..., 0] = np.cos(ph)
        tw[..., 1] = -np.sin(ph)
        # the full K^d band: negative last-axis frequencies by the reflection
        # F(k', -k_last) = F(-k', k_last) of fused_weights_full (F is even)
        Fneg = Fb[..., 1:][tuple([slice(None, None, -1)] * (d - 1) + [slice(None, None, -1)])]
        Ffull = np.concatenate([Fneg, Fb], axis=-1) / float(ng) ** d
        D = np.arange(-(L - 1), L)
        A = np.exp(2j * math.pi * np.outer(kfull, D) / ng)                       # K x (2L-1)
        conv = None
        if d <= 2:
            # spatial kernel Kc[D] = sum_k F(k) exp(2 pi i k.D/ng) over the full
            # band (F even -> real); D = -(L-1)..(L-1) per axis
            Kc = (Ffull @ A).real if d == 1 else (A.T @ Ffull @ A).real
            conv = np.ascontiguousarray(Kc)
        # Separable fast path: for a Gaussian whose regularised profile equals
        # exp(-|y|^2/s^2) to below double precision on the whole sampling cube
        # (true when K(1/2) / K(0) is negligible), F(k) = prod_a f(k_a) and the
        # convolution is d one-dimensional convolutions with
        # c[D] = sum_k f(k) cos(2 pi k D / ng).  Used only if the rank-1 tensor
        # reproduces F to 1e-13 of its maximum (i.e. to rounding); otherwise the
        # general stages run.
        sep = None
        center = (N // 2,) * d
        f0 = Ffull[center]
        if d >= 2 and f0 > 0:
            c0 = f0 ** (1.0 / d)
            line = [slice(None) if a == 0 else N // 2 for a in range(d)]
            f = Ffull[tuple(line)] / c0 ** (d - 1)
            Fsep = f
            for _ in range(1, d):
                Fsep = np.multiply.outer(Fsep, f)
            if np.max(np.abs(Ffull - Fsep)) <= 1e-13 * np.max(np.abs(Ffull)):
                sep = np.ascontiguousarray((f @ A).real)
        return dict(bin_lo=blo, bin_hi=bhi, L=L, ulo=ulo, fused_band=np.ascontiguousarray(band),
                    twiddle=np.ascontiguousarray(tw), conv_kernel=conv, sep_kernel=sep)

    def fused_weights_full(self):
        """The full (ng,)*d fused weights (the reference keeps the R2C half; the
        array is even, so the missing half is its reflection)."""
        ng, d = self.n_grid, self.d
        h = self.fused_weights
        full = np.empty((ng,) * d)
        full[..., : ng // 2 + 1] = h
        k = np.arange(ng // 2 + 1, ng)
        src = np.mod(-k, ng)
        refl = h
        for ax in range(d - 1):
            refl = np.take(refl, np.mod(-np.arange(ng), ng), axis=ax)
        full[..., ng // 2 + 1:] = refl[..., src]
        return full

    def device_plan(self, device=0, domain="box"):
        key = (int(device), domain)
        h = self._device.get(key)
        if h is not None:
            return h
        lib = _lib.lib()
        t = self.device_tables(domain)
        wc = np.ascontiguousarray(self.win_coef)
        conv, sep = t["conv_kernel"], t["sep_kernel"]
        desc = _lib.PlanDesc(self.d, self.N, self.m_nfft, self.n_grid, t["bin_lo"], t["bin_hi"],
                             self.win_deg, float(self.K0), t["fused_band"].ctypes.data,
                             t["twiddle"].ctypes.data, wc.ctypes.data,
                             None if conv is None else conv.ctypes.data,
                             None if sep is None else sep.ctypes.data)
        out = C.c_void_p()
        _lib.check(lib.mlb_plan_create(C.byref(desc), int(device), C.byref(out)))
        h = _PlanHandle(out, t)
        self._device[key] = h
        return h


class _PlanHandle:
    def __init__(self, ptr, tables):
        self.ptr = ptr
        self.L = tables["L"]
        self.ulo = tables["ulo"]
        self.bin_lo, self.bin_hi = tables["bin_lo"], tables["bin_hi"]

    def __del__(self):
        try:
            if self.ptr:
                _lib.load().mlb_plan_destroy(self.ptr)
        except Exception:
            pass


def build_plan(kernel, d, N=DEFAULT_N, m_nfft=DEFAULT_M, eps_b=DEFAULT_EPS_B, p_nfft=DEFAULT_P, rho=DEFAULT_RHO):
    """Build a fastsum plan (fastsum.py:256-313); host math, device tables lazily."""
    if d not in (1, 2, 3):
        raise ConfigError(f"fastsum supports d in {{1, 2, 3}}, got d={d}")
    if N < 4 or N % 2:
        raise ConfigError(f"N must be even and >= 4, got {N}")
    if m_nfft < 2:
        raise ConfigError(f"m_nfft must be >= 2, got {m_nfft}")
    n_grid = int(round(rho * N))
    if n_grid < N + 2 or n_grid % 2:
        raise ConfigError(f"oversampling rho={rho} gives invalid grid size {n_grid}")
    ball_scale = 1.0 / math.sqrt(d)
    kernel_eff = kernel.scaled(ball_scale)
    coeffs = kernel_fourier_coefficients(kernel_eff, d, N, eps_b, p_nfft)
    b = math.pi * (2.0 - N / n_grid)
    deconv_axis = _kb_deconv(np.fft.fftfreq(N) * N, n_grid, m_nfft, b)
    leak = np.max(np.abs(coeffs.imag)) if coeffs.size else 0.0
    if leak > 1e-12 * max(1.0, np.max(np.abs(coeffs.real))):
        raise NumericalError("kernel coefficients are not real; kernel not even?")
    win_coef, win_deg = (None, 13)
    if m_nfft <= 6:
        win_coef, win_deg = window_polynomials(m_nfft, b)
    return FastsumPlan(kernel=kernel, d=d, N=N, m_nfft=m_nfft, eps_b=eps_b, p_nfft=p_nfft, rho=rho,
                       n_grid=n_grid, ball_scale=ball_scale, kernel_eff=kernel_eff, window="kaiser-bessel",
                       window_shape=b, coeffs=coeffs, deconv_axis=deconv_axis,
                       K0=kernel.value_at_zero(), win_coef=win_coef, win_deg=win_deg)


# ---------------------------------------------------------------- binding --
class PointBinding:
    """Device binding of one point set (replaces PointBinding, fastsum.py:320-330).

    Holds the libmlb binding: cell-sorted permutation, fractional offsets,
    chunk/segment tables and scratch, built by mlb_bind_ex with every
    per-point step on the GPU.  `points`: an (n, >= d) float64 array (host)
    or CUDA tensor (device-resident points are bound in place); `columns`
    picks the d coordinate columns of a wider feature matrix; `box_map`
    (datapipe.BoxMap) maps raw feature columns into the box on the device
    (feature_group's scaling folded into the bind); `validate` runs
    validate_box (fastsum.py:66-80) on the device.  `node_ids` places the
    points inside a longer node vector (component blocks, graphs.py:99-129).
    """

    def __init__(self, plan, points, scale, domain="box", device=None, node_ids=None, box_map=None,
                 columns=None, validate=False):
        import torch
        self.plan = plan
        self.device = torch.cuda.current_device() if device is None else int(device)
        if isinstance(points, torch.Tensor):
            src = points.to(device=f"cuda:{self.device}", dtype=torch.float64).contiguous()
            on_dev, ptr = 1, src.data_ptr()
        else:
            src = np.ascontiguousarray(points, dtype=float)
            on_dev, ptr = 0, src.ctypes.data
        if src.ndim != 2:
            raise ConfigError(f"points must be a 2-d array, got shape {tuple(src.shape)}")
        self.n = int(src.shape[0])
        self.d = plan.d
        cols = None if columns is None else np.ascontiguousarray(columns, dtype=np.int32)
        if cols is None and src.shape[1] != plan.d:
            raise ConfigError(f"points have dimension {src.shape[1]}, plan expects {plan.d}")
        if cols is not None and cols.shape != (plan.d,):
            raise ConfigError(f"expected {plan.d} coordinate columns, got {len(cols)}")
        self.n_grid = plan.n_grid
        self.grid_size = plan.n_grid ** plan.d
        self._plan_handle = plan.device_plan(self.device, domain)
        ids = None if node_ids is None else np.ascontiguousarray(node_ids, dtype=np.int32)
        mid = None if box_map is None else np.ascontiguousarray(np.broadcast_to(box_map.mid, (plan.d,)), dtype=float)
        desc = _lib.BindDesc(
            points=ptr if self.n else None, points_on_device=on_dev, n=self.n, ld=int(src.shape[1]),
            cols=None if cols is None else cols.ctypes.data, scale=float(scale),
            box_mid=None if mid is None else mid.ctypes.data,
            box_half=0.0 if box_map is None else float(box_map.half),
            box_s=0.0 if box_map is None else float(box_map.s),
            box_hw=box_halfwidth(plan.eps_b) if validate else 0.0,
            node_ids=None if ids is None else ids.ctypes.data,
            stream=torch.cuda.current_stream(self.device).cuda_stream)
        if box_map is not None and box_map.half == 0.0:
            raise ConfigError("a constant column group maps to the origin; bind its zero points instead")
        out = C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib().mlb_bind_ex(self._plan_handle.ptr, C.byref(desc), C.byref(out)))
        self.ptr = out

    def stats(self):
        o = (C.c_int64 * 8)()
        _lib.check(_lib.load().mlb_binding_stats(self.ptr, o))
        lat = (C.c_int64 * 2)()
        _lib.check(_lib.load().mlb_binding_lattice(self.ptr, lat))
        return dict(zip(("n", "chunks", "segments", "bricks", "tile_cells", "grid_cells", "band_ctas",
                         "band_tile_cells", "lattice_items", "lattice_points"), list(o) + list(lat)))

    def sorted_perm(self):
        out = np.empty(self.n, dtype=np.int32)
        _lib.check(_lib.load().mlb_binding_perm(self.ptr, out.ctypes.data))
        return out

    def __del__(self):
        try:
            if getattr(self, "ptr", None):
                _lib.load().mlb_binding_destroy(self.ptr)
                self.ptr = None
        except Exception:
            pass


def bind_points(plan, points, sort=None, device=None, node_ids=None):
    """Validate the box and bind the points on the device (fastsum.py:375-386).

    `sort` is accepted for compatibility: the device binding always orders
    points by cell.
    """
    import torch
    if not isinstance(points, torch.Tensor):
        points = np.asarray(points, dtype=float)
    if points.ndim != 2:
        raise ConfigError(f"points must be a 2-d array, got shape {tuple(points.shape)}")
    if points.shape[1] != plan.d:
        raise ConfigError(f"points have dimension {points.shape[1]}, plan expects {plan.d}")
    # validate_box (non-finite values, |x|_inf <= 1/4 - eps_b/2) runs on the device inside the bind
    return PointBinding(plan, points, plan.ball_scale, "box", device, node_ids, validate=True)


# ------------------------------------------------------------------ apply --
def _as_device(v, device):
    """(tensor fp64 on device, was_numpy)."""
    import torch
    if isinstance(v, torch.Tensor):
        return v.to(device=f"cuda:{device}", dtype=torch.float64).contiguous(), False
    arr = np.ascontiguousarray(np.asarray(v, dtype=float))
    return torch.from_numpy(arr).to(f"cuda:{device}"), True


def apply_binding(binding, v_dev, y_dev, alpha, beta, gamma, flags, stream=None):
    """Raw mlb_apply on device tensors."""
    _lib.check(_lib.lib().mlb_apply(binding.ptr, _lib.ptr(v_dev), _lib.ptr(y_dev), float(alpha), float(beta),
                                    float(gamma), int(flags), _lib.stream_ptr(stream)))


def fastsum_apply(points, v, plan, binding=None):
    """W v with W_ij = K(x_i - x_j), W_ii = 0 (fastsum.py:475-497), on the GPU."""
    import torch
    if binding is None:
        binding = bind_points(plan, points)
    if isinstance(v, torch.Tensor):
        vd, host = _as_device(v, binding.device)
    else:
        v = np.asarray(v, dtype=float)
        if v.shape != (binding.n,):
            raise ConfigError("v must be a real vector matching the number of points")
        vd, host = _as_device(v, binding.device)
    if tuple(vd.shape) != (binding.n,):
        raise ConfigError("v must be a real vector matching the number of points")
    if binding.n == 0:
        return np.zeros(0) if host else vd.clone()
    y = torch.empty_like(vd)
    apply_binding(binding, vd, y, -plan.K0, 1.0, 0.0, 0)
    return y.cpu().numpy() if host else y


def direct_apply(points, v, kernel, block_rows=None):
    """Exact W v (zero diagonal) on the GPU (fastsum.py:500-553); the O(n^2) oracle path."""
    from .direct import direct_apply as _d
    return _d(points, v, kernel, block_rows)


def nfft_adjoint(points, v, plan):
    from .nfft import nfft_adjoint as _a
    return _a(points, v, plan)


def nfft_forward(coeffs, points, plan):
    from .nfft import nfft_forward as _f
    return _f(coeffs, points, plan)
