"""Bare nonequispaced transforms on the torus (fastsum.py:418-468) on the GPU.

nfft_adjoint:  ghat_l = sum_j v_j exp(-2 pi i l.x_j),  l in I_N (FFT order)
nfft_forward:  f_i    = sum_l c_l exp(+2 pi i l.x_i)

Same pipeline as the reference: window spread on the oversampled torus grid
(real and imaginary parts separately), band DFT (mlb_band_dft), truncation to
I_N and the Kaiser-Bessel deconvolution -- and the reverse for the forward
transform.  The points are bound in "torus" mode (no box margin, no 1/sqrt(d)).
"""

import numpy as np

from . import _lib
from .errors import ConfigError
from .fastsum import PointBinding


def _torch():
    import torch
    return torch


def _check_torus(points, d):
    points = np.asarray(points, dtype=float)
    if points.ndim != 2 or points.shape[1] != d:
        raise ConfigError(f"points must have shape (n, {d})")
    if points.shape[0] and np.max(np.abs(points)) >= 0.5:
        raise ConfigError("nfft points must lie in [-1/2, 1/2)")
    return points


def _band_index(N):
    """positions of I_N (FFT order 0..N/2-1, -N/2..-1) inside the band -N/2..N/2."""
    k = np.fft.fftfreq(N) * N
    return (k + N // 2).astype(np.int64)


def _deconv_nd(plan, torch, device):
    dc = torch.from_numpy(plan.deconv_axis).to(device)
    out = dc
    for _ in range(1, plan.d):
        out = out[..., None] * dc
    return out


def nfft_adjoint(points, v, plan):
    torch = _torch()
    pts = _check_torus(points, plan.d)
    v = np.asarray(v)
    if v.shape != (pts.shape[0],):
        raise ConfigError("v must be a vector matching the number of points")
    b = PointBinding(plan, pts, 1.0, "torus")
    lib = _lib.lib()
    dev = f"cuda:{b.device}"
    L, d, N = b._plan_handle.L, plan.d, plan.N
    K = N + 1
    grids = []
    for part in (np.real(v), np.imag(v) if np.iscomplexobj(v) else None):
        g = torch.zeros(L ** d, dtype=torch.float64, device=dev)
        if part is not None and b.n:
            x = torch.from_numpy(np.ascontiguousarray(part, dtype=float)).to(dev)
            _lib.check(lib.mlb_spread(b.ptr, _lib.ptr(x), _lib.ptr(g), 0, _lib.stream_ptr()))
        grids.append(g)
    cgrid = torch.complex(grids[0], grids[1]).contiguous()
    spec = torch.empty(K ** d, dtype=torch.complex128, device=dev)
    _lib.check(lib.mlb_band_dft(b.ptr, _lib.ptr(cgrid), _lib.ptr(spec), 0, _lib.stream_ptr()))
    spec = spec.reshape((K,) * d)
    idx = torch.from_numpy(_band_index(N)).to(dev)
    for ax in range(d):
        spec = spec.index_select(ax, idx)
    spec = spec * _deconv_nd(plan, torch, dev)
    return spec.cpu().numpy()


def nfft_forward(coeffs, points, plan):
    torch = _torch()
    pts = _check_torus(points, plan.d)
    c = np.asarray(coeffs, dtype=complex)
    if c.shape != (plan.N,) * plan.d:
        raise ConfigError(f"coeffs must have shape {(plan.N,) * plan.d}")
    b = PointBinding(plan, pts, 1.0, "torus")
    lib = _lib.lib()
    dev = f"cuda:{b.device}"
    L, d, N = b._plan_handle.L, plan.d, plan.N
    K = N + 1
    ct = torch.from_numpy(c).to(dev) * _deconv_nd(plan, torch, dev)
    # embed I_N into the band without Nyquist splitting (the -N/2 slot)
    band = torch.zeros((K,) * d, dtype=torch.complex128, device=dev)
    sl = tuple(torch.from_numpy(_band_index(N)).to(dev) for _ in range(d))
    band[torch.meshgrid(*sl, indexing="ij")] = ct
    grid = torch.empty(L ** d, dtype=torch.complex128, device=dev)
    _lib.check(lib.mlb_band_dft(b.ptr, _lib.ptr(band.contiguous()), _lib.ptr(grid), 1, _lib.stream_ptr()))
    out = []
    for part in (grid.real.contiguous(), grid.imag.contiguous()):
        y = torch.empty(b.n, dtype=torch.float64, device=dev)
        if b.n:
            _lib.check(lib.mlb_gather(b.ptr, _lib.ptr(part), _lib.ptr(y), 0, _lib.stream_ptr()))
        out.append(y.cpu().numpy())
    return out[0] + 1j * out[1]
