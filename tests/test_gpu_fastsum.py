"""GPU parity of the NFFT matvec path against the reference golden vectors and
the numpy oracle (same seeded inputs).  Tolerance (BASELINE north star):
matvecs within 1e-8 relative; in practice the device path agrees to ~1e-13.
"""

import math

import numpy as np
import pytest
from numpy.testing import assert_allclose

from conftest import load_golden
from oracle import fastsum_oracle as fo

pytestmark = pytest.mark.gpu

CASES = ["d1_n400", "d1_n300_m4", "d2_n500", "d2_n500_m3", "d2_n400_lap", "d2_n300_N64m5",
         "d3_n300", "d3_n250_m6", "d3_n300_N32", "d3_n200_N64m5"]
FAM = {0: "gaussian", 1: "laplacian"}
RTOL = 1e-8  # north-star matvec tolerance; observed ~1e-13


def _plan(spec):
    from paper_2007_05239_b200 import KernelSpec, build_plan
    fam, s, d, N, m, p = spec
    return build_plan(KernelSpec(FAM[int(fam)], float(s)), d=int(d), N=int(N), m_nfft=int(m), p_nfft=int(p))


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("name", CASES)
def test_fastsum_matches_reference_golden(name):
    from paper_2007_05239_b200 import bind_points, fastsum_apply
    g = load_golden("fastsum")
    plan = _plan(g[name + "/spec"])
    pts, v = g[name + "/points"], g[name + "/v"]
    b = bind_points(plan, pts)
    got = fastsum_apply(None, v, plan, binding=b)
    assert rel(got, g[name + "/Wv"]) < 1e-12, rel(got, g[name + "/Wv"])
    ones = fastsum_apply(None, np.ones(len(v)), plan, binding=b)
    assert rel(ones, g[name + "/ones"]) < 1e-12
    # bitwise-identical repeated applies (test_fastsum.py:241-252)
    again = fastsum_apply(None, v, plan, binding=b)
    assert np.array_equal(got, again)
    assert np.array_equal(got, fastsum_apply(pts, v, plan))


def test_two_point_hand_sum():
    from paper_2007_05239_b200 import KernelSpec, build_plan, fastsum_apply
    g = load_golden("fastsum")
    plan = build_plan(KernelSpec("gaussian", 0.1), d=2)
    got = fastsum_apply(g["two_point/points"], g["two_point/v"], plan)
    assert_allclose(got, g["two_point/Wv"], rtol=1e-12)
    assert_allclose(got, math.exp(-4.0) * np.array([2.0, 1.0]), rtol=1e-6)


@pytest.mark.parametrize("d,N,m,sigma", [(1, 32, 4, 0.15), (2, 32, 4, 0.15), (2, 64, 5, 0.15), (3, 16, 4, 0.15),
                                         (3, 32, 5, 0.15), (2, 16, 6, 0.15), (3, 16, 6, 0.15), (3, 64, 4, 0.15),
                                         (2, 32, 4, 0.05), (3, 32, 4, 0.05), (3, 64, 4, 0.08), (3, 16, 6, 0.05)])
def test_stages_match_oracle(d, N, m, sigma):
    """spread grid, convolved grid and gather, each against the oracle
    (sigma <= 0.1 exercises the separable convolution path)."""
    import torch
    from paper_2007_05239_b200 import KernelSpec, bind_points, build_plan
    from paper_2007_05239_b200 import _lib
    rng = np.random.default_rng(100 + 10 * d + m)
    n = 700
    hw = 0.25 - 0.5 / 16
    pts = rng.uniform(-hw, hw, size=(n, d))
    v = rng.standard_normal(n)
    plan = build_plan(KernelSpec("gaussian", sigma), d=d, N=N, m_nfft=m, p_nfft=8)
    b = bind_points(plan, pts)
    L, ulo = b._plan_handle.L, b._plan_handle.ulo
    lib = _lib.lib()
    vd = torch.from_numpy(v).cuda()
    grid = torch.zeros(L ** d, dtype=torch.float64, device="cuda")
    _lib.check(lib.mlb_spread(b.ptr, _lib.ptr(vd), _lib.ptr(grid), 0, _lib.stream_ptr()))
    # oracle spread on the full ng^d torus, folded onto the sub-box indices
    op = fo.OraclePlan("gaussian", sigma, d, N, m, p=8)
    ob = fo.bind(op, pts)
    full = fo.spread(ob, v).reshape((op.ng,) * d)
    idx = np.mod(np.arange(ulo, ulo + L), op.ng)
    sub = full[np.ix_(*([idx] * d))]
    assert rel(grid.cpu().numpy().reshape((L,) * d), sub) < 1e-13
    if d == 2:  # the grouped-lane spread (large layers) on the same points
        import os
        os.environ["MLB_D2_GROUPED"] = "1"
        try:
            g2 = torch.zeros_like(grid)
            _lib.check(lib.mlb_spread(b.ptr, _lib.ptr(vd), _lib.ptr(g2), 0, _lib.stream_ptr()))
        finally:
            del os.environ["MLB_D2_GROUPED"]
        assert rel(g2.cpu().numpy().reshape((L,) * d), sub) < 1e-13
    # convolution
    out = torch.zeros_like(grid)
    _lib.check(lib.mlb_convolve(b.ptr, _lib.ptr(grid), _lib.ptr(out), _lib.stream_ptr()))
    conv_full = fo.convolve_grid(op, full.ravel()).reshape((op.ng,) * d)
    assert rel(out.cpu().numpy().reshape((L,) * d), conv_full[np.ix_(*([idx] * d))]) < 1e-12
    # gather of the oracle's convolved grid
    y = torch.zeros(n, dtype=torch.float64, device="cuda")
    src = torch.from_numpy(np.ascontiguousarray(conv_full[np.ix_(*([idx] * d))]).ravel()).cuda()
    _lib.check(lib.mlb_gather(b.ptr, _lib.ptr(src), _lib.ptr(y), 0, _lib.stream_ptr()))
    assert rel(y.cpu().numpy(), fo.gather(ob, conv_full.ravel())) < 1e-13


@pytest.mark.parametrize("grouped", ["1", "0"])
@pytest.mark.parametrize("layout", ["square", "blobs"])
def test_banded_d2_spread_matches_oracle(grouped, layout):
    """The banded d = 2 spread (CTAs over contiguous cell ranges, band tiles,
    band_sum_kernel; default for n >= 2^20) forced on a 60k-point layer:
    spread grid vs the oracle, the whole fastsum vs the full-tile path, and
    repeated spreads bitwise identical."""
    import os

    import torch
    from paper_2007_05239_b200 import KernelSpec, bind_points, build_plan
    from paper_2007_05239_b200 import _lib
    from paper_2007_05239_b200.fastsum import fastsum_apply
    rng = np.random.default_rng(77)
    n = 60_000
    if layout == "square":   # image coordinates: every cell evenly filled
        pts = rng.uniform(-0.17, 0.17, size=(n, 2))
    else:                    # clustered: bands of very different widths
        c = rng.uniform(-0.15, 0.15, size=(6, 2))
        pts = np.clip(c[rng.integers(0, 6, n)] + 0.02 * rng.standard_normal((n, 2)), -0.2, 0.2)
    v = rng.standard_normal(n)
    plan = build_plan(KernelSpec("gaussian", 0.1), d=2, N=64, m_nfft=5, p_nfft=8)
    os.environ["MLB_D2_GROUPED"] = grouped
    os.environ["MLB_D2_BANDED"] = "1"
    try:
        b = bind_points(plan, pts)
        assert b.stats()["band_ctas"] > 0
        L, ulo = b._plan_handle.L, b._plan_handle.ulo
        lib = _lib.lib()
        vd = torch.from_numpy(v).cuda()
        grids = []
        for _ in range(2):
            g = torch.zeros(L * L, dtype=torch.float64, device="cuda")
            _lib.check(lib.mlb_spread(b.ptr, _lib.ptr(vd), _lib.ptr(g), 0, _lib.stream_ptr()))
            grids.append(g.cpu().numpy())
        y_band = fastsum_apply(pts, v, plan, binding=b)
        os.environ["MLB_D2_BANDED"] = "0"
        b0 = bind_points(plan, pts)
        assert b0.stats()["band_ctas"] == 0
        y_full = fastsum_apply(pts, v, plan, binding=b0)
    finally:
        del os.environ["MLB_D2_GROUPED"], os.environ["MLB_D2_BANDED"]
    assert np.array_equal(grids[0], grids[1])
    op = fo.OraclePlan("gaussian", 0.1, 2, 64, 5, p=8)
    full = fo.spread(fo.bind(op, pts), v).reshape(op.ng, op.ng)
    idx = np.mod(np.arange(ulo, ulo + L), op.ng)
    assert rel(grids[0].reshape(L, L), full[np.ix_(idx, idx)]) < 1e-13
    assert rel(y_band, y_full) < 1e-14


@pytest.mark.parametrize("layout,N", [("uniform", 64), ("clustered", 64), ("uniform", 2048), ("uniform", 4096)])
def test_streaming_d1_kernels_match_oracle(layout, N):
    """The streaming d = 1 spread / gather (contiguous warp ranges, per-cell
    start table; used from 2^16 points): spread grid and gather against the
    oracle, the fused Laplacian in node and cell order and with accumulation
    against the sub-chunk kernels (MLB_D1_STREAM=0), repeated spreads bitwise.
    N = 2048: the grid tables near the shared-memory budget; N = 4096: over
    it, so the sub-chunk kernels run (same assertions)."""
    import os

    import torch
    from paper_2007_05239_b200 import KernelSpec, bind_points, build_plan
    from paper_2007_05239_b200 import _lib
    rng = np.random.default_rng(91)
    n = 150_001
    if layout == "uniform":
        pts = rng.uniform(-0.2, 0.2, size=(n, 1))
    else:   # empty cells, light cells and heavy ones
        c = np.array([-0.15, -0.02, 0.0, 0.11])
        pts = np.clip(c[rng.integers(0, 4, n)] + 0.004 * rng.standard_normal(n), -0.2, 0.2)[:, None]
        pts[:40, 0] = np.linspace(-0.2, 0.2, 40)
    v = rng.standard_normal(n)
    plan = build_plan(KernelSpec("gaussian", 0.1), d=1, N=N, m_nfft=4, p_nfft=8)
    b = bind_points(plan, pts)
    L, ulo = b._plan_handle.L, b._plan_handle.ulo
    lib = _lib.lib()
    sp = _lib.stream_ptr()
    vd = torch.from_numpy(v).cuda()
    g1, g2 = (torch.zeros(L, dtype=torch.float64, device="cuda") for _ in range(2))
    _lib.check(lib.mlb_spread(b.ptr, _lib.ptr(vd), _lib.ptr(g1), 0, sp))
    _lib.check(lib.mlb_spread(b.ptr, _lib.ptr(vd), _lib.ptr(g2), 0, sp))
    assert torch.equal(g1, g2)
    op = fo.OraclePlan("gaussian", 0.1, 1, N, 4, p=8)
    ob = fo.bind(op, pts)
    full = fo.spread(ob, v)
    idx = np.mod(np.arange(ulo, ulo + L), op.ng)
    assert rel(g1.cpu().numpy(), full[idx]) < 1e-13
    conv = fo.convolve_grid(op, full)
    y = torch.zeros(n, dtype=torch.float64, device="cuda")
    src = torch.from_numpy(np.ascontiguousarray(conv[idx])).cuda()
    _lib.check(lib.mlb_gather(b.ptr, _lib.ptr(src), _lib.ptr(y), 0, sp))
    assert rel(y.cpu().numpy(), fo.gather(ob, conv)) < 1e-13
    # the fused Laplacian (node order, cell order, accumulate) vs the sub-chunk kernels
    isd = torch.from_numpy(rng.uniform(0.5, 2.0, n)).cuda()
    os.environ["MLB_D1_STREAM"] = "0"
    try:
        b0 = bind_points(plan, pts)
    finally:
        del os.environ["MLB_D1_STREAM"]
    outs = []
    for bb in (b, b0):
        _lib.check(lib.mlb_binding_set_isd(bb.ptr, _lib.ptr(isd), sp))
        r = []
        for flags in (_lib.MLB_USE_ISD, _lib.MLB_USE_ISD | _lib.MLB_ACCUMULATE):
            yy = torch.ones(n, dtype=torch.float64, device="cuda")
            _lib.check(lib.mlb_apply(bb.ptr, _lib.ptr(vd), _lib.ptr(yy), 1.7, -1.0, 1.0, flags, sp))
            r.append(yy.cpu().numpy())
        vs = torch.empty_like(vd)
        _lib.check(lib.mlb_to_sorted(bb.ptr, _lib.ptr(vd), _lib.ptr(vs), sp))
        ys = torch.empty_like(vd)
        _lib.check(lib.mlb_apply(bb.ptr, _lib.ptr(vs), _lib.ptr(ys), 1.7, -1.0, 1.0,
                                 _lib.MLB_USE_ISD | _lib.MLB_SORTED, sp))
        yn = torch.empty_like(vd)
        _lib.check(lib.mlb_to_node(bb.ptr, _lib.ptr(ys), _lib.ptr(yn), 0, sp))
        r.append(yn.cpu().numpy())
        outs.append(r)
    for a_, b_ in zip(*outs):
        assert rel(a_, b_) < 1e-14


def test_laplacian_matches_reference_golden():
    from paper_2007_05239_b200 import KernelSpec, build_plan
    from paper_2007_05239_b200.graphs import KernelWeights, apply_sym_laplacian, build_layer, with_shift
    g = load_golden("solvers")
    layers = []
    for key in ("3", "2"):
        plan = _plan(g["spec" + key])
        fam, s = FAM[int(g["spec" + key][0])], float(g["spec" + key][1])
        layers.append(build_layer(KernelWeights(g["pts" + key], KernelSpec(fam, s), plan=plan)))
    L3, L2 = layers
    assert rel(L3.degrees, g["deg3"]) < 1e-13
    assert rel(L2.degrees, g["deg2"]) < 1e-13
    v = g["v"]
    assert rel(apply_sym_laplacian(with_shift(L3, math.log(2.0)), v), g["Lv3_shift"]) < 1e-12
    assert rel(apply_sym_laplacian(L2, v), g["Lv2_noshift"]) < 1e-12
    # D^1/2 1 is (numerically) in the kernel of the unshifted operator
    r = apply_sym_laplacian(L2, np.sqrt(L2.degrees))
    assert np.linalg.norm(r) < 1e-10 * np.linalg.norm(np.sqrt(L2.degrees))


def test_laplacian_batch_matches_per_layer():
    """LaplacianBatch / apply_sym_laplacians (streams + CUDA graphs, host and
    device inputs, persistent host buffers) == the per-layer operator, bitwise."""
    import torch
    from paper_2007_05239_b200 import KernelSpec, LaplacianBatch, MultilayerGraph, apply_sym_laplacians
    from paper_2007_05239_b200.graphs import KernelWeights, apply_sym_laplacian, build_layer, with_shift
    g = load_golden("solvers")
    layers = []
    for key in ("3", "2"):
        plan = _plan(g["spec" + key])
        fam, s = FAM[int(g["spec" + key][0])], float(g["spec" + key][1])
        layers.append(with_shift(build_layer(KernelWeights(g["pts" + key], KernelSpec(fam, s), plan=plan)), 0.3))
    G = MultilayerGraph(tuple(layers))
    v = g["v"]
    ref = np.stack([apply_sym_laplacian(layer, v) for layer in layers])
    assert np.array_equal(apply_sym_laplacians(G, v), ref)
    assert np.array_equal(apply_sym_laplacians(G, v, use_graph=False), ref)
    batch = LaplacianBatch(G)
    vp = torch.from_numpy(v).pin_memory()
    out = torch.empty((G.T, G.n), dtype=torch.float64, pin_memory=True)
    for _ in range(4):  # first calls per-layer graphs, then the whole-step graph
        out.zero_()
        batch.apply(vp, out=out)
        assert np.array_equal(out.numpy(), ref)
    assert np.array_equal(batch.apply(torch.from_numpy(v).cuda()).cpu().numpy(), ref)
    w = np.random.default_rng(5).standard_normal(G.n)
    ref_w = np.stack([apply_sym_laplacian(layer, w) for layer in layers])
    vp.copy_(torch.from_numpy(w))  # same host buffers, new contents: the graph re-reads them
    assert np.array_equal(batch.apply(vp, out=out).numpy(), ref_w)
    # streamed multi-vector apply (double-buffered, copies overlapped): bitwise the same
    rng = np.random.default_rng(9)
    V = rng.standard_normal((7, G.n))
    refs = np.stack([np.stack([apply_sym_laplacian(layer, x) for layer in layers]) for x in V])
    for use_graph in (True, False):
        b2 = LaplacianBatch(G, use_graph=use_graph)
        assert np.array_equal(b2.apply_many(V).numpy(), refs)
        Vp = torch.from_numpy(V).pin_memory()
        outp = torch.empty((7, G.T, G.n), dtype=torch.float64, pin_memory=True)
        assert np.array_equal(b2.apply_many(Vp, out=outp).numpy(), refs)
        assert np.array_equal(b2.apply_many(Vp[:1].clone().pin_memory()).numpy(), refs[:1])


def test_apply_batched_c_abi_is_bitwise_per_layer():
    """mlb_apply_batched (layers on library streams, C hosts) == mlb_apply per layer."""
    import ctypes
    import torch
    from paper_2007_05239_b200 import KernelSpec, _lib
    from paper_2007_05239_b200.graphs import KernelWeights, build_layer, with_shift
    g = load_golden("solvers")
    layers = []
    for key in ("3", "2"):
        plan = _plan(g["spec" + key])
        fam, s = FAM[int(g["spec" + key][0])], float(g["spec" + key][1])
        layers.append(with_shift(build_layer(KernelWeights(g["pts" + key], KernelSpec(fam, s), plan=plan)), 0.4))
    lib = _lib.lib()
    v = torch.from_numpy(g["v"]).cuda()
    bs = [lay.weights._bindings[0] for lay in layers]
    for lay in layers:
        lay.weights.set_isd(lay.isd_device(lay.weights.device))
    coeff = [(1.0 + lay.shift, -1.0, lay.weights.kernel.value_at_zero()) for lay in layers]
    ref = []
    for b, (a, bt, gm) in zip(bs, coeff):
        y = torch.empty_like(v)
        _lib.check(lib.mlb_apply(b.ptr, _lib.ptr(v), _lib.ptr(y), a, bt, gm, _lib.MLB_USE_ISD, _lib.stream_ptr()))
        ref.append(y)
    ys = [torch.full_like(v, float("nan")) for _ in layers]
    T = len(layers)
    arr = lambda ctype, vals: (ctype * T)(*vals)  # noqa: E731
    _lib.check(lib.mlb_apply_batched(arr(ctypes.c_void_p, [b.ptr.value for b in bs]), T, _lib.ptr(v),
                                     arr(ctypes.c_void_p, [y.data_ptr() for y in ys]),
                                     arr(ctypes.c_double, [c[0] for c in coeff]),
                                     arr(ctypes.c_double, [c[1] for c in coeff]),
                                     arr(ctypes.c_double, [c[2] for c in coeff]), _lib.MLB_USE_ISD,
                                     _lib.stream_ptr()))
    torch.cuda.synchronize()
    for y, r in zip(ys, ref):
        assert torch.equal(y, r)


def test_per_component_blocks_match_oracle():
    from paper_2007_05239_b200 import KernelSpec, build_plan
    from paper_2007_05239_b200.graphs import KernelWeights
    rng = np.random.default_rng(7)
    pts = rng.uniform(-0.2, 0.2, size=(600, 2))
    comp = rng.integers(0, 3, 600)
    plan = build_plan(KernelSpec("gaussian", 0.1), d=2, N=32, m_nfft=4, p_nfft=8)
    w = KernelWeights(pts, KernelSpec("gaussian", 0.1), plan=plan, components=comp)
    v = rng.standard_normal(600)
    got = w.matvec(v)
    op = fo.OraclePlan("gaussian", 0.1, 2, 32, 4, p=8)
    ref = np.zeros(600)
    for c in range(3):
        idx = np.flatnonzero(comp == c)
        ref[idx] = fo.fastsum(op, v[idx], points=pts[idx])
    assert rel(got, ref) < 1e-12


def test_empty_and_errors():
    from paper_2007_05239_b200 import ConfigError, KernelSpec, build_plan, fastsum_apply
    plan = build_plan(KernelSpec("gaussian", 0.3), d=2)
    assert fastsum_apply(np.zeros((0, 2)), np.zeros(0), plan).shape == (0,)
    with pytest.raises(ConfigError):
        fastsum_apply(np.zeros((3, 2)), np.zeros(4), plan)
    with pytest.raises(ConfigError):
        fastsum_apply(np.array([[0.3, 0.0]]), np.ones(1), plan)


def test_large_property_checks():
    """n = 2e5, d = 3: linearity and symmetry <u, Wv> = <Wu, v> at full size."""
    from paper_2007_05239_b200 import KernelSpec, bind_points, build_plan, fastsum_apply
    rng = np.random.default_rng(9)
    n = 200_000
    g = rng.standard_normal((n, 3))
    g /= np.linalg.norm(g, axis=1, keepdims=True)
    pts = g * (0.21875 * rng.random(n) ** (1 / 3))[:, None]
    plan = build_plan(KernelSpec("gaussian", 0.05), d=3, N=32, m_nfft=4, p_nfft=8)
    b = bind_points(plan, pts)
    u, v = rng.standard_normal(n), rng.standard_normal(n)
    Wu = fastsum_apply(None, u, plan, binding=b)
    Wv = fastsum_apply(None, v, plan, binding=b)
    Wuv = fastsum_apply(None, 2.0 * u - 3.0 * v, plan, binding=b)
    assert rel(Wuv, 2.0 * Wu - 3.0 * Wv) < 1e-12
    assert abs(u @ Wv - Wu @ v) < 1e-11 * np.linalg.norm(Wu) * np.linalg.norm(v)
    # chunked oracle on a subsample of targets is too slow at 2e5; compare
    # against the oracle on the first 20k points as their own point set
    sub = pts[:20000]
    b2 = bind_points(plan, sub)
    op = fo.OraclePlan("gaussian", 0.05, 3, 32, 4, p=8)
    ref = fo.fastsum(op, u[:20000], points=sub)
    assert rel(fastsum_apply(None, u[:20000], plan, binding=b2), ref) < 1e-12


@pytest.mark.parametrize("d", [1, 2])
def test_bare_nfft_matches_reference_golden(d):
    """nfft_adjoint / nfft_forward (fastsum.py:418-468) vs reference outputs,
    plus exact adjointness <forward(c), v> = <c, conj(adjoint(v))>."""
    from paper_2007_05239_b200 import KernelSpec, build_plan
    from paper_2007_05239_b200.fastsum import nfft_adjoint, nfft_forward
    g = load_golden("nfft")
    plan = build_plan(KernelSpec("gaussian", 0.2), d=d, N=16)
    pts, v, c = g[f"d{d}/points"], g[f"d{d}/v"], g[f"d{d}/coeffs"]
    adj = nfft_adjoint(pts, v, plan)
    ref = g[f"d{d}/adjoint"]
    assert np.abs(adj - ref).max() <= 1e-12 * np.abs(ref).max()
    fwd = nfft_forward(c, pts, plan)
    ref = g[f"d{d}/forward"]
    assert np.abs(fwd - ref).max() <= 1e-12 * np.abs(ref).max()
    lhs = np.sum(fwd * v)
    rhs = np.sum(c * np.conj(adj))
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)


def test_sharded_layer_single_rank_matches_layer():
    """dist.ShardedLayer + BindingEngine (NCCL, world size 1) == the fused layer."""
    import os
    import torch
    import torch.distributed as dist
    from paper_2007_05239_b200 import KernelSpec, KernelWeights, build_layer, build_plan, with_shift
    from paper_2007_05239_b200.dist import BindingEngine, Comm, ShardedLayer, sharded_pksm
    from paper_2007_05239_b200.graphs import apply_sym_laplacian
    from paper_2007_05239_b200.krylov import pksm_apply
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        rng = np.random.default_rng(5)
        n = 3000
        pts = np.clip(rng.normal(0, 0.07, size=(n, 3)), -0.21875, 0.21875)
        kern = KernelSpec("gaussian", 0.12)
        plan = build_plan(kern, d=3, N=32, m_nfft=4, p_nfft=8)
        layer = with_shift(build_layer(KernelWeights(pts, kern, plan=plan)), math.log(2.0))
        v = rng.standard_normal(n)
        sl = ShardedLayer(BindingEngine(plan, pts), n, 0, n, Comm(), K0=1.0, shift=math.log(2.0)).build()
        vd = torch.from_numpy(v).cuda()
        assert rel(sl.apply_lsym(vd).cpu().numpy(), apply_sym_laplacian(layer, v)) < 1e-12
        assert rel(sharded_pksm(sl, -1.0, vd).cpu().numpy(), pksm_apply(layer, -1.0, v)) < 1e-9
        # the fused peer exchange (IPC handle of its own buffer, NCCL flag, slot sum)
        sp = ShardedLayer(BindingEngine(plan, pts).enable_peer_exchange(Comm()), n, 0, n, Comm(), K0=1.0,
                          shift=math.log(2.0)).build()
        assert np.array_equal(sp.apply_lsym(vd).cpu().numpy(), sl.apply_lsym(vd).cpu().numpy())
    finally:
        dist.destroy_process_group()


def test_peer_grid_exchange_two_emulated_ranks():
    """mlb_spread_peers + mlb_grid_sum_slots with two ranks emulated on one
    GPU (their receive buffers are local; the launches run one after the
    other, nothing waits on another kernel): every rank's buffer ends with the
    same grid, bitwise, equal to the one-binding spread."""
    import torch
    from paper_2007_05239_b200 import KernelSpec, build_plan, bind_points, _lib
    from paper_2007_05239_b200.dist import PeerGridExchange
    import os
    rng = np.random.default_rng(8)
    n = 4000
    for d, N, m, lattice in ((3, 32, 4, False), (2, 32, 4, False), (2, 64, 5, True)):
        if lattice:   # an image's pixels, ranks cutting its rows: lattice items + shard-cut segments
            pts = _lattice_points(80, 50)
            os.environ["MLB_LATTICE"] = "1"
        else:
            pts = np.clip(rng.normal(0, 0.07, size=(n, d)), -0.21875, 0.21875)
        n = len(pts)
        v = rng.standard_normal(n)
        plan = build_plan(KernelSpec("gaussian", 0.12), d=d, N=N, m_nfft=m, p_nfft=8)
        full = bind_points(plan, pts)
        assert (full.stats()["lattice_items"] > 0) == lattice
        cells = full.stats()["grid_cells"]
        ref = torch.zeros(cells, dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().mlb_spread(full.ptr, _lib.ptr(torch.from_numpy(v).cuda()), _lib.ptr(ref), 0,
                                         _lib.stream_ptr()))
        halves = [(0, n // 2 + 17), (n // 2 + 17, n)]
        recv = [torch.full((2 * cells,), float("nan"), dtype=torch.float64, device="cuda") for _ in range(2)]
        grids = []
        for r, (lo, hi) in enumerate(halves):
            b = bind_points(plan, pts[lo:hi])
            ex = PeerGridExchange(None, cells, 0, recv=recv[r],
                                  slots=[recv[q].data_ptr() + 8 * r * cells for q in range(2)])
            ex.world, ex.rank = 2, r
            _lib.check(_lib.lib().mlb_spread_peers(b.ptr, _lib.ptr(torch.from_numpy(v[lo:hi]).cuda()), ex.slots[0], 2,
                                                   0, _lib.stream_ptr()))
            grids.append(ex)
        out = []
        for r in range(2):
            g = torch.empty(cells, dtype=torch.float64, device="cuda")
            _lib.check(_lib.lib().mlb_grid_sum_slots(_lib.ptr(recv[r]), 2, cells, _lib.ptr(g), _lib.stream_ptr()))
            out.append(g.cpu().numpy())
        os.environ.pop("MLB_LATTICE", None)
        assert np.array_equal(out[0], out[1])
        assert rel(out[0], ref.cpu().numpy()) < 1e-13


@pytest.mark.parametrize("d,m", [(1, 4), (2, 4), (3, 4), (3, 5), (3, 6), (3, 3)])
def test_tiny_and_ragged_sizes_match_oracle(d, m):
    """Partial sub-chunks, single-point cells, one-item CTAs, 1 / 2 / 31 / 33 /
    65 / 257 points, clustered so one cell holds many of them."""
    from paper_2007_05239_b200 import KernelSpec, bind_points, build_plan, fastsum_apply
    rng = np.random.default_rng(40 + 10 * d + m)
    plan = build_plan(KernelSpec("gaussian", 0.15), d=d, N=32, m_nfft=m, p_nfft=8)
    oplan = fo.OraclePlan("gaussian", 0.15, d, 32, m, p=8)
    hw = fo.box_halfwidth(1.0 / 16)
    for n in (1, 2, 31, 33, 65, 257):
        pts = np.clip(0.01 * rng.standard_normal((n, d)) + rng.uniform(-0.1, 0.1, d), -hw, hw)
        pts[: n // 3] = pts[0]  # a heavy cell
        v = rng.standard_normal(n)
        got = fastsum_apply(None, v, plan, binding=bind_points(plan, pts))
        ref = fo.fastsum(oplan, v, points=pts)
        # scale by |v| too: for n = 1 the result is the O(1e-8) NFFT residual of W v = 0
        err = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), np.linalg.norm(v))
        assert err < 1e-11, (n, err)


def test_device_bind_paths_agree_and_validate():
    """mlb_bind_ex: host points, device points and the device box map of raw
    feature columns (feature_group's scaling folded into the bind) give the
    same binding -- identical permutation, bitwise identical degrees -- and
    the device-side validate_box raises the reference's ConfigErrors."""
    import torch
    from paper_2007_05239_b200 import (ConfigError, GroupingSpec, GroupSpec, KernelSpec, KernelWeights, bind_points,
                                       build_layer, build_plan, datapipe, feature_group)
    from paper_2007_05239_b200.fastsum import PointBinding
    rng = np.random.default_rng(77)
    n = 20000
    X = np.concatenate([rng.normal(0.3, 0.1, (n, 3)), rng.uniform(-5, 7, (n, 2))], axis=1)
    spec = GroupingSpec((GroupSpec((0, 1, 2), KernelSpec("gaussian", 0.1)), GroupSpec((3, 4), KernelSpec("gaussian", 1.0))))
    params = dict(N=32, m_nfft=4, p_nfft=8)
    G = feature_group(X, spec, fastsum_params=params)
    for g, layer in zip(spec.groups, G.layers):
        Xb, kb = datapipe.box_points(X[:, list(g.columns)], g.kernel)
        plan = build_plan(kb, d=len(g.columns), **params)
        ref = build_layer(KernelWeights(Xb, kb, plan=plan))
        assert np.array_equal(layer.degrees, ref.degrees)
        assert np.array_equal(layer.weights._bindings[0].sorted_perm(), ref.weights._bindings[0].sorted_perm())
        assert np.array_equal(layer.weights.points, Xb)           # lazily materialised box coordinates
        bd = PointBinding(plan, torch.from_numpy(Xb).cuda(), plan.ball_scale, validate=True)
        assert np.array_equal(bd.sorted_perm(), ref.weights._bindings[0].sorted_perm())
    plan = build_plan(KernelSpec("gaussian", 0.1), d=2, N=16, m_nfft=4, p_nfft=8)
    with pytest.raises(ConfigError, match="points exceed the admissible box"):
        bind_points(plan, np.array([[0.0, 0.1], [0.3, 0.0]]))
    with pytest.raises(ConfigError, match="non-finite"):
        bind_points(plan, np.array([[0.0, np.nan]]))
    assert bind_points(plan, np.zeros((0, 2))).n == 0


@pytest.mark.parametrize("d", [1, 2, 3])
def test_bare_nfft_matches_naive_dft_and_oracle(d):
    """The reference's own naive-DFT checks of nfft_adjoint / nfft_forward
    (test_fastsum.py:48-73, there for d = 1, 2) extended to d = 3: GPU
    transforms vs the naive sums (the reference's assert_allclose bar) and vs the
    numpy oracle of the reference algorithm (<= 1e-12); adjointness."""
    from paper_2007_05239_b200 import KernelSpec, build_plan
    from paper_2007_05239_b200.fastsum import nfft_adjoint, nfft_forward
    rng = np.random.default_rng(10 + d)
    N, n = 16, 37
    plan = build_plan(KernelSpec("gaussian", 0.2), d=d, N=N)
    oplan = fo.OraclePlan("gaussian", 0.2, d, N, 5, p=5)
    pts = rng.uniform(-0.5, 0.4999, size=(n, d))
    v = rng.standard_normal(n)
    ax = np.fft.fftfreq(N) * N
    freqs = np.stack([m.ravel() for m in np.meshgrid(*([ax] * d), indexing="ij")], axis=1)
    adj = nfft_adjoint(pts, v, plan)
    naive = np.exp(-2j * np.pi * (freqs @ pts.T)) @ v
    # the reference's bar: assert_allclose(got, naive, atol=1e-9 max|naive|), rtol default
    np.testing.assert_allclose(adj.ravel(), naive, atol=1e-9 * np.abs(naive).max())
    ref = fo.nfft_adjoint(oplan, pts, v)
    assert np.abs(adj - ref).max() <= 1e-12 * np.abs(ref).max()
    c = rng.standard_normal((N,) * d) + 1j * rng.standard_normal((N,) * d)
    fwd = nfft_forward(c, pts, plan)
    naive = np.exp(+2j * np.pi * (pts @ freqs.T)) @ c.ravel()
    np.testing.assert_allclose(fwd, naive, atol=1e-9 * np.abs(naive).max())
    ref = fo.nfft_forward(oplan, c, pts)
    assert np.abs(fwd - ref).max() <= 1e-12 * np.abs(ref).max()
    lhs, rhs = np.sum(fwd * v), np.sum(c * np.conj(adj))
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)


def _lattice_points(W, H, lo=-0.2, hi=0.2, transpose=False):
    """Pixel coordinates of a W x H image in the box (node = row * W + col)."""
    xs, ys = np.linspace(lo, hi, W), np.linspace(-0.2, 0.2, H)
    X, Y = np.meshgrid(xs, ys)   # row-major: Y constant along a row
    pts = np.stack([X.ravel(), Y.ravel()], axis=1)
    return pts[:, ::-1].copy() if transpose else pts


@pytest.mark.parametrize("layout,m", [("image", 5), ("image_t", 4), ("mixed", 5), ("image", 3), ("cut", 6),
                                      ("cut_t", 5), ("image", 2)])
def test_lattice_d2_kernels_match_oracle(layout, m):
    """The d = 2 lattice kernels (cells whose points form R x C product sets:
    spread = Ws^T (SV Wf), gather = (Ws G) Wf^T; non-lattice cells as
    diagonal items) forced on: spread grid vs the oracle, fastsum and the
    fused Laplacian epilogue (node / cell order, accumulate) vs the general
    kernels (MLB_LATTICE=0), repeated spreads bitwise identical."""
    import os

    import torch
    from paper_2007_05239_b200 import KernelSpec, bind_points, build_plan
    from paper_2007_05239_b200 import _lib
    from paper_2007_05239_b200.fastsum import fastsum_apply
    rng = np.random.default_rng(31)
    if layout in ("image", "image_t"):
        pts = _lattice_points(173, 151, transpose=layout == "image_t")
    elif layout == "mixed":   # an image plus scattered points (diagonal items)
        img = _lattice_points(120, 90, -0.2, 0.0)
        pts = np.concatenate([img, rng.uniform(0.02, 0.2, size=(3000, 2)), img[::97] + 1e-3])
    else:                     # a node range cutting rows (a shard of an image)
        pts = _lattice_points(160, 160, transpose=layout == "cut_t")[1234:21234]
    n = len(pts)
    v = rng.standard_normal(n)
    plan = build_plan(KernelSpec("gaussian", 0.1), d=2, N=64, m_nfft=m, p_nfft=8)
    lib = _lib.lib()
    L, ulo = None, None
    try:
        os.environ["MLB_LATTICE"] = "1"
        b = bind_points(plan, pts)
        st = b.stats()
        assert st["lattice_items"] > 0
        # (a node range cutting rows: partial first / last runs are segments of their own)
        assert st["lattice_points"] >= (0.5 * n if not layout.startswith("cut") else 0.95 * n)
        L, ulo = b._plan_handle.L, b._plan_handle.ulo
        vd = torch.from_numpy(v).cuda()
        grids = []
        for _ in range(2):
            g = torch.zeros(L * L, dtype=torch.float64, device="cuda")
            _lib.check(lib.mlb_spread(b.ptr, _lib.ptr(vd), _lib.ptr(g), 0, _lib.stream_ptr()))
            grids.append(g.cpu().numpy())
        y_lat = fastsum_apply(pts, v, plan, binding=b)
        os.environ["MLB_LATTICE"] = "0"
        b0 = bind_points(plan, pts)
        assert b0.stats()["lattice_items"] == 0
        y_gen = fastsum_apply(pts, v, plan, binding=b0)
    finally:
        del os.environ["MLB_LATTICE"]
    assert np.array_equal(grids[0], grids[1])
    op = fo.OraclePlan("gaussian", 0.1, 2, 64, m, p=8)
    full = fo.spread(fo.bind(op, pts), v).reshape(op.ng, op.ng)
    idx = np.mod(np.arange(ulo, ulo + L), op.ng)
    assert rel(grids[0].reshape(L, L), full[np.ix_(idx, idx)]) < 1e-13
    assert rel(y_lat, y_gen) < 1e-13
    ref = fo.fastsum(op, v, points=pts) if n <= 20000 else None
    if ref is not None:
        assert rel(y_lat, ref) < 1e-12
    # fused epilogue: y = a v + s (b acc + c s v), node and cell order, accumulate
    s = torch.from_numpy(rng.uniform(0.5, 2.0, n)).cuda()
    for bb in (b, b0):
        _lib.check(lib.mlb_binding_set_isd(bb.ptr, _lib.ptr(s), _lib.stream_ptr()))
    outs = []
    for bb in (b, b0):
        y = torch.full((n,), 0.25, dtype=torch.float64, device="cuda")
        _lib.check(lib.mlb_apply(bb.ptr, _lib.ptr(vd), _lib.ptr(y), 1.3, -0.7, 0.2, 1 | 2, _lib.stream_ptr()))
        perm = torch.from_numpy(bb.sorted_perm().astype(np.int64)).cuda()
        vs = vd[perm].contiguous()
        ys = torch.empty_like(vs)
        _lib.check(lib.mlb_apply(bb.ptr, _lib.ptr(vs), _lib.ptr(ys), 1.3, -0.7, 0.2, 1 | 4, _lib.stream_ptr()))
        yn = torch.empty_like(ys)
        yn[perm] = ys
        outs.append((y.cpu().numpy(), yn.cpu().numpy()))
    assert rel(outs[0][0], outs[1][0]) < 1e-13
    assert rel(outs[0][1], outs[1][1]) < 1e-13
