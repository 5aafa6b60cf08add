"""GPU parity of the Krylov / power-mean / Allen-Cahn path against reference
golden vectors and the numpy oracle.

North-star tolerances: eigenvalues within 1e-7 (relative), labels identical
on >= 99.9% of nodes; PKSM / operator applies within 1e-8.
"""

import math

import numpy as np
import pytest
from numpy.testing import assert_allclose

from conftest import load_golden
from oracle import solvers_oracle as so

pytestmark = pytest.mark.gpu
FAM = {0: "gaussian", 1: "laplacian"}


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _layers(g):
    from paper_2007_05239_b200 import KernelSpec, KernelWeights, build_layer, build_plan
    out = []
    for key in ("3", "2"):
        fam, s, d, N, m, p = g["spec" + key]
        kern = KernelSpec(FAM[int(fam)], float(s))
        plan = build_plan(kern, d=int(d), N=int(N), m_nfft=int(m), p_nfft=int(p))
        out.append(build_layer(KernelWeights(g["pts" + key], kern, plan=plan)))
    return out


def test_pksm_and_power_operators_match_golden():
    from paper_2007_05239_b200 import MultilayerGraph, PowerMeanConfig, apply_Lp_power, apply_one_minus_L1
    from paper_2007_05239_b200 import pksm_apply, with_shift
    g = load_golden("solvers")
    L3, L2 = _layers(g)
    v = g["v"]
    dl = math.log(2.0)
    assert rel(pksm_apply(with_shift(L3, dl), -1.0, v), g["pksm3"]) < 1e-9
    assert rel(pksm_apply(with_shift(L2, math.log(6.0)), -5.0, v), g["pksm2_p5"]) < 1e-9
    G = MultilayerGraph((L3, L2))
    assert rel(apply_Lp_power(G.with_shift(dl), PowerMeanConfig(p=-1.0), v), g["Lp_apply"]) < 1e-9
    assert rel(apply_one_minus_L1(G, v), g["one_minus_L1"]) < 1e-12


def test_batched_pksm_is_bitwise_sequential():
    """The lockstep multi-layer PKSM (one graph replay and one host read per
    step for all layers) reproduces the per-layer loop: bit for bit with the
    host's batched eigh (MLB_PKSM_DEVICE_COEFFS=0), to rounding (<= 1e-13)
    with the coefficients on the device (default); the layer-order sum too."""
    import os

    import torch
    from paper_2007_05239_b200 import with_shift
    from paper_2007_05239_b200.krylov import pksm_layer_dev, pksm_layers_dev
    g = load_golden("solvers")
    L3, L2 = _layers(g)
    dl = math.log(2.0)
    layers = [with_shift(L3, dl), with_shift(L2, dl), with_shift(L3, dl)]
    v = torch.from_numpy(g["v"]).cuda()
    for p in (-1.0, -3.0):
        seq = torch.zeros_like(v)
        for layer in layers:
            pksm_layer_dev(layer, p, v, seq, 1.0, True)
        bat = torch.zeros_like(v)
        pksm_layers_dev(layers, p, v, bat, 1.0)
        assert rel(bat.cpu().numpy(), seq.cpu().numpy()) < 1e-13
        os.environ["MLB_PKSM_DEVICE_COEFFS"] = "0"
        try:
            hb = torch.zeros_like(v)
            pksm_layers_dev(layers, p, v, hb, 1.0)
        finally:
            del os.environ["MLB_PKSM_DEVICE_COEFFS"]
        assert torch.equal(seq, hb)
    # the device's run-ahead depth changes no value (discarded steps only)
    res, resb = [], []
    for depth in ("1", "3"):
        os.environ["MLB_PKSM_DEPTH"] = depth
        try:
            a = torch.zeros_like(v)
            for layer in layers:
                pksm_layer_dev(layer, -1.0, v, a, 1.0, True)
            b = torch.zeros_like(v)
            pksm_layers_dev(layers, -1.0, v, b, 1.0)
        finally:
            del os.environ["MLB_PKSM_DEPTH"]
        assert rel(b.cpu().numpy(), a.cpu().numpy()) < 1e-13
        res.append(a)
        resb.append(b)
    assert torch.equal(res[0], res[1]) and torch.equal(resb[0], resb[1])


@pytest.mark.parametrize("p", [-1.0, -3.0, 0.5, 2.0])
def test_device_tridiagonal_coefficients_match_host_eigh(p):
    """mlb_tridiag_fn_batched (implicit QL per warp) against the host's batched
    eigh (krylov._coeffs, the reference's krylov.py:200-206 arithmetic) on
    random Lanczos-like tridiagonals, every step j of dim = 64 chains, plus the
    stop statistics and the min eigenvalue of an indefinite chain."""
    import ctypes as C

    import torch
    from paper_2007_05239_b200 import _lib
    from paper_2007_05239_b200.krylov import _coeffs
    rng = np.random.default_rng(11)
    T, dim = 5, 64
    ld = 2 * dim + 5
    al = rng.uniform(2.0, 3.0, (T, dim))               # Gershgorin: lambda >= 0.2
    be = rng.uniform(0.0, 0.9, (T, dim))
    be[1, 7] = 0.0                                   # an exactly split matrix
    al[4, :] = rng.uniform(-1.0, 1.0, dim)           # indefinite chain
    vv = rng.uniform(0.5, 4.0, T)
    AB = torch.zeros((T, ld), dtype=torch.float64, device="cuda")
    hist = torch.zeros((T, 2 * dim), dtype=torch.float64, device="cuda")
    Cc = torch.zeros((T, dim, dim), dtype=torch.float64, device="cuda")
    lib = _lib.lib()
    fn = lambda lam: np.maximum(lam, 0.0) ** p   # noqa: E731
    prev = None
    for j in range(dim):
        row = np.zeros((T, ld))
        row[:, j] = al[:, j]
        row[:, dim + j] = be[:, j] ** 2
        row[:, 2 * dim] = vv
        AB.copy_(torch.from_numpy(row))
        _lib.check(lib.mlb_tridiag_fn_batched(T, C.c_void_p(AB.data_ptr()), ld, dim, j, p,
                                              C.c_void_p(hist.data_ptr()), C.c_void_p(Cc.data_ptr()), _lib.stream_ptr()))
        out = AB.cpu().numpy()
        s = j + 1
        lam = np.array([np.linalg.eigvalsh(np.diag(al[t, :s]) + np.diag(be[t, :s - 1], 1) + np.diag(be[t, :s - 1], -1))
                        for t in range(T)])
        assert np.all(out[:, 2 * dim + 4] == 0)
        if p == -1.0:   # T^{-1} e1 by one LDL^T solve: SPD chains report a positive pivot, others the QL minimum
            spd = lam.min(axis=1) > 0
            assert np.all(out[spd, 2 * dim + 1] > 0)
            assert np.allclose(out[~spd, 2 * dim + 1], lam.min(axis=1)[~spd], rtol=0, atol=1e-13 * np.abs(lam).max())
        else:
            assert np.allclose(out[:, 2 * dim + 1], lam.min(axis=1), rtol=0, atol=1e-13 * np.abs(lam).max())
        ok = [t for t in range(T) if lam[t].min() > 1e-3]   # the power is defined on these chains
        ref = _coeffs(al[ok], be[ok], s, np.sqrt(vv[ok]), fn)
        got = Cc[ok, j, :s].cpu().numpy()
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max(), j
        assert np.allclose(out[ok, 2 * dim + 2], (ref * ref).sum(axis=1), rtol=1e-12)
        if prev is not None:
            d = ref.copy()
            d[:, :s - 1] -= prev
            # ||c - c_prev|| to rounding relative to ||c|| (what the stop test compares it with)
            err = np.abs(np.sqrt(out[ok, 2 * dim + 3]) - np.sqrt((d * d).sum(axis=1)))
            assert np.all(err <= 1e-13 * np.sqrt((ref * ref).sum(axis=1)))
        prev = ref
    assert np.array_equal(hist[:, :dim].cpu().numpy(), al)
    assert np.array_equal(hist[:, dim:].cpu().numpy(), np.sqrt(be ** 2))


def test_power_mean_eigs_match_golden():
    from paper_2007_05239_b200 import MultilayerGraph, PowerMeanConfig, power_mean_eigs
    g = load_golden("solvers")
    G = MultilayerGraph(tuple(_layers(g)))
    basis = power_mean_eigs(G, PowerMeanConfig(p=-1.0), k=5, seed=0)
    assert_allclose(basis.values, g["eig_m1_values"], rtol=1e-7)
    P = basis.vectors @ basis.vectors.T
    Pr = g["eig_m1_vectors"] @ g["eig_m1_vectors"].T
    assert np.abs(P - Pr).max() < 1e-6
    b1 = power_mean_eigs(G, PowerMeanConfig(p=1.0), k=5, seed=0)
    assert_allclose(b1.values, g["eig_p1_values"], rtol=1e-7, atol=1e-10)
    # bitwise seed determinism (test_powermean.py:152-159)
    again = power_mean_eigs(G, PowerMeanConfig(p=-1.0), k=5, seed=0)
    assert np.array_equal(again.values, basis.values)
    assert np.array_equal(again.vectors, basis.vectors)
    # the per-layer solves of large layers, one after the other and run
    # concurrently (a stream and a host thread each): bitwise the same
    from paper_2007_05239_b200 import powermean as pm
    saved = pm._SEQ_GRAPHS, pm._CONCURRENT, pm._CONC_MIN_N
    try:
        got = {}
        for conc in (False, True):
            pm._SEQ_GRAPHS, pm._CONCURRENT, pm._CONC_MIN_N = False, conc, 0
            got[conc] = power_mean_eigs(G, PowerMeanConfig(p=-1.0), k=5, seed=0)
    finally:
        pm._SEQ_GRAPHS, pm._CONCURRENT, pm._CONC_MIN_N = saved
    assert np.array_equal(got[True].values, got[False].values)
    assert np.array_equal(got[True].vectors, got[False].vectors)
    assert_allclose(got[True].values, g["eig_m1_values"], rtol=1e-7)


def test_allen_cahn_matches_golden():
    from paper_2007_05239_b200 import AllenCahnParams, LabelData, SpectralBasis, allen_cahn_solve, predict_labels
    g = load_golden("solvers")
    ids = g["label_ids"]
    labels = LabelData.from_class_ids(ids, int(ids.max()) + 1, 1000.0)
    basis = SpectralBasis(values=g["eig_m1_values"], vectors=g["eig_m1_vectors"])
    res = allen_cahn_solve(basis, labels, AllenCahnParams())
    assert [res.iterations, int(res.converged)] == list(g["ac_iters"])
    assert np.abs(res.scores - g["ac_scores"]).max() < 1e-9
    assert np.array_equal(predict_labels(res.scores), g["ac_pred"])
    # the device runs one iteration ahead of the stopping test: the same
    # iterates as one at a time, and as with a callback (which sees each)
    import os
    seen = []
    os.environ["MLB_AC_DEPTH"] = "1"
    try:
        one = allen_cahn_solve(basis, labels, AllenCahnParams())
    finally:
        del os.environ["MLB_AC_DEPTH"]
    cb = allen_cahn_solve(basis, labels, AllenCahnParams(), callback=lambda it, U: seen.append(it))
    for other in (one, cb):
        assert other.iterations == res.iterations and other.converged == res.converged
        assert np.array_equal(other.scores, res.scores)
    assert seen == list(range(1, res.iterations + 1))
    capped = allen_cahn_solve(basis, labels, AllenCahnParams(max_iter=3))
    assert capped.iterations == 3 and not capped.converged


def test_end_to_end_labels_match_oracle():
    """feature layers -> eigs -> Allen-Cahn on GPU vs the oracle: >= 99.9% labels."""
    from paper_2007_05239_b200 import (AllenCahnParams, MultilayerGraph, PowerMeanConfig, allen_cahn_solve,
                                       power_mean_eigs, predict_labels, sample_labels)
    g = load_golden("solvers")
    G = MultilayerGraph(tuple(_layers(g)))
    basis = power_mean_eigs(G, PowerMeanConfig(p=-1.0), k=5, seed=0)
    labels = sample_labels(g["truth"], 0.05, seed=3)
    res = allen_cahn_solve(basis, labels, AllenCahnParams())
    pred = predict_labels(res.scores)
    U, _, _ = so.allen_cahn(g["eig_m1_values"], g["eig_m1_vectors"], labels.F, labels.fidelity)
    assert np.mean(pred == so.predict(U)) >= 0.999


def test_krylov_dense_operators():
    """Reference krylov tests on dense operators (test_krylov.py:22-166)."""
    from paper_2007_05239_b200 import NumericalError, SymmetricOperator, lanczos_fn_apply, lanczos_largest_eigs
    from paper_2007_05239_b200 import pksm_apply

    def matrix_op(A):
        return SymmetricOperator(A.shape[0], lambda v: A @ v)

    vals = np.linspace(0.1, 3.0, 40)
    res = lanczos_largest_eigs(matrix_op(np.diag(vals)), k=5, seed=1)
    assert_allclose(res.values, vals[-5:][::-1], atol=1e-9)
    rng = np.random.default_rng(2)
    A = rng.standard_normal((60, 60))
    A = 0.5 * (A + A.T)
    lam = np.linalg.eigvalsh(A)
    res = lanczos_largest_eigs(matrix_op(A), k=6, seed=0)
    assert_allclose(res.values, lam[::-1][:6], atol=1e-8 * np.abs(lam).max())
    got = pksm_apply(matrix_op(np.diag([1.0, 2.0, 4.0])), -1.0, np.ones(3))
    assert_allclose(got, [1.0, 0.5, 0.25], rtol=1e-12)
    B = rng.standard_normal((80, 80))
    A = B @ B.T / 80 + np.log(2) * np.eye(80)
    lam, Q = np.linalg.eigh(A)
    v = rng.standard_normal(80)
    oracle = (Q * lam ** -1.0) @ (Q.T @ v)
    assert rel(pksm_apply(matrix_op(A), -1.0, v), oracle) < 1e-8
    with pytest.raises(NumericalError):
        pksm_apply(matrix_op(np.diag([1.0, -0.5, 2.0])), -1.0, np.ones(3))
    with pytest.raises(NumericalError, match="symmetry"):
        lanczos_largest_eigs(matrix_op(rng.standard_normal((20, 20))), k=2)
    vals = np.linspace(-1.0, 1.0, 25)
    v = rng.standard_normal(25)
    got = lanczos_fn_apply(matrix_op(np.diag(vals)), v, np.exp, tol=1e-14)
    assert rel(got, np.exp(vals) * v) < 1e-12


def test_feature_group_matches_golden():
    from paper_2007_05239_b200 import GroupingSpec, GroupSpec, KernelSpec, feature_group
    g = load_golden("featuregroup")
    spec = GroupingSpec((GroupSpec((0, 1, 2), KernelSpec("gaussian", 0.3)),
                         GroupSpec((3, 4), KernelSpec("gaussian", 1.0))))
    G = feature_group(g["X"], spec, fastsum_params=dict(N=32, m_nfft=4, p_nfft=8))
    for t, lay in enumerate(G.layers):
        assert_allclose(lay.weights.points, g[f"points{t}"], rtol=0, atol=0)
        assert_allclose(lay.weights.kernel.sigma, g[f"sigma{t}"][0], rtol=1e-15)
        assert rel(lay.degrees, g[f"deg{t}"]) < 1e-13


def test_direct_apply_matches_oracle():
    from paper_2007_05239_b200 import KernelSpec, direct_apply
    g = load_golden("fastsum")
    for name in ("d1_n400", "d2_n400_lap", "d3_n300"):
        fam, s = FAM[int(g[name + "/spec"][0])], float(g[name + "/spec"][1])
        got = direct_apply(g[name + "/points"], g[name + "/v"], KernelSpec(fam, s))
        assert_allclose(got, g[name + "/direct"], atol=1e-11)


def test_config1_pipeline_matches_reference():
    """BASELINE configs[0] end to end (GPU) vs the reference run frozen in
    golden_cfg1.npz: eigenvalues <= 1e-7 relative, same Allen-Cahn iteration
    count, labels identical on >= 99.9% of the nodes."""
    import synth
    from paper_2007_05239_b200 import (AllenCahnParams, LabelData, PowerMeanConfig, allen_cahn_solve,
                                       power_mean_eigs, predict_labels)
    g = load_golden("cfg1")
    wl = synth.config1_toy(seed=0)
    assert np.array_equal(wl.X, g["X"])
    G = synth.build_graph(wl)
    assert rel(G.layers[0].degrees, g["deg0"]) < 1e-12
    assert rel(G.layers[1].degrees, g["deg1"]) < 1e-12
    basis = power_mean_eigs(G, PowerMeanConfig(p=-1.0), k=wl.k, seed=0)
    assert np.max(np.abs(basis.values - g["values"]) / np.abs(g["values"])) <= 1e-7
    P = basis.vectors @ basis.vectors.T
    Pr = g["vectors"] @ g["vectors"].T
    assert np.abs(P - Pr).max() < 1e-5
    ids = g["label_ids"]
    labels = LabelData.from_class_ids(ids, int(ids.max()) + 1, 1000.0)
    res = allen_cahn_solve(basis, labels, AllenCahnParams())
    pred = predict_labels(res.scores)
    assert np.mean(pred == g["pred"]) >= 0.999
    assert abs(res.iterations - int(g["iters"][0])) <= 1


def test_binary_allen_cahn_and_energy_match_golden():
    """GPU binary scheme (mlb_bac_step) and the energy diagnostic vs the
    reference run frozen in golden_binary.npz."""
    import torch
    from paper_2007_05239_b200 import (AllenCahnParams, LabelData, SpectralBasis, binary_allen_cahn_solve,
                                       ginzburg_landau_energy, predict_binary)
    gs = load_golden("solvers")
    gb = load_golden("binary")
    basis = SpectralBasis(values=gs["eig_m1_values"], vectors=gs["eig_m1_vectors"])
    res = binary_allen_cahn_solve(basis, gb["f"], AllenCahnParams())
    assert [res.iterations, int(res.converged)] == list(gb["bac_iters"])
    assert np.abs(res.scores - gb["bac_scores"]).max() < 1e-9
    assert np.array_equal(predict_binary(res.scores), gb["bac_pred"])
    d = binary_allen_cahn_solve(basis, torch.from_numpy(gb["f"]).cuda(), AllenCahnParams(), return_device=True)
    assert np.array_equal(predict_binary(d.scores).cpu().numpy(), gb["bac_pred"])
    with pytest.raises(Exception, match="binary labels"):
        binary_allen_cahn_solve(basis, 2.0 * gb["f"], AllenCahnParams())
    ids = gs["label_ids"]
    labels = LabelData.from_class_ids(ids, int(ids.max()) + 1, 1000.0)
    e = ginzburg_landau_energy(gs["ac_scores"], basis, labels, 5e-3)
    assert abs(e - gb["energy_basis"][0]) <= 1e-10 * abs(gb["energy_basis"][0])
    lab64 = LabelData.from_class_ids(ids[:64], int(ids.max()) + 1, 1000.0)
    e64 = ginzburg_landau_energy(gs["ac_scores"][:64], gb["L_dense64"], lab64, 5e-3)
    assert abs(e64 - gb["energy_dense64"][0]) <= 1e-10 * abs(gb["energy_dense64"][0])


def test_multi_layer_apply_matches_per_layer_apply():
    """mlb_apply_multi (one launch per stage for T small layers: config 3's
    lockstep matvec) against mlb_apply per layer, to rounding; the lockstep
    PKSM with and without it (MLB_PKSM_MULTI=0) agree to 1e-13."""
    import ctypes as C
    import os

    import torch

    import synth
    from paper_2007_05239_b200 import _lib, with_shift
    from paper_2007_05239_b200.krylov import pksm_layers_dev
    wl = synth.CONFIGS[3](seed=0)
    G = synth.build_graph(wl, device=0)
    layers = [with_shift(lay, math.log(2.0)) for lay in G.layers[:12]]
    T, n = len(layers), wl.n
    lib = _lib.lib()
    rng = np.random.default_rng(3)
    xs = [torch.from_numpy(rng.standard_normal(n)).cuda() for _ in range(T)]
    bs = [lay.weights._bindings[0] for lay in layers]
    for lay in layers:
        w = lay.weights
        if w._isd_dev is None:
            w.set_isd(lay.isd_device(w.device))
    ys = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(T)]
    ref = [torch.empty_like(y) for y in ys]
    abg = [1.0 + lay.shift for lay in layers] + [-1.0] * T + [lay.weights.kernel.value_at_zero() for lay in layers]
    flags = _lib.MLB_USE_ISD
    for t, b in enumerate(bs):
        _lib.check(lib.mlb_apply(b.ptr, _lib.ptr(xs[t]), _lib.ptr(ref[t]), abg[t], -1.0, abg[2 * T + t], flags,
                                 _lib.stream_ptr()))
    px = torch.tensor([x.data_ptr() for x in xs], dtype=torch.int64, device="cuda")
    py = torch.tensor([y.data_ptr() for y in ys], dtype=torch.int64, device="cuda")
    pabg = torch.tensor(abg, dtype=torch.float64, device="cuda")
    bh = (C.c_void_p * T)(*[b.ptr.value for b in bs])
    _lib.check(lib.mlb_apply_multi(bh, T, _lib.ptr(px), _lib.ptr(py), _lib.ptr(pabg), flags, _lib.stream_ptr()))
    for t in range(T):   # (its own CTA partition of each layer: summation order differs)
        assert rel(ys[t].cpu().numpy(), ref[t].cpu().numpy()) < 1e-14, t
    v = torch.from_numpy(rng.standard_normal(n)).cuda()
    out = torch.zeros_like(v)
    pksm_layers_dev(layers, -1.0, v, out, 1.0)
    os.environ["MLB_PKSM_MULTI"] = "0"
    try:
        out0 = torch.zeros_like(v)
        pksm_layers_dev(layers, -1.0, v, out0, 1.0)
    finally:
        del os.environ["MLB_PKSM_MULTI"]
    assert rel(out.cpu().numpy(), out0.cpu().numpy()) < 1e-13
