"""Pin the numpy oracle against golden vectors produced by the real reference.

CPU only.  The golden fixtures come from oracle/gen_golden.py, which ran
`multilap` 0.1.0 from /root/reference in the build container.
"""

import math

import numpy as np
import pytest
from numpy.testing import assert_allclose

from conftest import load_golden
from oracle import fastsum_oracle as fo
from oracle import solvers_oracle as so

FAM = {0: "gaussian", 1: "laplacian"}


def _spec(arr):
    fam, s, d, N, m, p = arr
    return FAM[int(fam)], float(s), int(d), int(N), int(m), int(p)


def test_window_matches_reference_bitwise():
    g = load_golden("window")
    for m in (2, 3, 4, 5, 6):
        got = fo.kb_window(g[f"t_m{m}"], m, 1.5 * math.pi)
        assert np.array_equal(got, g[f"phi_m{m}"])


def test_small_plans_match_reference():
    g = load_golden("plans")
    keys = sorted({k.split("/")[0] for k in g.files})
    assert len(keys) == 11
    for k in keys:
        parts = k.split("_")
        fam, s = parts[0], float(parts[1][1:])
        d, N, m, p = (int(x[1:]) for x in parts[2:])
        plan = fo.OraclePlan(fam, s, d, N, m, p=p)
        if k + "/fused" in g.files:
            ref = g[k + "/fused"]
            assert_allclose(plan.fused, ref, rtol=0, atol=1e-13 * np.abs(ref).max())
            assert_allclose(plan.deconv_axis, g[k + "/deconv"], rtol=1e-14)
        else:
            fw = plan.fused
            cs = np.array([fw.sum(), (fw * fw).sum(), np.abs(fw).max()])
            assert_allclose(cs, g[k + "/checksum"], rtol=1e-12)
            assert_allclose(fw.ravel()[g[k + "/sample_idx"]], g[k + "/sample_val"],
                            atol=1e-13 * np.abs(fw).max())


@pytest.mark.parametrize("name", ["d1_n400", "d1_n300_m4", "d2_n500", "d2_n500_m3", "d2_n400_lap",
                                  "d2_n300_N64m5", "d3_n300", "d3_n250_m6", "d3_n300_N32",
                                  "d3_n200_N64m5"])
def test_fastsum_matches_reference(name):
    g = load_golden("fastsum")
    fam, s, d, N, m, p = _spec(g[name + "/spec"])
    plan = fo.OraclePlan(fam, s, d, N, m, p=p)
    pts, v = g[name + "/points"], g[name + "/v"]
    b = fo.bind(plan, pts)
    ref = g[name + "/Wv"]
    got = fo.fastsum(plan, v, binding=b)
    assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref)
    assert_allclose(fo.fastsum(plan, np.ones(len(v)), binding=b), g[name + "/ones"], rtol=1e-12)
    # chunked restatement (config 4/5 oracle) agrees up to summation order
    got_c = fo.fastsum_chunked(plan, pts, v, chunk=97)
    assert np.linalg.norm(got_c - ref) <= 1e-13 * np.linalg.norm(ref)
    if name + "/direct" in g.files:
        assert_allclose(fo.direct(pts, v, fam, s), g[name + "/direct"], atol=1e-11)
    # the C restatement (full-size chunked oracle, oracle/c/mlb_oracle.c): W v and W 1
    # in one pass, on 3 host threads (a different summation order)
    from oracle import c_oracle as co
    both = co.fastsum_many(plan, pts, np.stack([v, np.ones(len(v))]), threads=3)
    assert np.linalg.norm(both[0] - ref) <= 1e-13 * np.linalg.norm(ref)
    assert_allclose(both[1], g[name + "/ones"], rtol=1e-12)


def test_c_oracle_window_matches_reference():
    from oracle import c_oracle as co
    g = load_golden("window")
    for m in (2, 3, 4, 5, 6):
        ref = g[f"phi_m{m}"]
        got = co.window(g[f"t_m{m}"], m, 1.5 * math.pi)
        assert np.abs(got - ref).max() <= 4e-16 * np.abs(ref).max(), m


def test_two_point_case():
    g = load_golden("fastsum")
    plan = fo.OraclePlan("gaussian", 0.1, 2)
    got = fo.fastsum(plan, g["two_point/v"], points=g["two_point/points"])
    assert_allclose(got, g["two_point/Wv"], rtol=1e-13)


@pytest.mark.parametrize("d", [1, 2])
def test_bare_nfft_matches_reference(d):
    g = load_golden("nfft")
    plan = fo.OraclePlan("gaussian", 0.2, d, 16)
    adj = fo.nfft_adjoint(plan, g[f"d{d}/points"], g[f"d{d}/v"])
    ref = g[f"d{d}/adjoint"]
    assert_allclose(adj, ref, atol=1e-13 * np.abs(ref).max())
    fwd = fo.nfft_forward(plan, g[f"d{d}/coeffs"], g[f"d{d}/points"])
    ref = g[f"d{d}/forward"]
    assert_allclose(fwd, ref, atol=1e-13 * np.abs(ref).max())


def _solver_layers(g):
    layers = []
    for key in ("3", "2"):
        fam, s, d, N, m, p = _spec(g["spec" + key])
        plan = fo.OraclePlan(fam, s, d, N, m, p=p)
        b = fo.bind(plan, g["pts" + key])
        layers.append(so.OracleLayer(lambda v, plan=plan, b=b: fo.fastsum(plan, v, binding=b), b.n))
    return layers


def test_solvers_match_reference():
    g = load_golden("solvers")
    L3, L2 = _solver_layers(g)
    assert_allclose(L3.degrees, g["deg3"], rtol=1e-13)
    assert_allclose(L2.degrees, g["deg2"], rtol=1e-13)
    v = g["v"]
    dl = math.log(2.0)
    assert_allclose(so.sym_laplacian(L3.shifted(dl), v), g["Lv3_shift"], atol=1e-12)
    assert_allclose(so.sym_laplacian(L2, v), g["Lv2_noshift"], atol=1e-12)
    assert_allclose(so.pksm(L3.shifted(dl), -1.0, v), g["pksm3"], atol=1e-11)
    assert_allclose(so.pksm(L2.shifted(math.log(6.0)), -5.0, v), g["pksm2_p5"], atol=1e-11)
    assert_allclose(so.apply_Lp_power([L3.shifted(dl), L2.shifted(dl)], -1.0, v), g["Lp_apply"], atol=1e-11)
    assert_allclose(so.apply_one_minus_L1([L3, L2], v), g["one_minus_L1"], atol=1e-12)


def test_eigs_and_allen_cahn_match_reference():
    g = load_golden("solvers")
    layers = _solver_layers(g)
    vals, vecs = so.power_mean_eigs(layers, -1.0, 5, seed=0)
    assert_allclose(vals, g["eig_m1_values"], rtol=1e-10)
    P = vecs @ vecs.T
    Pr = g["eig_m1_vectors"] @ g["eig_m1_vectors"].T
    assert np.abs(P - Pr).max() < 1e-7
    vals1, _ = so.power_mean_eigs(layers, 1.0, 5, seed=0)
    assert_allclose(vals1, g["eig_p1_values"], rtol=1e-9, atol=1e-12)
    ids = g["label_ids"]
    m = int(ids.max()) + 1
    F = np.zeros((len(ids), m))
    F[ids >= 0, ids[ids >= 0]] = 1.0
    fid = np.where(ids >= 0, 1000.0, 0.0)
    U, it, conv = so.allen_cahn(g["eig_m1_values"], g["eig_m1_vectors"], F, fid)
    assert_allclose(U, g["ac_scores"], atol=1e-10)
    assert [it, int(conv)] == list(g["ac_iters"])
    assert np.array_equal(so.predict(U), g["ac_pred"])


def test_allen_cahn_pieces_match_reference():
    g = load_golden("solvers")
    assert_allclose(so.well_force(np.array([[0.75, 0.25]])), g["T_hand"], atol=1e-15)
    assert_allclose(so.simplex_project(g["proj_in"]), g["proj_out"], atol=1e-15)
    assert_allclose(so.well_force(g["T_in"]), g["T_out"], rtol=1e-13, atol=1e-13)


def test_binary_allen_cahn_and_energy_match_reference():
    """Oracle binary scheme and Ginzburg-Landau energy vs the reference run
    frozen in golden_binary.npz (allencahn.py:232-314)."""
    gs = load_golden("solvers")
    gb = load_golden("binary")
    u, it, conv = so.binary_allen_cahn(gs["eig_m1_values"], gs["eig_m1_vectors"], gb["f"])
    assert [it, int(conv)] == list(gb["bac_iters"])
    assert np.abs(u - gb["bac_scores"]).max() < 1e-12
    assert np.array_equal(so.predict_binary(u), gb["bac_pred"])
    ids = gs["label_ids"]
    m = int(ids.max()) + 1
    F = np.zeros((ids.size, m))
    F[ids >= 0, ids[ids >= 0]] = 1.0
    fid = np.where(ids >= 0, 1000.0, 0.0)
    e = so.gl_energy(gs["ac_scores"], gs["eig_m1_values"], gs["eig_m1_vectors"], F, fid, 5e-3)
    assert abs(e - gb["energy_basis"][0]) <= 1e-12 * abs(gb["energy_basis"][0])
    e64 = so.gl_energy(gs["ac_scores"][:64], None, None, F[:64], fid[:64], 5e-3, L_dense=gb["L_dense64"])
    assert abs(e64 - gb["energy_dense64"][0]) <= 1e-12 * abs(gb["energy_dense64"][0])


def test_parallel_reference_arm_matches_serial_oracle():
    """bench.py's multi-process reference arm (oracle/parallel_ref.py) computes
    the same shifted normalized-Laplacian matvecs as the serial oracle."""
    from oracle.parallel_ref import check_against_serial
    rng = np.random.default_rng(5)
    hw = fo.box_halfwidth(1.0 / 16)
    specs = []
    for d, N in ((3, 16), (2, 32)):
        pts = np.clip(0.05 * rng.standard_normal((700, d)), -hw, hw)
        specs.append((fo.OraclePlan("gaussian", 0.12, d, N, 4, p=8), pts))
    v = rng.standard_normal(700)
    assert check_against_serial(specs, math.log(2.0), v, procs=3) < 1e-13
    # workers started from a clean interpreter (what CUDA-running callers use)
    assert check_against_serial(specs, math.log(2.0), v, procs=2, start_method="forkserver") < 1e-13
