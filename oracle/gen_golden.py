"""Generate tests/golden/*.npz by running the REAL reference (build container only).

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden.py

The reference (`multilap` 0.1.0) is pure Python and importable here but does
not exist on the GPU box, so its outputs are frozen as small fixtures.  The
fixtures pin both the numpy oracle (tests/test_oracle_golden.py) and the GPU
path (tests/test_gpu_parity.py).  Inputs are seeded; sizes are chosen so
the oracle reproduces every case in seconds.
"""

import math
import os
import sys

import numpy as np

REF = os.environ.get("MULTILAP_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

import multilap  # noqa: E402
from multilap import fastsum, graphs, krylov, powermean, allencahn, datapipe  # noqa: E402
from multilap.kernels import KernelSpec  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")

# (family, sigma, d, N, m, p) -- plans whose fused weights are stored whole
SMALL_PLANS = [
    ("gaussian", 0.3, 1, 16, 4, 5),
    ("gaussian", 0.05, 1, 64, 6, 8),
    ("gaussian", 0.2, 2, 16, 3, 8),
    ("gaussian", 0.15, 2, 32, 4, 8),
    ("laplacian", 0.3, 2, 16, 4, 5),
    ("gaussian", 0.1, 3, 16, 4, 8),
    ("gaussian", 0.25, 3, 16, 6, 5),
    ("gaussian", 0.2, 2, 64, 5, 5),
]
# plans pinned by checksums only (too large to store)
BIG_PLANS = [
    ("gaussian", 0.1, 3, 32, 4, 8),
    ("gaussian", 0.1, 3, 64, 4, 8),
    ("gaussian", 0.1, 3, 64, 5, 5),
]


def box_points(rng, n, d, eps_b=fastsum.DEFAULT_EPS_B):
    hw = fastsum.box_halfwidth(eps_b)
    return rng.uniform(-hw, hw, size=(n, d))


def ball_points(rng, n, d, radius=0.21875):
    g = rng.standard_normal((n, d))
    g /= np.linalg.norm(g, axis=1, keepdims=True)
    return g * (radius * rng.random(n) ** (1.0 / d))[:, None]


def plan_key(fam, s, d, N, m, p):
    return f"{fam}_s{s}_d{d}_N{N}_m{m}_p{p}"


def gen_window():
    out = {}
    for m in (2, 3, 4, 5, 6):
        b = 1.5 * math.pi
        f = np.concatenate([np.linspace(0.0, 1.0, 257)[:-1], [0.5, 1e-17, 1 - 2 ** -52]])
        t = (f[:, None] - np.arange(-m, m + 1)[None, :]).ravel()
        out[f"t_m{m}"] = t
        out[f"phi_m{m}"] = fastsum._kb_window(t, m, b)
    return out


def gen_plans():
    out = {}
    for spec in SMALL_PLANS:
        fam, s, d, N, m, p = spec
        plan = fastsum.build_plan(KernelSpec(fam, s), d=d, N=N, m_nfft=m, p_nfft=p)
        k = plan_key(*spec)
        out[k + "/fused"] = plan.fused_weights
        out[k + "/deconv"] = plan.deconv_axis
        out[k + "/coeffs_real"] = plan.coeffs.real
    for spec in BIG_PLANS:
        fam, s, d, N, m, p = spec
        plan = fastsum.build_plan(KernelSpec(fam, s), d=d, N=N, m_nfft=m, p_nfft=p)
        k = plan_key(*spec)
        fw = plan.fused_weights
        out[k + "/checksum"] = np.array([fw.sum(), (fw * fw).sum(), np.abs(fw).max()])
        idx = np.random.default_rng(5).integers(0, fw.size, 512)
        out[k + "/sample_idx"] = idx
        out[k + "/sample_val"] = fw.ravel()[idx]
    return out


FASTSUM_CASES = [
    # name, (family, sigma, d, N, m, p), n, seed, point generator
    ("d1_n400", ("gaussian", 0.05, 1, 64, 6, 8), 400, 1, "box"),
    ("d1_n300_m4", ("gaussian", 0.3, 1, 16, 4, 5), 300, 2, "box"),
    ("d2_n500", ("gaussian", 0.15, 2, 32, 4, 8), 500, 3, "box"),
    ("d2_n500_m3", ("gaussian", 0.2, 2, 16, 3, 8), 500, 4, "ball"),
    ("d2_n400_lap", ("laplacian", 0.3, 2, 16, 4, 5), 400, 5, "box"),
    ("d2_n300_N64m5", ("gaussian", 0.2, 2, 64, 5, 5), 300, 6, "box"),
    ("d3_n300", ("gaussian", 0.1, 3, 16, 4, 8), 300, 7, "box"),
    ("d3_n250_m6", ("gaussian", 0.25, 3, 16, 6, 5), 250, 8, "ball"),
    ("d3_n300_N32", ("gaussian", 0.1, 3, 32, 4, 8), 300, 9, "ball"),
    ("d3_n200_N64m5", ("gaussian", 0.1, 3, 64, 5, 5), 200, 10, "ball"),
]


def gen_fastsum():
    out = {}
    for name, spec, n, seed, gen in FASTSUM_CASES:
        fam, s, d, N, m, p = spec
        rng = np.random.default_rng(seed)
        pts = box_points(rng, n, d) if gen == "box" else ball_points(rng, n, d)
        if name.startswith("d2_n500") and gen == "box":
            # exact grid-node points (integer ng*x/sqrt(d)) and box corners
            ng = 2 * N
            pts[:4] = np.array([[0.0, 0.0], [4.0, -2.0], [-6.0, 3.0], [1.0, 1.0]]) * math.sqrt(2) / ng
            pts[4] = [fastsum.box_halfwidth(fastsum.DEFAULT_EPS_B)] * 2
            pts[5] = [-fastsum.box_halfwidth(fastsum.DEFAULT_EPS_B)] * 2
        v = rng.standard_normal(n)
        plan = fastsum.build_plan(KernelSpec(fam, s), d=d, N=N, m_nfft=m, p_nfft=p)
        out[name + "/points"] = pts
        out[name + "/v"] = v
        out[name + "/Wv"] = fastsum.fastsum_apply(pts, v, plan)
        out[name + "/ones"] = fastsum.fastsum_apply(pts, np.ones(n), plan)
        out[name + "/spec"] = np.array([0 if fam == "gaussian" else 1, s, d, N, m, p], dtype=float)
        if n <= 400:
            out[name + "/direct"] = fastsum.direct_apply(pts, v, KernelSpec(fam, s))
    # the two-point hand sum (test_fastsum.py:180-188)
    plan = fastsum.build_plan(KernelSpec("gaussian", 0.1), d=2)
    pts = np.array([[-0.1, 0.0], [0.1, 0.0]])
    out["two_point/points"] = pts
    out["two_point/v"] = np.array([1.0, 2.0])
    out["two_point/Wv"] = fastsum.fastsum_apply(pts, np.array([1.0, 2.0]), plan)
    return out


def gen_nfft():
    out = {}
    for d in (1, 2):
        rng = np.random.default_rng(40 + d)
        N, n = 16, 37
        plan = fastsum.build_plan(KernelSpec("gaussian", 0.2), d=d, N=N)
        pts = rng.uniform(-0.5, 0.4999, size=(n, d))
        v = rng.standard_normal(n)
        c = rng.standard_normal((N,) * d) + 1j * rng.standard_normal((N,) * d)
        out[f"d{d}/points"] = pts
        out[f"d{d}/v"] = v
        out[f"d{d}/coeffs"] = c
        out[f"d{d}/adjoint"] = fastsum.nfft_adjoint(pts, v, plan)
        out[f"d{d}/forward"] = fastsum.nfft_forward(c, pts, plan)
    return out


def kernel_layer(pts, fam, s, N, m, p):
    plan = fastsum.build_plan(KernelSpec(fam, s), d=pts.shape[1], N=N, m_nfft=m, p_nfft=p)
    return graphs.build_layer(graphs.KernelWeights(pts, KernelSpec(fam, s), plan=plan))


def clustered_points(rng, n, d, k=4, spread=0.03):
    cent = rng.uniform(-0.15, 0.15, size=(k, d))
    lab = rng.integers(0, k, n)
    pts = cent[lab] + spread * rng.standard_normal((n, d))
    hw = fastsum.box_halfwidth(fastsum.DEFAULT_EPS_B)
    return np.clip(pts, -hw, hw), lab


def gen_solvers():
    out = {}
    rng = np.random.default_rng(50)
    n = 400
    p3, lab = clustered_points(rng, n, 3, k=3, spread=0.04)
    p2 = ball_points(rng, n, 2)
    L3 = kernel_layer(p3, "gaussian", 0.15, 32, 4, 8)
    L2 = kernel_layer(p2, "gaussian", 0.2, 32, 4, 8)
    out["pts3"], out["pts2"], out["truth"] = p3, p2, lab
    out["spec3"] = np.array([0, 0.15, 3, 32, 4, 8.0])
    out["spec2"] = np.array([0, 0.2, 2, 32, 4, 8.0])
    out["deg3"], out["deg2"] = L3.degrees, L2.degrees
    v = rng.standard_normal(n)
    out["v"] = v
    dl = math.log(2.0)
    out["Lv3_shift"] = graphs.apply_sym_laplacian(graphs.with_shift(L3, dl), v)
    out["Lv2_noshift"] = graphs.apply_sym_laplacian(L2, v)
    out["pksm3"] = krylov.pksm_apply(graphs.with_shift(L3, dl), -1.0, v)
    out["pksm2_p5"] = krylov.pksm_apply(graphs.with_shift(L2, math.log(6.0)), -5.0, v)
    G = graphs.MultilayerGraph((L3, L2))
    cfg = powermean.PowerMeanConfig(p=-1.0)
    out["Lp_apply"] = powermean.apply_Lp_power(G.with_shift(dl), cfg, v)
    out["one_minus_L1"] = powermean.apply_one_minus_L1(G, v)
    basis = powermean.power_mean_eigs(G, cfg, k=5, seed=0)
    out["eig_m1_values"], out["eig_m1_vectors"] = basis.values, basis.vectors
    basis1 = powermean.power_mean_eigs(G, powermean.PowerMeanConfig(p=1.0), k=5, seed=0)
    out["eig_p1_values"], out["eig_p1_vectors"] = basis1.values, basis1.vectors
    labels = datapipe.sample_labels(lab, 0.05, seed=3)
    out["label_ids"] = np.where(labels.labeled_mask, np.argmax(labels.F, axis=1), -1)
    res = allencahn.allen_cahn_solve(basis, labels, allencahn.AllenCahnParams())
    out["ac_scores"], out["ac_iters"] = res.scores, np.array([res.iterations, int(res.converged)])
    out["ac_pred"] = allencahn.predict_labels(res.scores)
    # hand values
    out["T_hand"] = allencahn.nonlinearity_T(np.array([[0.75, 0.25]]))
    Urand = np.random.default_rng(51).uniform(-2, 2, size=(64, 5))
    out["proj_in"], out["proj_out"] = Urand, allencahn.simplex_project_rows(Urand)
    out["T_in"], out["T_out"] = Urand, allencahn.nonlinearity_T(Urand)
    return out


def gen_featuregroup():
    out = {}
    rng = np.random.default_rng(60)
    n = 300
    X = np.concatenate([rng.random((n, 3)), rng.random((n, 2)) * 5.0 + 2.0], axis=1)
    spec = datapipe.GroupingSpec((
        datapipe.GroupSpec((0, 1, 2), KernelSpec("gaussian", 0.3)),
        datapipe.GroupSpec((3, 4), KernelSpec("gaussian", 1.0)),
    ))
    G = datapipe.feature_group(X, spec, fastsum_params=dict(N=32, m_nfft=4, p_nfft=8))
    out["X"] = X
    for t, lay in enumerate(G.layers):
        out[f"deg{t}"] = lay.degrees
        out[f"points{t}"] = lay.weights.points
        out[f"sigma{t}"] = np.array([lay.weights.kernel.sigma])
    return out


def gen_binary():
    """Binary Allen-Cahn and the Ginzburg-Landau energy (allencahn.py:232-314)
    on the eigenbasis frozen in golden_solvers.npz."""
    g = np.load(os.path.join(OUT, "golden_solvers.npz"))
    out = {}
    basis = powermean.SpectralBasis(values=g["eig_m1_values"], vectors=g["eig_m1_vectors"])
    truth = g["truth"]
    rng = np.random.default_rng(70)
    f = np.where(truth == 0, 1.0, -1.0)
    f[rng.random(f.shape[0]) > 0.1] = 0.0  # ~10 % labeled, +1 / -1
    out["f"] = f
    res = allencahn.binary_allen_cahn_solve(basis, f, allencahn.AllenCahnParams())
    out["bac_scores"] = res.scores
    out["bac_iters"] = np.array([res.iterations, int(res.converged)])
    out["bac_pred"] = allencahn.predict_binary(res.scores)
    ids = g["label_ids"]
    labels = allencahn.LabelData.from_class_ids(ids, int(ids.max()) + 1, 1000.0)
    U = g["ac_scores"]
    out["energy_basis"] = np.array([allencahn.ginzburg_landau_energy(U, basis, labels, 5e-3)])
    # dense-operator branch on a 64-node slice (the reference accepts any dense Laplacian)
    L2 = kernel_layer(g["pts2"], "gaussian", 0.2, 32, 4, 8)
    Ld = graphs.materialize_sym_laplacian(L2)[:64, :64]
    lab64 = allencahn.LabelData.from_class_ids(ids[:64], int(ids.max()) + 1, 1000.0)
    out["energy_dense64"] = np.array([allencahn.ginzburg_landau_energy(U[:64], Ld, lab64, 5e-3)])
    out["L_dense64"] = Ld
    return out


def main():
    os.makedirs(OUT, exist_ok=True)
    only = sys.argv[1:]  # e.g. `python oracle/gen_golden.py binary`
    for name, fn in [("window", gen_window), ("plans", gen_plans), ("fastsum", gen_fastsum),
                     ("nfft", gen_nfft), ("solvers", gen_solvers), ("featuregroup", gen_featuregroup),
                     ("binary", gen_binary)]:
        if only and name not in only:
            continue
        data = fn()
        path = os.path.join(OUT, f"golden_{name}.npz")
        np.savez_compressed(path, **data)
        print(f"wrote {path}: {len(data)} arrays, {os.path.getsize(path)/1e3:.1f} kB")
    with open(os.path.join(OUT, "SOURCE.txt"), "w") as fh:
        fh.write(f"generated by oracle/gen_golden.py from multilap {multilap.__version__} "
                 f"at {REF}; numpy {np.__version__}\n")


if __name__ == "__main__":
    main()
