"""Host-side logic on CPU: the drop-in API pieces that need no GPU, checked
against the reference package itself when it is importable (this build
container: /root/reference/pkg/src; skipped elsewhere), plus the bench's
roofline bookkeeping and the sharded solvers' single-rank algebra."""

import math
import os
import sys

import numpy as np
import pytest

REF = os.environ.get("MULTILAP_REF", "/root/reference/pkg/src")


def _ref():
    if not os.path.isdir(os.path.join(REF, "multilap")):
        pytest.skip("reference package not available")
    if REF not in sys.path:
        sys.path.append(REF)
    import multilap
    return multilap


def test_box_map_and_label_sampling_equal_the_reference():
    ref = _ref()
    from multilap import datapipe as R

    from paper_2007_05239_b200 import datapipe as D
    rng = np.random.default_rng(5)
    for shape in ((700, 3), (300, 2), (50, 1)):
        X = rng.normal(0.3, 2.0, shape)
        X[:, 0] *= 7.0                                   # anisotropic ranges: one common factor
        xa, ia = R.scale_for_fastsum(X)
        xb, ib = D.scale_for_fastsum(X)
        assert np.array_equal(xa, xb) and ia.factor == ib.factor and np.array_equal(ia.midpoints, ib.midpoints)
        bm = D.BoxMap.fit(np.concatenate([rng.normal(size=(len(X), 2)), X], axis=1),
                          columns=range(2, 2 + shape[1]))
        assert np.array_equal(bm(X), xa)
    const = np.ones((10, 2))
    assert np.array_equal(R.scale_for_fastsum(const)[0], D.scale_for_fastsum(const)[0])
    for trial in range(12):
        truth = rng.integers(0, 4, size=int(rng.integers(20, 2000)))
        if len(np.unique(truth)) < 4:
            continue
        f = float(rng.uniform(0.001, 1.0))
        a, b = R.sample_labels(truth, f, seed=trial), D.sample_labels(truth, f, seed=trial)
        assert np.array_equal(a.F, b.F) and np.array_equal(a.fidelity, b.fidelity)
    with pytest.raises(D.ConfigError, match="class 1 absent"):
        D.sample_labels(np.array([0, 0, 2]), 0.5, 0)


def test_errors_derive_from_the_reference_classes_when_installed():
    """With multilap importable first, `except multilap.ConfigError` catches
    this backend's errors (fresh interpreter: the import order decides)."""
    _ref()
    import subprocess
    code = ("import sys; sys.path.insert(0, %r); sys.path.insert(0, %r); import multilap\n"
            "from paper_2007_05239_b200 import errors as e\n"
            "assert issubclass(e.ConfigError, multilap.errors.ConfigError)\n"
            "assert issubclass(e.ConvergenceError, multilap.errors.NumericalError)\n"
            "try:\n    raise e.NumericalError('x')\nexcept multilap.errors.MultilapError:\n    print('caught')\n"
            % (REF, os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    assert r.returncode == 0 and "caught" in r.stdout, r.stderr


def test_group_spec_errors_match_the_reference():
    _ref()
    from multilap import datapipe as R
    from multilap.kernels import KernelSpec as RK

    from paper_2007_05239_b200 import datapipe as D
    from paper_2007_05239_b200.kernels import KernelSpec as DK
    cases = [((), "fastsum-box"), ((0, 0), "fastsum-box"), ((0,), "bogus"), ((0, 1, 2, 3), "fastsum-box")]
    for cols, mode in cases:
        msgs = []
        for mod, K in ((R, RK), (D, DK)):
            try:
                mod.GroupSpec(cols, K("gaussian", 0.1), mode=mode)
            except Exception as e:
                msgs.append(str(e))
        assert len(msgs) == 2 and msgs[0] == msgs[1], (cols, mode, msgs)
    msgs = []
    for mod, K in ((R, RK), (D, DK)):
        try:
            mod.GroupingSpec((mod.GroupSpec((0, 1), K("gaussian", 0.1)), mod.GroupSpec((1, 2), K("gaussian", 0.1))))
        except Exception as e:
            msgs.append(str(e))
    assert msgs[0] == msgs[1]


def test_config_error_order_matches_the_reference():
    _ref()
    from multilap.config import merge_config as R

    from paper_2007_05239_b200.config import merge_config as D
    for bad in ({"power": {"bogus": 1}, "zzz": 1}, {"zzz": 1, "power": {"bogus": 1}},
                {"eig": {"k": 1, "kk": 2}}, {"fastsum": 3}):
        msgs = []
        for fn in (R, D):
            try:
                fn(bad)
            except Exception as e:
                msgs.append(str(e))
        assert len(msgs) == 2 and msgs[0] == msgs[1], (bad, msgs)


def test_bench_roofline_bookkeeping():
    import bench
    st = [{"layer": 0, "d": 3, "N": 64, "m": 5, "n": 1000, "spread_ms": 2.0, "reduce_ms": 0.1, "convolve_ms": 0.1,
           "gather_ms": 3.0, "stats": {"grid_cells": 100}},
          {"layer": 1, "d": 1, "N": 64, "m": 3, "n": 10 ** 7, "spread_ms": 1.0, "reduce_ms": 0.1,
           "convolve_ms": 0.1, "gather_ms": 1.5, "stats": {"grid_cells": 100}}]
    rows = bench.kernel_table(st, "none", 6548.5, 35.0)
    g3 = next(r for r in rows if r["kernel"] == "gather" and r["d"] == 3)
    assert g3["alg_bytes"] == (8 * 3 + 24) * 1000 and g3["alg_flops"] == 2 * 11 ** 3 * 1000
    roof = bench.roofline_of(rows, 6548.5, "measured", 35.0)
    assert roof["kernel"].startswith("gather (layer d=3") and roof["bound"] == "fp64"   # 55 flop/B > ridge
    assert abs(roof["frac"] - g3["fp64_frac"]) < 1e-15 and roof["hbm"]["unit"] == "GB/s"
    rows1 = bench.kernel_table(st[1:], "none", 6548.5, 35.0)
    roof1 = bench.roofline_of(rows1, 6548.5, "measured", 35.0)
    assert roof1["bound"] == "hbm" and roof1["unit"] == "GB/s"                        # d=1, m=3: 14 flop / 32 B
    assert bench.algorithmic_bytes(2) == 72 and bench.algorithmic_flops(3, 4) == 2916


def test_sharded_algebra_single_rank_matches_numpy():
    """ShardContext on CPU with no process group: CGS2 with the fused norm,
    PKSM on a dense SPD operator, thick-restart Lanczos on a diagonal."""
    import torch

    from paper_2007_05239_b200.krylov import power_fn
    from paper_2007_05239_b200.sharded import ShardContext, sharded_lanczos_fn, sharded_lanczos_largest_eigs
    rng = np.random.default_rng(2)
    n = 300
    ctx = ShardContext(None, n, 0, n, device=None)
    Q, _ = np.linalg.qr(rng.standard_normal((n, 6)))
    V = torch.from_numpy(np.ascontiguousarray(Q.T))
    w0 = rng.standard_normal(n)
    w = torch.from_numpy(w0.copy())
    buf = torch.empty(2 * 6 + 1, dtype=torch.float64)
    hh = ctx.cgs2(V, 6, w, buf)
    ref = w0 - Q @ (Q.T @ w0)
    ref = ref - Q @ (Q.T @ ref)
    assert np.allclose(w.numpy(), ref, atol=1e-13)
    assert abs(hh[12] - ref @ ref) <= 1e-12 * (ref @ ref)
    A = rng.standard_normal((n, n))
    A = A @ A.T / n + np.eye(n)
    v = rng.standard_normal(n)
    y = sharded_lanczos_fn(ctx, lambda x: torch.from_numpy(A @ x.numpy()), torch.from_numpy(v), power_fn(-1.0))
    assert np.linalg.norm(y.numpy() - np.linalg.solve(A, v)) <= 1e-7 * np.linalg.norm(np.linalg.solve(A, v))
    d = np.linspace(1.0, 2.0, n)
    res = sharded_lanczos_largest_eigs(ctx, lambda x: x * torch.from_numpy(d), 4, tol=1e-10)
    assert np.allclose(res.values, d[::-1][:4], rtol=1e-9)
