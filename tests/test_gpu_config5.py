"""BASELINE configs[4] (the matvec micro-benchmark): points uniform in the
0.21875-ball (the reference rejects radius 0.25), v ~ N(0,1),
x drawn before v from default_rng(0) (synth.config5_micro); the W v error
against exact summation on a 2,000-target sample (default_rng(1)), as
run_fastsum_bench reports it (runner.py:496-512).

Two statements per case:
  * parity: the GPU fastsum at the targets equals the reference algorithm's
    (the C restatement of its spread / gather + scipy FFT) to <= 1e-11, i.e.
    the GPU reproduces the reference's approximation, not just some
    approximation;
  * accuracy: the relative error vs exact summation (GPU direct sums at the
    targets) equals the reference algorithm's own error to 1e-6 relative
    and stays under the App. B.3 level for that (d, sigma, N, m) x 10.
"""

import numpy as np
import pytest

from oracle import c_oracle as co
from oracle import fastsum_oracle as fo

pytestmark = pytest.mark.gpu

# App. B.3 errors at n = 2e4 (d, sigma, N, m) -> level (order of magnitude)
B3 = {(1, 0.05, 64, 4): 2.4e-8, (1, 0.2, 32, 4): 5.2e-5, (2, 0.2, 32, 4): 4.0e-7, (2, 0.05, 64, 6): 7.8e-7,
      (2, 0.2, 64, 3): 4.3e-6, (3, 0.2, 32, 6): 1.1e-9, (3, 0.2, 64, 4): 6.3e-8, (3, 0.05, 64, 3): 1.0e-4,
      (3, 0.2, 16, 4): 2.4e-5, (1, 0.2, 64, 6): 5.5e-6}


def _case(n, d, sigma, N, m):
    import synth
    from paper_2007_05239_b200 import KernelSpec, bind_points, build_plan, fastsum_apply
    from paper_2007_05239_b200.direct import direct_at_targets
    x, v = synth.config5_micro(n, d, seed=0)
    targets = np.sort(np.random.default_rng(1).choice(n, size=2000, replace=False))
    kern = KernelSpec("gaussian", sigma)
    plan = build_plan(kern, d=d, N=N, m_nfft=m, p_nfft=8)
    fast = fastsum_apply(None, v, plan, binding=bind_points(plan, x))[targets]
    exact = direct_at_targets(x, v, kern, targets)
    op = fo.OraclePlan("gaussian", sigma, d, N, m, p=8)
    conv = fo.convolve_grid(op, co.spread(op, x, v[None, :])[0])
    ref = co.gather(op, x[targets], conv[None, :])[0] - v[targets]
    par = np.linalg.norm(fast - ref) / np.linalg.norm(ref)
    err = np.linalg.norm(fast - exact) / np.linalg.norm(exact)
    err_ref = np.linalg.norm(ref - exact) / np.linalg.norm(exact)
    print(f"n={n} d={d} sigma={sigma} N={N} m={m}: parity {par:.2e}, error vs direct {err:.3e} "
          f"(reference algorithm {err_ref:.3e})")
    return par, err, err_ref


@pytest.mark.parametrize("key", sorted(B3), ids=[f"d{k[0]}_s{k[1]}_N{k[2]}_m{k[3]}" for k in sorted(B3)])
def test_config5_error_vs_direct_n1e5(key):
    d, sigma, N, m = key
    par, err, err_ref = _case(100_000, d, sigma, N, m)
    assert par <= 1e-11
    assert abs(err - err_ref) <= 1e-6 * err_ref + 1e-13
    assert err <= 10 * B3[key]


@pytest.mark.parametrize("d", [1, 2, 3])
def test_config5_error_vs_direct_n1e7(d):
    """The 10^7-point end of the sweep (N=64, m=4, sigma=0.2)."""
    par, err, err_ref = _case(10_000_000, d, 0.2, 64, 4)
    assert par <= 1e-11
    assert abs(err - err_ref) <= 1e-6 * err_ref + 1e-13
    assert err <= 1e-4
