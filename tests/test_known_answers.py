"""Hand-computed known answers from the reference's own tests:
P3 Laplacian (test_graphs.py:24-33), shifted apply (:36-44), single-layer
power-mean spectrum (test_powermean.py:40-47), flat kernel -> delta
(test_fastsum.py:114-118), well force T(0.75, 0.25) (test_allencahn.py:96-100).
The graph ones run on the device (layers are device-resident)."""

import math

import numpy as np
import pytest
from numpy.testing import assert_allclose

P3 = np.array([[0.0, 1.0, 0.0], [1.0, 0.0, 1.0], [0.0, 1.0, 0.0]])


def _p3_graph():
    from paper_2007_05239_b200 import DenseWeights, MultilayerGraph, build_layer
    return MultilayerGraph((build_layer(DenseWeights(P3)),))


@pytest.mark.gpu
def test_p3_degrees_and_middle_basis_vector():
    from paper_2007_05239_b200 import apply_sym_laplacian
    G = _p3_graph()
    assert_allclose(G.layers[0].degrees, [1.0, 2.0, 1.0])
    s = 1.0 / math.sqrt(2.0)
    out = apply_sym_laplacian(G.layers[0], np.array([0.0, 1.0, 0.0]))
    assert_allclose(out, [-s, 1.0, -s], atol=1e-15)
    # sqrt(degrees) spans the null space of L_sym
    assert_allclose(apply_sym_laplacian(G.layers[0], np.sqrt([1.0, 2.0, 1.0])), 0.0, atol=1e-14)


@pytest.mark.gpu
def test_shifted_apply_adds_delta_times_v():
    from paper_2007_05239_b200 import ConfigError, apply_sym_laplacian, with_shift
    layer = _p3_graph().layers[0]
    v = np.random.default_rng(0).standard_normal(3)
    assert_allclose(apply_sym_laplacian(with_shift(layer, 0.7), v),
                    apply_sym_laplacian(layer, v) + 0.7 * v, rtol=1e-14)
    with pytest.raises(ConfigError):
        with_shift(layer, -0.1)


@pytest.mark.gpu
def test_single_layer_negative_power_spectrum():
    from paper_2007_05239_b200 import PowerMeanConfig, power_mean_eigs
    delta = math.log(3.0)  # log(1 + |p|) at p = -2
    basis = power_mean_eigs(_p3_graph(), PowerMeanConfig(p=-2.0), k=2, seed=0)
    assert_allclose(basis.values, [delta, 1.0 + delta], atol=1e-9)
    assert basis.k == 2 and basis.values[0] <= basis.values[1]


def test_flat_kernel_coefficients_are_a_delta():
    from paper_2007_05239_b200 import KernelSpec
    from paper_2007_05239_b200.fastsum import kernel_fourier_coefficients
    c = kernel_fourier_coefficients(KernelSpec("gaussian", 1e8), 1, 32, 1 / 16, 5)
    assert_allclose(c[0], 1.0, rtol=1e-12)
    assert np.max(np.abs(c[1:])) < 1e-12


def test_well_force_hand_value():
    from paper_2007_05239_b200 import nonlinearity_T
    assert_allclose(nonlinearity_T(np.array([[0.75, 0.25]])), [[-0.09375, 0.09375]], atol=1e-15)
