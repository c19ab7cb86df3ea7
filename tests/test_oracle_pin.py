"""The C restatement (oracle/oracle.c) is pinned bit-for-bit to the reference compiled in place
(oracle/_ref) and to the committed golden fixtures generated from it (tests/golden/make_golden.py),
plus the SPEC's known-answer cases for the hot-path kernels."""
import os

import numpy as np
import pytest

import oracle
from paper_2510_12739_b200 import graph as G

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = {"cfg1": (11, 72), "cfg2": (12, 20), "cfg4": (13, 16)}


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg4"])
def test_restatement_matches_golden_bitwise(oracle_lib, name):
    d = np.load(os.path.join(GOLD, "forward.npz"))
    g = G.CONFIGS[name].graph(seed=CASES[name][0])
    got = oracle.forward(g, d[f"{name}_x"])
    assert np.array_equal(got, d[f"{name}_llr"]), np.abs(got - d[f"{name}_llr"]).max()
    # forward_concurrent (network.hpp:186-212) computes the same nodes: identical result
    assert np.array_equal(d[f"{name}_llr_concurrent"], d[f"{name}_llr"])


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg4"])
def test_restatement_matches_reference_live(ref, name):
    g = G.CONFIGS[name].graph(seed=5)
    x = np.random.default_rng(9).standard_normal((2, 14, 24, g.in_channels)).astype(np.float32)
    assert np.array_equal(oracle.forward(g, x), oracle.RefNet.from_graph(g).forward(x))


def test_fusion_identity_golden(oracle_lib):
    """supports forced to ones under mul fusion == build_reference_main."""
    d = np.load(os.path.join(GOLD, "forward.npz"))
    np.testing.assert_allclose(d["fusion_identity_llr"], d["fusion_identity_main_llr"], rtol=1e-6, atol=1e-6)


def _one_conv(kh, cin, cout, bias):
    g = G.Graph()
    x = g.add_input(cin)
    g.set_output(g.add_conv(x, "c", kh, cin, cout, bias))
    return g


def test_conv_scalar_affine_kat(oracle_lib):
    g = _one_conv(1, 1, 1, True)
    g.params[0].value[:] = 2.0
    g.params[1].value[:] = 1.0
    y = oracle.forward(g, np.full((1, 1, 1, 1), 5.0, np.float32))
    assert y.ravel()[0] == 11.0


def test_conv_identity_kernel_kat(oracle_lib):
    g = _one_conv(3, 1, 1, False)
    w = np.zeros((3, 3, 1, 1), np.float32)
    w[1, 1] = 1.0
    g.params[0].value = w
    x = np.ones((1, 3, 3, 1), np.float32)
    assert np.array_equal(oracle.forward(g, x), x)


def test_conv_brute_force_double(oracle_lib):
    """six-nested-loop oracle; the float restatement agrees to float rounding."""
    rng = np.random.default_rng(0)
    x = rng.standard_normal((1, 4, 4, 2)).astype(np.float32)
    w = rng.standard_normal((3, 3, 2, 3)).astype(np.float32)
    g = _one_conv(3, 2, 3, False)
    g.params[0].value = w
    y = oracle.forward(g, x)
    ref = np.zeros((1, 4, 4, 3))
    for t in range(4):
        for f in range(4):
            for dt in range(3):
                for df in range(3):
                    ti, fi = t + dt - 1, f + df - 1
                    if 0 <= ti < 4 and 0 <= fi < 4:
                        ref[0, t, f] += x[0, ti, fi].astype(np.float64) @ w[dt, df].astype(np.float64)
    np.testing.assert_allclose(y, ref, rtol=1e-5, atol=1e-5)


def test_relu_bn_elementwise_kats(oracle_lib):
    # relu [-1,0,2] -> [0,0,2]
    g = G.Graph()
    x = g.add_input(1)
    g.set_output(g.add_relu(x))
    assert oracle.forward(g, np.array([-1, 0, 2], np.float32).reshape(1, 1, 3, 1)).ravel().tolist() == [0, 0, 2]
    # eval BN with statistics of {1,3}: (x - 2)/1 -> {-1, +1} (eps -> 0 tolerance)
    g = G.Graph()
    x = g.add_input(1)
    g.set_output(g.add_norm(x, "bn", "n", 1))
    g.params[2].value[:] = 2.0
    g.params[3].value[:] = 1.0
    g.bn_ready = [1]
    y = oracle.forward(g, np.array([1, 3], np.float32).reshape(1, 1, 2, 1)).ravel()
    np.testing.assert_allclose(y, [-1, 1], rtol=1e-5)
    # mul(x, 1) = x and add(x, 0) = x bitwise
    rng = np.random.default_rng(3)
    a = rng.standard_normal((1, 2, 3, 4)).astype(np.float32)
    for op, fill in ((G.OP_MUL, 1.0), (G.OP_ADD, 0.0)):
        g = G.Graph()
        x = g.add_input(4)
        c = g.add_conv(x, "k", 1, 4, 4, True)
        g.set_output(g.add_binary(op, x, c))
        g.params[0].value[:] = 0.0
        g.params[1].value[:] = fill
        assert np.array_equal(oracle.forward(g, a), a)


def test_bn_not_ready_is_runtime_error(oracle_lib):
    g = G.CONFIGS["cfg2"].graph_fn()  # BNs never marked ready
    with pytest.raises(oracle.RefError) as e:
        oracle.forward(g, np.zeros((1, 14, 4, 12), np.float32))
    assert e.value.code == 2 and "eval mode" in str(e.value)


def test_channel_mismatch_is_invalid_argument(oracle_lib):
    g = G.CONFIGS["cfg2"].graph()
    with pytest.raises(oracle.RefError) as e:
        oracle.forward(g, np.zeros((1, 14, 4, 10), np.float32))
    assert e.value.code == 1 and "expects 12 input channels" in str(e.value)


def test_dilation_one_is_reference_conv(ref):
    """The dilation extension (config 3) reduces to the reference conv2d at dilation 1."""
    g = G.CONFIGS["cfg2"].graph(seed=2)
    x = np.random.default_rng(4).standard_normal((1, 14, 20, 12)).astype(np.float32)
    assert np.array_equal(oracle.forward(g, x), oracle.RefNet.from_graph(g).forward(x))


def test_dilated_conv_matches_numpy(oracle_lib):
    rng = np.random.default_rng(1)
    x = rng.standard_normal((1, 5, 9, 2)).astype(np.float32)
    w = rng.standard_normal((3, 3, 2, 2)).astype(np.float32)
    g = G.Graph()
    i = g.add_input(2)
    g.set_output(g.add_conv(i, "c", 3, 2, 2, False, dilation_f=2))
    g.params[0].value = w
    y = oracle.forward(g, x)
    ref = np.zeros((1, 5, 9, 2))
    for t in range(5):
        for f in range(9):
            for dt in range(3):
                for df in range(3):
                    ti, fi = t + dt - 1, f + 2 * (df - 1)
                    if 0 <= ti < 5 and 0 <= fi < 9:
                        ref[0, t, f] += x[0, ti, fi] @ w[dt, df]
    np.testing.assert_allclose(y, ref, rtol=1e-5, atol=1e-5)
