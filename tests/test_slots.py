"""Synthetic-slot pieces pinned to the reference PHY helpers (golden fixtures from oracle/_ref)."""
import os

import numpy as np
import pytest

import oracle
from paper_2510_12739_b200 import graph as G, slots

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_rng_matches_reference_golden():
    d = np.load(os.path.join(GOLD, "phy.npz"))
    r = slots.Rng(12345)
    assert [r.next_u64() for _ in range(16)] == [int(v) for v in d["rng_u64_seed12345"]]
    r = slots.Rng(7)
    assert np.array_equal([r.uniform() for _ in range(16)], d["rng_uniform_seed7"])


def test_qam_matches_reference_golden():
    d = np.load(os.path.join(GOLD, "phy.npz"))
    for order in (4, 16, 64):
        nb = slots.bits_per_symbol(order)
        labels = np.arange(order)
        bits = ((labels[:, None] >> (nb - 1 - np.arange(nb))[None, :]) & 1).astype(np.uint8)
        pts = slots.qam_map(bits, order)
        np.testing.assert_array_equal(np.stack([pts.real, pts.imag], -1), d[f"qam{order}"])
        assert abs(np.mean(np.abs(pts) ** 2) - 1.0) < 1e-12
    assert slots.qam_map(np.array([0, 0]), 4) == (1 + 1j) / np.sqrt(2)


def test_pilot_pattern_matches_reference_golden():
    d = np.load(os.path.join(GOLD, "phy.npz"))
    for F in (64, 72, 612):
        m, v = slots.pilot_pattern(14, F, (2,), 2)
        assert np.array_equal(m, d[f"pilots_T14_F{F}_mask"])
        np.testing.assert_array_equal(np.stack([v.real, v.imag], -1), d[f"pilots_T14_F{F}_values"])
    assert slots.pilot_pattern(14, 64, (2,), 2)[0].sum() == 32


def test_two_symbol_pilots_match_oracle(oracle_lib):
    m, v = slots.pilot_pattern(14, 612, (2, 11), 2)
    m2, v2 = oracle.pilot_pattern(14, 612, (2, 11), 2)
    assert np.array_equal(m, m2) and np.array_equal(v, v2)


def test_tap_powers_match_reference_golden():
    d = np.load(os.path.join(GOLD, "phy.npz"))
    np.testing.assert_allclose(slots.tap_powers(300e-9, 1.0 / (64 * 30e3), 16), d["tap_powers_300ns_F64"],
                               rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_generator_statistics(name):
    link = G.CONFIGS[name].link
    b = slots.generate(link, 64, 3)
    assert b.y.shape == (64, 14, link.F, link.N)
    assert abs(np.mean(np.abs(b.h) ** 2) - 1.0) < 0.2  # unit average channel power
    assert b.data_mask.sum() == 14 * link.F - b.pilot_mask.sum()
    if link.doppler_max_hz == 0:
        assert np.abs(b.h[:, 0] - b.h[:, 13]).max() < 1e-5  # static channel


def test_featurize_oracle_kat(oracle_lib):
    """Noiseless flat channel h=1: LS estimate recovers 1 everywhere; features carry y and pilots."""
    T, F = 14, 16
    mask, pv = slots.pilot_pattern(T, F, (2, 11), 2)
    y = np.ones((1, T, F, 1), np.complex64)
    y[0, mask == 1, 0] = pv[mask == 1]
    feat = oracle.featurize(y, pv.astype(np.complex64), mask)
    np.testing.assert_allclose(feat[..., 4], 1.0, atol=1e-6)
    np.testing.assert_allclose(feat[..., 5], 0.0, atol=1e-6)
    np.testing.assert_array_equal(feat[0, :, :, 2], pv.real.astype(np.float32))


def _linear_channel_slot(T, F, N, a, bf, ct, syms=(2, 11), spacing=2, seed=0):
    """Noiseless slot through h[t, f, n] = a_n + bf_n * f + ct_n * t (complex), random QPSK data."""
    rng = np.random.default_rng(seed)
    mask, pv = slots.pilot_pattern(T, F, syms, spacing)
    x = (rng.choice([-1.0, 1.0], (T, F)) + 1j * rng.choice([-1.0, 1.0], (T, F))) / np.sqrt(2)
    x[mask == 1] = pv[mask == 1]
    t = np.arange(T)[:, None, None]
    f = np.arange(F)[None, :, None]
    h = np.asarray(a)[None, None, :] + np.asarray(bf)[None, None, :] * f + np.asarray(ct)[None, None, :] * t
    y = (h * x[:, :, None])[None].astype(np.complex64)
    return y, h, mask, pv


def _hhat(feat, N):
    return feat[..., 4::6][..., :N] + 1j * feat[..., 5::6][..., :N]


@pytest.mark.parametrize("N", [1, 2])
def test_featurize_kat_linear_in_frequency(oracle_lib, N):
    """SPEC.md:277 (noiseless -> h_hat at pilots equals the true h) and SPEC.md:287 (channel linear in
    the subcarrier index, pilots every 2nd subcarrier, noiseless -> exact recovery at interior REs;
    nearest pilot beyond the edge pilots)."""
    T, F = 14, 24
    y, h, mask, pv = _linear_channel_slot(T, F, N, [0.3 + 0.2j, -0.5 + 0.1j][:N], [0.05 - 0.02j, 0.01 + 0.03j][:N],
                                          [0, 0][:N])
    hh = _hhat(oracle.featurize(y, pv.astype(np.complex64), mask)[0], N)
    for t in (2, 11):
        pf = np.nonzero(mask[t])[0]
        np.testing.assert_allclose(hh[t, pf], h[t, pf], atol=2e-6)                     # at pilots
        interior = np.arange(pf[0], pf[-1] + 1)
        np.testing.assert_allclose(hh[t, interior], h[t, interior], atol=2e-6)         # interior: exact
        np.testing.assert_allclose(hh[t, pf[-1] + 1:], np.broadcast_to(h[t, pf[-1]], hh[t, pf[-1] + 1:].shape),
                                   atol=2e-6)                                           # edge: nearest
    # static in time: every symbol carries the pilot symbols' estimate
    np.testing.assert_allclose(hh, np.broadcast_to(hh[2], hh.shape), atol=2e-6)


def test_featurize_kat_linear_in_time(oracle_lib):
    """Two DM-RS symbols (2 and 11): the estimate is linear in T between them (exact for a channel
    linear in t) and nearest outside (symbols 0-1 take symbol 2's estimate, 12-13 symbol 11's)."""
    T, F, N = 14, 20, 1
    y, h, mask, pv = _linear_channel_slot(T, F, N, [0.4 - 0.3j], [0], [0.02 + 0.05j])
    hh = _hhat(oracle.featurize(y, pv.astype(np.complex64), mask)[0], N)
    for t in range(T):
        want = h[min(max(t, 2), 11)]
        np.testing.assert_allclose(hh[t], want, atol=2e-6, err_msg=f"symbol {t}")


def test_featurize_kat_bilinear_and_feature_layout(oracle_lib):
    """h linear in both f and t: exact inside the pilot hull; features 6a+k = [Re y, Im y, Re x_p, Im x_p,
    Re h_hat, Im h_hat] per antenna, pilot channels zero off-pilot."""
    T, F, N = 14, 30, 2
    y, h, mask, pv = _linear_channel_slot(T, F, N, [1.0, 0.2 + 0.7j], [0.03j, -0.02], [0.01, 0.04 - 0.01j])
    feat = oracle.featurize(y, pv.astype(np.complex64), mask)[0]
    hh = _hhat(feat, N)
    pf = np.nonzero(mask[2])[0]
    inner = np.ix_(np.arange(2, 12), np.arange(pf[0], pf[-1] + 1))
    np.testing.assert_allclose(hh[inner], h[inner], atol=3e-6)
    for a in range(N):
        np.testing.assert_array_equal(feat[..., 6 * a], y[0, ..., a].real)
        np.testing.assert_array_equal(feat[..., 6 * a + 1], y[0, ..., a].imag)
        np.testing.assert_array_equal(feat[..., 6 * a + 2], np.where(mask == 1, pv.real, 0).astype(np.float32))
        np.testing.assert_array_equal(feat[..., 6 * a + 3], np.where(mask == 1, pv.imag, 0).astype(np.float32))
