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
