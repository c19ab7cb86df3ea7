"""Classical baseline receiver (csrc/classic.cu: LMMSE + max-log) against the exhaustive-search oracle
(oracle/classic.py) and the SPEC's analytic checks (acceptance criteria)."""
import dataclasses
import math

import numpy as np
import pytest

import oracle.classic as K
import oracle.slotgen as S
from paper_2510_12739_b200 import graph as G
from paper_2510_12739_b200 import slots


def test_maxlog_oracle_examples():
    # x_hat = 0 for QPSK -> all LLRs 0 (equidistant); on the (1,1)-bit point -> both large positive
    assert np.all(K.maxlog(np.array([0j]), np.array([0.1]), 4) == 0)
    p = slots.qam_map(np.array([1, 1], np.uint8), 4)
    llr = K.maxlog(np.array([p]), np.array([0.01]), 4)
    assert np.all(llr > 100)
    # separable per-axis minimum == exhaustive 2-D minimum (what the GPU kernel relies on)
    rng = np.random.default_rng(0)
    for order in (4, 16, 64):
        z = rng.standard_normal(500) + 1j * rng.standard_normal(500)
        pts, lab = K.constellation(order)
        b = lab.shape[1]
        levels = np.unique(pts.real)
        for k in range(b):
            axis = z.real if k % 2 == 0 else z.imag
            ax_pts = pts.real if k % 2 == 0 else pts.imag
            d0 = np.array([min((a - v) ** 2 for v, l in zip(ax_pts, lab[:, k]) if l == 0) for a in axis])
            d1 = np.array([min((a - v) ** 2 for v, l in zip(ax_pts, lab[:, k]) if l == 1) for a in axis])
            np.testing.assert_allclose(K.maxlog(z, np.ones(500), order)[:, k], d0 - d1, rtol=1e-12, atol=1e-12)
        assert len(levels) == int(math.isqrt(order))


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_slot_noise_var_matches_restatement(name):
    from paper_2510_12739_b200 import plan as P
    link = G.CONFIGS[name].link
    got = P.slot_noise_var(link, 6, 31, slot0=4)
    want = []
    for b in range(6):
        ws = S._draw(31, 4 + b, S.P_SLOT, np.zeros(1, np.uint64))
        snr = link.snr_db[0] + (link.snr_db[1] - link.snr_db[0]) * S.uniform(ws[0])[0]
        v = 10 ** (-snr / 10)
        if link.sir_db is not None:
            sir = link.sir_db[0] + (link.sir_db[1] - link.sir_db[0]) * S.uniform(ws[2])[0]
            v += 10 ** (-sir / 10)
        want.append(v)
    np.testing.assert_allclose(got, want, rtol=2e-6)


def _q(x):
    return 0.5 * math.erfc(x / math.sqrt(2))


@pytest.mark.gpu
@pytest.mark.parametrize("order", [4, 16, 64])
def test_demapper_equals_exhaustive_search(order):
    """SPEC acceptance 'Demapper oracle': max-log LLRs equal the exhaustive constellation search over 1e4
    random inputs (fp32 kernel vs float64 oracle)."""
    import torch
    from paper_2510_12739_b200 import plan as P
    rng = np.random.default_rng(order)
    B, T, F, N = 2, 10, 500, 1
    y = ((rng.standard_normal((B, T, F, N)) + 1j * rng.standard_normal((B, T, F, N))) * 0.8).astype(np.complex64)
    h = np.ones_like(y)
    nv = np.array([0.05, 0.3], np.float32)
    p = P.Plan(G.CONFIGS["cfg1"].graph(), "fp32")
    got = P.classical_receive_device(p, torch.from_numpy(y).cuda(), nv, order, h=torch.from_numpy(h).cuda())
    want = K.lmmse_maxlog(y.astype(np.complex128), h.astype(np.complex128), nv.astype(np.float64), order)
    np.testing.assert_allclose(got.cpu().numpy(), want, rtol=1e-4, atol=1e-3)


@pytest.mark.gpu
def test_perfect_and_ls_lmmse_match_oracle_on_generated_slots():
    import torch
    from paper_2510_12739_b200 import plan as P
    link = dataclasses.replace(G.CONFIGS["cfg2"].link, F=96)
    B = 3
    y, bits, h = P.generate_slots_device(link, B, 5, with_h=True)
    nv = P.slot_noise_var(link, B, 5)
    pmask, pvals = slots.pilot_pattern(link.T, link.F, link.pilot_symbols, link.pilot_spacing)
    p = P.Plan(G.CONFIGS["cfg2"].graph(), "bf16")
    p.set_pilots(pvals.astype(np.complex64), pmask)
    yn, hn = y.cpu().numpy().astype(np.complex128), h.cpu().numpy().astype(np.complex128)
    perfect = P.classical_receive_device(p, y, nv, link.mod_order, h=h).cpu().numpy()
    np.testing.assert_allclose(perfect, K.lmmse_maxlog(yn, hn, nv.astype(np.float64), link.mod_order),
                               rtol=2e-4, atol=2e-3)
    ls = P.classical_receive_device(p, y, nv, link.mod_order).cpu().numpy()
    h_ls = K.ls_estimate(y.cpu().numpy(), pvals.astype(np.complex64), pmask).astype(np.complex128)
    np.testing.assert_allclose(ls, K.lmmse_maxlog(yn, h_ls, nv.astype(np.float64), link.mod_order),
                               rtol=2e-4, atol=2e-3)
    # all-zero channel at an RE -> LLRs 0
    h0 = h.clone()
    h0[0, 0, 0] = 0
    z = P.classical_receive_device(p, y, nv, link.mod_order, h=h0).cpu().numpy()
    assert np.all(z[0, 0, 0] == 0)


@pytest.mark.gpu
def test_awgn_qpsk_ber_matches_q_function():
    """SPEC acceptance 'Classical-chain oracle': perfect-CSI LMMSE on flat AWGN, QPSK, N=1 -> per-bit
    error rate Q(sqrt(Es/N0)) (= Q(sqrt(2 Eb/N0))) within 3 sigma, >= 2e5 bits per point."""
    import torch
    from paper_2510_12739_b200 import plan as P
    rng = np.random.default_rng(11)
    p = P.Plan(G.CONFIGS["cfg1"].graph(), "fp32")
    B, T, F = 8, 14, 1000  # 112k symbols = 224k bits per SNR point
    for snr_db in (0, 2, 4, 6, 8):
        bits = rng.integers(0, 2, (B, T, F, 2)).astype(np.uint8)
        x = slots.qam_map(bits, 4)
        s2 = 10 ** (-snr_db / 10)
        n = (rng.standard_normal(x.shape) + 1j * rng.standard_normal(x.shape)) * math.sqrt(s2 / 2)
        y = (x + n)[..., None].astype(np.complex64)
        h = np.ones_like(y)
        llr = P.classical_receive_device(p, torch.from_numpy(y).cuda(), np.full(B, s2, np.float32), 4,
                                         h=torch.from_numpy(h).cuda()).cpu().numpy()
        ber = float(((llr > 0).astype(np.uint8) != bits).mean())
        pth = _q(math.sqrt(10 ** (snr_db / 10)))
        sigma = math.sqrt(pth * (1 - pth) / bits.size)
        assert abs(ber - pth) <= 3 * sigma + 1e-12, (snr_db, ber, pth, sigma)


@pytest.mark.gpu
def test_perfect_csi_not_worse_than_ls():
    import torch
    from paper_2510_12739_b200 import plan as P
    link = dataclasses.replace(G.CONFIGS["cfg2"].link, F=612, snr_db=(8.0, 12.0))
    B = 16
    y, bits, h = P.generate_slots_device(link, B, 9, with_h=True)
    nv = P.slot_noise_var(link, B, 9)
    pmask, pvals = slots.pilot_pattern(link.T, link.F, link.pilot_symbols, link.pilot_spacing)
    p = P.Plan(G.CONFIGS["cfg2"].graph(), "bf16")
    p.set_pilots(pvals.astype(np.complex64), pmask)
    data = torch.from_numpy(pmask == 0)
    e_perf = int(P.count_bit_errors(P.classical_receive_device(p, y, nv, 16, h=h), bits, data).sum())
    e_ls = int(P.count_bit_errors(P.classical_receive_device(p, y, nv, 16), bits, data).sum())
    assert e_perf <= e_ls
