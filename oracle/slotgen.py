"""TEST INFRASTRUCTURE — CPU restatement of the on-GPU synthetic-slot generator and BER count
(paper_2510_12739_b200/csrc/slotgen.cu).  Only tests/ may use it, as the checker.

The algorithm is the reference's slot model (SPEC.md:212-220 `generate_tti`; QAM qam.cpp:10-52; TDL
with exponential PDP channel.cpp:37-111; hard decisions / BER SPEC.md:467-475, :498) with a
counter-based random source so that every random draw is addressable in parallel:

  Philox4x32-10 (Salmon et al., SC'11 — the published algorithm, restated here in numpy), key =
  (lo32(seed), hi32(seed)), counter = (index, purpose, lo32(slot), hi32(slot)).

  purpose 1 (slot)   index 0: u0 -> SNR, u1 -> Doppler, u2 -> SIR
  purpose 2 (bits)   index t*F + f: bits 0..b-1 of word 0 are the RE's bits (even -> I, odd -> Q)
  purpose 3/4 (Jakes, user / interferer channel) index (n*L + l)*S + s: u0 -> arrival angle, u1 -> phase
  purpose 5 (noise)  index (t*F + f)*N + n: Box-Muller of words 0, 1
  purpose 6 (interferer QPSK bits) index t*F + f: bits 0, 1 of word 0
  uniform(w) = (w >> 8) * 2^-24;   Box-Muller: r = sqrt(-2 ln(((w0 >> 8) + 1) 2^-24)), th = 2 pi uniform(w1)

Everything is float64 here; the GPU computes in fp32 (tests compare bits exactly, y with a tolerance).
"""
from __future__ import annotations

import numpy as np

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
P_SLOT, P_BITS, P_JAKES, P_JAKES_I, P_NOISE, P_IBITS = 1, 2, 3, 4, 5, 6
N_SIN = 20


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 over uint32 arrays (broadcast); returns 4 uint32 arrays."""
    c = [np.asarray(v, np.uint64) & 0xFFFFFFFF for v in (c0, c1, c2, c3)]
    k0 = np.uint64(k0 & 0xFFFFFFFF)
    k1 = np.uint64(k1 & 0xFFFFFFFF)
    c = list(np.broadcast_arrays(*c))
    c = [v.copy() for v in c]
    mask = np.uint64(0xFFFFFFFF)
    for r in range(10):
        p0 = np.uint64(M0) * c[0]
        p1 = np.uint64(M1) * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & mask
        hi1, lo1 = p1 >> np.uint64(32), p1 & mask
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
        k0 = (k0 + np.uint64(W0)) & mask
        k1 = (k1 + np.uint64(W1)) & mask
    return [v.astype(np.uint32) for v in c]


def uniform(w):
    return (np.asarray(w, np.uint64) >> np.uint64(8)).astype(np.float64) * 2.0 ** -24


def _draw(seed, slot, purpose, index):
    s = np.uint64(slot)
    return philox4x32_10(index, purpose, int(s) & 0xFFFFFFFF, (int(s) >> 32) & 0xFFFFFFFF, seed & 0xFFFFFFFF,
                         (seed >> 32) & 0xFFFFFFFF)


def tap_profile(link):
    """Tap powers and delays exactly as slots.tdl_response chooses them."""
    from paper_2510_12739_b200 import slots
    L, F = link.n_taps, link.F
    spacing = link.tap_spacing_s or (1.0 / (F * link.scs_hz) if not link.rms_delay_s else link.rms_delay_s / 3.0)
    if link.rms_delay_s > 0:
        p = slots.tap_powers(link.rms_delay_s, spacing, L)
    else:
        p = np.exp(-np.arange(L, dtype=np.float64))
        p /= p.sum()
    return p, np.arange(L) * spacing


def _channel(seed, slot, purpose, link, fd, p, tau):
    T, F, N, L = link.T, link.F, link.N, link.n_taps
    idx = np.arange(N * L * N_SIN, dtype=np.uint64)
    w = _draw(seed, slot, purpose, idx)
    ang = uniform(w[0]).reshape(N, L, N_SIN)
    ph = uniform(w[1]).reshape(N, L, N_SIN)
    omega = 2 * np.pi * fd * np.cos(2 * np.pi * ang)
    phase = 2 * np.pi * ph
    tsym = (1.0 + link.cp_fraction) / link.scs_hz
    t = np.arange(T) * tsym
    arg = omega[None] * t[:, None, None, None] + phase[None]                       # [T,N,L,S]
    taps = np.exp(1j * arg).sum(-1) * np.sqrt(p / N_SIN)[None, None, :]          # [T,N,L]
    frac = np.mod(np.arange(F)[:, None] * link.scs_hz * tau[None, :], 1.0)        # [F,L]
    tw = np.exp(-2j * np.pi * frac)
    return np.einsum("tnl,fl->tfn", taps, tw)                                     # [T,F,N]


def _qam(bits, order):
    from paper_2510_12739_b200 import slots
    return slots.qam_map(bits, order)


def generate(link, B: int, seed: int, slot0: int = 0, with_h: bool = False):
    """-> (y complex128 [B,T,F,N], bits uint8 [B,T,F,b], (h [B,T,F,N]))."""
    from paper_2510_12739_b200 import slots
    T, F, N = link.T, link.F, link.N
    nb = link.bits
    pmask, pvals = slots.pilot_pattern(T, F, link.pilot_symbols, link.pilot_spacing)
    p, tau = tap_profile(link)
    re = np.arange(T * F, dtype=np.uint64)
    ys, bs, hs = [], [], []
    for b in range(B):
        slot = slot0 + b
        ws = _draw(seed, slot, P_SLOT, np.zeros(1, np.uint64))
        snr = link.snr_db[0] + (link.snr_db[1] - link.snr_db[0]) * uniform(ws[0])[0]
        fd = link.doppler_max_hz * uniform(ws[1])[0] if link.doppler_max_hz > 0 else 0.0
        wb = _draw(seed, slot, P_BITS, re)[0]
        bits = ((wb[:, None] >> np.arange(nb, dtype=np.uint32)[None, :]) & 1).astype(np.uint8).reshape(T, F, nb)
        bits[pmask != 0] = 0
        x = _qam(bits, link.mod_order)
        x[pmask != 0] = pvals[pmask != 0]
        h = _channel(seed, slot, P_JAKES, link, fd, p, tau)
        y = h * x[..., None]
        if link.sir_db is not None:
            sir = link.sir_db[0] + (link.sir_db[1] - link.sir_db[0]) * uniform(ws[2])[0]
            g = _channel(seed, slot, P_JAKES_I, link, fd, p, tau)
            wi = _draw(seed, slot, P_IBITS, re)[0]
            zb = ((wi[:, None] >> np.arange(2, dtype=np.uint32)[None, :]) & 1).astype(np.uint8).reshape(T, F, 2)
            z = _qam(zb, 4) * np.sqrt(10.0 ** (-sir / 10.0))
            y = y + g * z[..., None]
        sigma2 = 10.0 ** (-snr / 10.0)
        wn = _draw(seed, slot, P_NOISE, np.arange(T * F * N, dtype=np.uint64))
        r = np.sqrt(-2.0 * np.log(((np.asarray(wn[0], np.uint64) >> np.uint64(8)).astype(np.float64) + 1.0) * 2.0 ** -24))
        th = 2 * np.pi * uniform(wn[1])
        n = (r * np.cos(th) + 1j * r * np.sin(th)).reshape(T, F, N) * np.sqrt(sigma2 / 2.0)
        ys.append(y + n)
        bs.append(bits)
        hs.append(h)
    out = (np.stack(ys), np.stack(bs))
    return out + (np.stack(hs),) if with_h else out


def bit_errors(llr: np.ndarray, bits: np.ndarray, data_mask: np.ndarray) -> np.ndarray:
    """Per-slot count of hard-decision errors (LLR > 0 => 1) over data REs."""
    hb = (llr > 0).astype(np.uint8)
    err = (hb != bits) & data_mask[None, :, :, None].astype(bool)
    return err.reshape(err.shape[0], -1).sum(1).astype(np.int64)
