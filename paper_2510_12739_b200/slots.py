"""Seeded synthetic OFDM slots for the BASELINE configs (host-side input synthesis, numpy).

There is no public dataset for this path; seeded synthetic slots with BASELINE's
shapes and distributions stand in.  The pieces restate the reference's PHY helpers and extend them
where BASELINE asks for more than the snapshot implements:

* QAM: Gray map, even bits -> I, odd -> Q, unit energy (qam.cpp:10-52).
* Pilots: the fixed "PILOT"-seeded QPSK stream (pilots.cpp:13-31) on every `spacing`-th subcarrier,
  extended from one pilot symbol (PilotConfig, link_config.hpp:9-12) to the DM-RS symbols 2 and 11.
  The Rng restatement (splitmix64-seeded mt19937_64, rng.hpp:14-69) makes a one-symbol pattern
  bit-identical to the reference's (tests/test_slots.py).
* Channel: tapped delay line with an exponential power-delay profile whose RMS delay spread is solved
  by bisection (channel.cpp:37-50), per-tap Rayleigh processes as a 20-sinusoid Jakes sum, block
  fading per OFDM symbol, H[t,f] = sum_l a_l(t) exp(-j 2 pi f df tau_l) (channel.cpp:52-111).  The
  reference fixes 16 taps on the 1/(F df) grid; BASELINE needs 3 / 12 / 23 taps and RMS spreads the
  1/(F df) grid cannot reach with that many taps, so tap count and spacing are parameters here.
* y = h x + g z + n: AWGN at SNR ~ U[lo, hi] dB per slot; for config 3 a
  co-channel QPSK interferer z through an independent channel g at SIR ~ U[lo, hi] dB.

The generator is not on the timed path: bench.py builds one batch per run and reuses it.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from .graph import LinkSpec

_MASK64 = (1 << 64) - 1
_PILOT_SEED = 0x50494C4F54  # "PILOT", pilots.cpp:10


def _splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _MASK64
    return x ^ (x >> 31)


class Rng:
    """conetrx::Rng (rng.hpp:14-69): std::mt19937_64 seeded with splitmix64(seed)."""

    def __init__(self, seed: int):
        mt = [0] * 312
        mt[0] = _splitmix64(seed & _MASK64)
        for i in range(1, 312):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _MASK64
        self.mt, self.idx = mt, 312

    def next_u64(self) -> int:
        mt = self.mt
        if self.idx >= 312:
            for i in range(312):
                y = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                mt[i] = mt[(i + 156) % 312] ^ (y >> 1) ^ (0xB5026F5AA96619E9 if y & 1 else 0)
            self.idx = 0
        y = mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _MASK64

    def uniform(self) -> float:
        return (self.next_u64() >> 11) * 2.0 ** -53

    def bit(self) -> int:
        return self.next_u64() >> 63


def bits_per_symbol(order: int) -> int:
    if order not in (4, 16, 64):
        raise ValueError(f"modulation order must be 4, 16 or 64, got {order}")
    return {4: 2, 16: 4, 64: 6}[order]


def qam_map(bits: np.ndarray, order: int) -> np.ndarray:
    """Vectorised qam_map (qam.cpp:42-52): bits [..., b] -> complex [...]."""
    b = bits_per_symbol(order)
    half = b // 2
    bits = np.asarray(bits, np.float64)
    ib, qb = bits[..., 0::2], bits[..., 1::2]

    def axis(v):  # axis_level, qam.cpp:23-30
        s0 = 1.0 - 2.0 * v[..., 0]
        if half == 1:
            return s0
        s1 = 1.0 - 2.0 * v[..., 1]
        if half == 2:
            return s0 * (2.0 - s1)
        s2 = 1.0 - 2.0 * v[..., 2]
        return s0 * (4.0 - s1 * (2.0 - s2))

    nf = {4: np.sqrt(2.0), 16: np.sqrt(10.0), 64: np.sqrt(42.0)}[order]
    return (axis(ib) + 1j * axis(qb)) / nf


def pilot_pattern(T: int, F: int, symbols: Sequence[int] = (2, 11), spacing: int = 2):
    """pilots.cpp:13-31 generalised to several DM-RS symbols. Returns (mask uint8 [T,F], values complex128)."""
    if spacing < 1 or F < spacing:
        raise ValueError("pilot spacing must fit the subcarrier count")
    rng = Rng(_PILOT_SEED)
    mask = np.zeros((T, F), np.uint8)
    vals = np.zeros((T, F), np.complex128)
    for t in symbols:
        if not 0 <= t < T:
            raise ValueError("pilot symbol index out of range")
        for f in range(0, F, spacing):
            b = np.array([rng.bit(), rng.bit()], np.uint8)
            mask[t, f] = 1
            vals[t, f] = qam_map(b, 4)
    return mask, vals


def tap_powers(rms_delay_s: float, spacing_s: float, n_taps: int) -> np.ndarray:
    """tdl_tap_powers (channel.cpp:37-50): exponential PDP, decay bisected in log space to the RMS."""
    tau = np.arange(n_taps) * spacing_s

    def powers(beta):
        p = np.exp(-tau / beta)
        return p / p.sum()

    def rms(p):
        m1 = (p * tau).sum()
        v = (p * tau * tau).sum() - m1 * m1
        return np.sqrt(v) if v > 0 else 0.0

    lo, hi = np.log(1e-12), np.log(1.0)
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if rms(powers(np.exp(mid))) < rms_delay_s:
            lo = mid
        else:
            hi = mid
    return powers(np.exp(0.5 * (lo + hi)))


def tdl_response(rng: np.random.Generator, B: int, link: LinkSpec, n_sin: int = 20) -> np.ndarray:
    """Per-slot TDL/Jakes frequency response H [B,T,F,N] (channel.cpp:52-111, parameterised taps)."""
    T, F, N, L = link.T, link.F, link.N, link.n_taps
    spacing = link.tap_spacing_s or (1.0 / (F * link.scs_hz) if not link.rms_delay_s else link.rms_delay_s / 3.0)
    if link.rms_delay_s > 0:
        p = tap_powers(link.rms_delay_s, spacing, L)
    else:
        p = np.exp(-np.arange(L, dtype=np.float64))
        p /= p.sum()
    tau = np.arange(L) * spacing
    tsym = (1.0 + link.cp_fraction) / link.scs_hz
    fd = rng.uniform(0.0, link.doppler_max_hz, size=B) if link.doppler_max_hz > 0 else np.zeros(B)
    wd = 2 * np.pi * fd
    omega = wd[:, None, None, None] * np.cos(2 * np.pi * rng.uniform(size=(B, N, L, n_sin)))
    phase = 2 * np.pi * rng.uniform(size=(B, N, L, n_sin))
    time = np.arange(T) * tsym
    arg = omega[:, None] * time[None, :, None, None, None] + phase[:, None]          # [B,T,N,L,S]
    taps = np.exp(1j * arg).sum(-1) * (np.sqrt(p) / np.sqrt(n_sin))[None, None, None, :]  # [B,T,N,L]
    tw = np.exp(-2j * np.pi * np.arange(F)[:, None] * link.scs_hz * tau[None, :])      # [F,L]
    return np.einsum("btnl,fl->btfn", taps, tw)


@dataclass
class SlotBatch:
    y: np.ndarray        # complex64 [B,T,F,N] received grid
    bits: np.ndarray     # uint8 [B,T,F,b] transmitted bits (pilot REs: 0)
    data_mask: np.ndarray  # bool [T,F] data REs (pilots excluded)
    pilots: np.ndarray   # complex64 [T,F]
    pilot_mask: np.ndarray  # uint8 [T,F]
    snr_db: np.ndarray   # [B]
    h: np.ndarray        # complex64 [B,T,F,N] user channel


def generate(link: LinkSpec, B: int, seed: int) -> SlotBatch:
    rng = np.random.default_rng(seed)
    T, F, N = link.T, link.F, link.N
    nb = bits_per_symbol(link.mod_order)
    pmask, pvals = pilot_pattern(T, F, link.pilot_symbols, link.pilot_spacing)
    data = pmask == 0
    bits = rng.integers(0, 2, size=(B, T, F, nb), dtype=np.uint8)
    bits[:, ~data] = 0
    x = qam_map(bits, link.mod_order)
    x[:, ~data] = pvals[~data]
    h = tdl_response(rng, B, link)
    y = h * x[..., None]
    if link.sir_db is not None:
        g = tdl_response(rng, B, link)
        zb = rng.integers(0, 2, size=(B, T, F, 2), dtype=np.uint8)
        z = qam_map(zb, 4)
        sir = rng.uniform(*link.sir_db, size=B)
        y = y + g * (z * np.sqrt(10.0 ** (-sir / 10.0))[:, None, None])[..., None]
    snr = rng.uniform(*link.snr_db, size=B)
    sigma2 = 10.0 ** (-snr / 10.0)
    n = (rng.standard_normal((B, T, F, N)) + 1j * rng.standard_normal((B, T, F, N))) * np.sqrt(sigma2 / 2.0)[
        :, None, None, None]
    y = y + n
    return SlotBatch(y.astype(np.complex64), bits, data, pvals.astype(np.complex64), pmask, snr,
                     h.astype(np.complex64))


def hard_bits(llr: np.ndarray) -> np.ndarray:
    """Hard decision: positive LLR => bit 1."""
    return (llr > 0).astype(np.uint8)


def ber(llr: np.ndarray, batch: SlotBatch) -> float:
    """Uncoded BER on data REs only (pilots excluded)."""
    hb = hard_bits(llr)[:, batch.data_mask]
    tb = batch.bits[:, batch.data_mask]
    return float((hb != tb).mean())
