"""TEST INFRASTRUCTURE — CPU restatement of the classical baseline receiver (csrc/classic.cu;
SPEC.md:290-316 lmmse_equalize / maxlog_demap / classical_receiver): LMMSE combining and max-log
demapping by EXHAUSTIVE search over all constellation points (the SPEC's demapper oracle), in float64.
Only tests/ may use it, as the checker."""
from __future__ import annotations

import numpy as np


def constellation(order: int):
    """All points of the Gray map (qam.cpp:42-52) and their bit labels: (points [M], bits [M, b])."""
    from paper_2510_12739_b200 import slots
    b = slots.bits_per_symbol(order)
    labels = ((np.arange(order)[:, None] >> np.arange(b)[None, :]) & 1).astype(np.uint8)
    return slots.qam_map(labels, order), labels


def maxlog(z: np.ndarray, nu: np.ndarray, order: int) -> np.ndarray:
    """LLR_b = (min_{s:b=0}|z-s|^2 - min_{s:b=1}|z-s|^2) / nu, positive => bit 1; z, nu broadcast."""
    pts, lab = constellation(order)
    d = np.abs(z[..., None] - pts) ** 2                                     # [..., M]
    out = []
    for k in range(lab.shape[1]):
        d0 = np.where(lab[:, k] == 0, d, np.inf).min(-1)
        d1 = np.where(lab[:, k] == 1, d, np.inf).min(-1)
        out.append((d0 - d1) / nu)
    return np.stack(out, -1)


def lmmse_maxlog(y: np.ndarray, h: np.ndarray, noise_var: np.ndarray, order: int) -> np.ndarray:
    """y, h [B,T,F,N] complex; noise_var [B] -> LLRs [B,T,F,b]: z = h^H y / h^H h, nu = s2 / h^H h."""
    g = (np.abs(h) ** 2).sum(-1)
    num = (np.conj(h) * y).sum(-1)
    with np.errstate(divide="ignore", invalid="ignore"):
        z = np.where(g > 0, num / np.where(g > 0, g, 1), 0)
        nu = np.where(g > 0, noise_var[:, None, None] / np.where(g > 0, g, 1), np.inf)
    llr = maxlog(z, nu, order)
    llr[g == 0] = 0.0
    return llr


def ls_estimate(y: np.ndarray, pilots: np.ndarray, mask: np.ndarray) -> np.ndarray:
    """The featurizer's LS + interpolation channel estimate (oracle.featurize channels 6a+4, 6a+5)."""
    import oracle
    feat = oracle.featurize(y, pilots, mask)
    N = y.shape[-1]
    return np.stack([feat[..., 6 * a + 4] + 1j * feat[..., 6 * a + 5] for a in range(N)], -1)
