"""GPU featurizer parity (csrc/featurize.cu) beyond the whole-network checks:

  * the SPEC known-answer tests (SPEC.md:277 LS at pilots exact; SPEC.md:287 channel linear in F ->
    exact recovery at interior REs; linear in T between the two DM-RS symbols, nearest outside) run
    through the fp32 reference-layout featurizer (cnrx_featurize_device);
  * the 16-bit planes the bf16 / fp16 plans actually feed their first convolutions
    (cnrx_feature_plane_device) equal round16(oracle.featurize) to within one 16-bit ulp (the kernel
    and the oracle compute the fp32 features in a different operation order), on the KAT slots and on
    random cfg2 slots at the full 612-subcarrier grid; padding channels are zero.
"""
import dataclasses

import numpy as np
import pytest

import oracle
from paper_2510_12739_b200 import graph as G, plan as P, slots
from test_slots import _hhat, _linear_channel_slot

pytestmark = pytest.mark.gpu


def _plan(prec, N):
    spec = G.conet_template(64, 2, [2], "mul", "bn", False, 6 * N, 4, "standard", 3, [1])
    for ns in [spec.main] + spec.supports:
        ns.kernel = 1
    g = G.build_conet(spec)
    g.init_he_normal(1, randomize_aux=True)
    return P.Plan(g, prec)


def _gpu_feat(p, y):
    import torch
    B, T, F, N = y.shape
    out = torch.empty((B, T, F, 6 * N), dtype=torch.float32, device="cuda")
    p.featurize_device(torch.from_numpy(y).cuda(), out)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("kind", ["freq", "time", "bilinear"])
def test_gpu_featurize_kats(kind):
    T, F, N = 14, 30, 2
    a, bf, ct = {"freq": ([0.3 + 0.2j, -0.5], [0.05 - 0.02j, 0.03j], [0, 0]),
                 "time": ([0.4 - 0.3j, 1.0], [0, 0], [0.02 + 0.05j, -0.01]),
                 "bilinear": ([1.0, 0.2 + 0.7j], [0.03j, -0.02], [0.01, 0.04 - 0.01j])}[kind]
    y, h, mask, pv = _linear_channel_slot(T, F, N, a, bf, ct)
    p = _plan("fp32", N)
    p.set_pilots(pv.astype(np.complex64), mask)
    hh = _hhat(_gpu_feat(p, y)[0], N)
    pf = np.nonzero(mask[2])[0]
    for t in (2, 11):
        np.testing.assert_allclose(hh[t, pf], h[t, pf], atol=3e-6)
    inner = np.ix_(np.arange(2, 12), np.arange(pf[0], pf[-1] + 1))
    np.testing.assert_allclose(hh[inner], h[inner], atol=3e-6)      # SPEC.md:287 (+ linear in T)
    for t in (0, 1, 12, 13):                                         # nearest outside the pilot symbols
        np.testing.assert_allclose(hh[t], hh[2 if t < 2 else 11], atol=3e-6)
    for t in (2, 11):                                                # nearest beyond the edge pilots
        np.testing.assert_allclose(hh[t, pf[-1]:], np.broadcast_to(hh[t, pf[-1]], hh[t, pf[-1]:].shape), atol=3e-6)
    np.testing.assert_allclose(_gpu_feat(p, y), oracle.featurize(y, pv.astype(np.complex64), mask), rtol=1e-5, atol=1e-6)


def _round16(x, prec):
    import torch
    dt = torch.float16 if prec == "fp16" else torch.bfloat16
    return torch.from_numpy(np.ascontiguousarray(x)).to(dt).float().numpy()


def _ulp16(x, prec):
    m = 10 if prec == "fp16" else 7
    e = np.floor(np.log2(np.maximum(np.abs(x), 1e-30)))
    return np.exp2(e - m)


@pytest.mark.parametrize("prec", ["bf16", "fp16"])
@pytest.mark.parametrize("case", ["kat", "cfg2_full"])
def test_feature_plane_equals_rounded_oracle(prec, case):
    import torch
    if case == "kat":
        y, h, mask, pv = _linear_channel_slot(14, 30, 2, [1.0, 0.2 + 0.7j], [0.03j, -0.02], [0.01, 0.04 - 0.01j])
        pv = pv.astype(np.complex64)
    else:
        link = G.CONFIGS["cfg2"].link
        b = slots.generate(link, 4, 23)
        y, mask, pv = b.y, b.pilot_mask, b.pilots
    N = y.shape[3]
    p = _plan(prec, N)
    p.set_pilots(pv, mask)
    plane = p.feature_plane(torch.from_numpy(y).cuda())
    ref = oracle.featurize(y, pv, mask)
    C = ref.shape[-1]
    assert plane.shape[-1] >= C and not plane[..., C:].any()  # padding channels are zero
    want = _round16(ref, prec)
    diff = np.abs(plane[..., :C] - want)
    # one 16-bit ulp, or 1e-6 absolute where the exact value is ~0 (e.g. Im h_hat of a real channel: the
    # kernel's fp32 complex products leave ~1e-8 residues where the oracle's are exactly zero)
    assert (diff <= np.maximum(_ulp16(want, prec), 1e-6)).all(), (diff.max(), (diff > 0).mean())
    assert (diff == 0).mean() > 0.99
