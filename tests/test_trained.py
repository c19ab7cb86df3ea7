"""Parity with TRAINED weights (tests/golden/cfg2_trained.cnck, made by tools/train_cfg.py on GPU-generated
slots): the fp32 plan is bit-exact with the reference on the loaded checkpoint, the bf16 plan makes the
same hard decisions (>= 99.99 % on confident decisions) and the same BER, and the trained
CoNet beats the LS-LMMSE baseline on the same slots."""
import dataclasses
import os

import numpy as np
import pytest

from paper_2510_12739_b200 import files as Fi
from paper_2510_12739_b200 import graph as G
from paper_2510_12739_b200 import slots

CKPT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cfg2_trained.cnck")
pytestmark = pytest.mark.skipif(not os.path.exists(CKPT), reason="trained checkpoint not generated")


def _graph():
    g = G.CONFIGS["cfg2"].graph_fn()
    Fi.load_checkpoint(g, CKPT)
    return g


def test_checkpoint_loads_into_cfg2():
    g = _graph()
    assert all(g.bn_ready) and g.learnable_count() == G.CONFIGS["cfg2"].graph_fn().learnable_count()
    assert all(np.isfinite(p.value).all() for p in g.params)


def test_checkpoint_round_trips_through_the_reference(ref, tmp_path):
    import oracle
    g = _graph()
    rn = oracle.RefNet.from_graph(g)
    path = str(tmp_path / "re.cnck")
    rn.save_checkpoint(path)
    assert open(path, "rb").read() == open(CKPT, "rb").read()


@pytest.mark.gpu
def test_trained_fp32_bit_exact_with_reference(ref):
    import oracle
    from paper_2510_12739_b200 import plan as P
    g = _graph()
    link = dataclasses.replace(G.CONFIGS["cfg2"].link, F=96)
    b = slots.generate(link, 2, 41)
    feat = oracle.featurize(b.y, b.pilots, b.pilot_mask)
    p = P.Plan(g, "fp32")
    assert np.array_equal(p.forward(feat), oracle.RefNet.from_graph(g).forward(feat))


@pytest.mark.gpu
def test_trained_bf16_hard_decisions_and_ber():
    import torch
    from paper_2510_12739_b200 import plan as P
    g = _graph()
    link = G.CONFIGS["cfg2"].link
    pmask, pvals = slots.pilot_pattern(link.T, link.F, link.pilot_symbols, link.pilot_spacing)
    p32, p16 = P.Plan(g, "fp32"), P.Plan(g, "bf16")
    for p in (p32, p16):
        p.set_pilots(pvals.astype(np.complex64), pmask)
    data = torch.from_numpy(pmask == 0).cuda()
    B = 32
    y, bits, h = P.generate_slots_device(link, B, 12345, slot0=0, with_h=True)
    l32 = torch.empty((B, link.T, link.F, link.bits), dtype=torch.float32, device="cuda")
    l16 = torch.empty_like(l32)
    st = torch.cuda.current_stream().cuda_stream
    p32.receive_device(y, l32, st)
    p16.receive_device(y, l16, st)
    m = data[None, :, :, None].expand_as(l32)
    a32, a16 = l32[m], l16[m]
    agree = float(((a32 > 0) == (a16 > 0)).float().mean())
    confident = a32.abs() >= 1.0  # |LLR| >= 1: P(bit) >= 0.73
    agree_conf = float(((a32 > 0) == (a16 > 0))[confident].float().mean())
    e32 = int(P.count_bit_errors(l32, bits, data).sum())
    e16 = int(P.count_bit_errors(l16, bits, data).sum())
    nbits = B * int(data.sum()) * link.bits
    nv = P.slot_noise_var(link, B, 12345)
    e_ls = int(P.count_bit_errors(P.classical_receive_device(p32, y, nv, link.mod_order), bits, data).sum())
    print(f"agree {agree:.6f} confident {agree_conf:.6f} ({float(confident.float().mean()):.3f} of bits) "
          f"BER fp32 {e32 / nbits:.5f} bf16 {e16 / nbits:.5f} LS-LMMSE {e_ls / nbits:.5f}")
    assert agree_conf >= 0.9999
    assert agree >= 0.999
    assert abs(e16 - e32) / nbits <= 5e-4  # same BER
    assert e32 < e_ls                       # the trained receiver beats LS-LMMSE on the same slots
