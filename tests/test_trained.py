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
CKPT3 = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cfg3_trained.cnck")
pytestmark = pytest.mark.skipif(not os.path.exists(CKPT), reason="trained checkpoint not generated")


def _graph(name="cfg2"):
    g = G.CONFIGS[name].graph_fn()
    Fi.load_checkpoint(g, CKPT if name == "cfg2" else CKPT3)
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


def _decision_run(precisions, n_batches=9, B=32, seed=12345, name="cfg2"):
    """Hard decisions of plans of the given precisions against the fp32 plan (bit-exact with the
    reference) on n_batches x B GPU-generated slots; data bits only (pilots excluded)."""
    import torch
    from paper_2510_12739_b200 import plan as P
    g = _graph(name)
    link = G.CONFIGS[name].link
    pmask, pvals = slots.pilot_pattern(link.T, link.F, link.pilot_symbols, link.pilot_spacing)
    plans = {pr: P.Plan(g, pr) for pr in ("fp32",) + tuple(precisions)}
    for p in plans.values():
        p.set_pilots(pvals.astype(np.complex64), pmask)
    data = torch.from_numpy(pmask == 0).cuda()
    st = torch.cuda.current_stream().cuda_stream
    res = {pr: dict(agree=0, conf_agree=0, conf=0, err=0) for pr in precisions}
    err32 = err_ls = nbits = 0
    for k in range(n_batches):
        y, bits, _ = P.generate_slots_device(link, B, seed, slot0=k * B, with_h=True)
        out = {}
        for pr, p in plans.items():
            out[pr] = torch.empty((B, link.T, link.F, link.bits), dtype=torch.float32, device="cuda")
            p.receive_device(y, out[pr], st)
        m = data[None, :, :, None].expand_as(out["fp32"])
        a32 = out["fp32"][m]
        confident = a32.abs() >= 1.0  # |LLR| >= 1: P(bit) >= 0.73
        nbits += a32.numel()
        err32 += int(P.count_bit_errors(out["fp32"], bits, data).sum())
        nv = P.slot_noise_var(link, B, seed, slot0=k * B)
        err_ls += int(P.count_bit_errors(P.classical_receive_device(plans["fp32"], y, nv, link.mod_order), bits,
                                         data).sum())
        for pr in precisions:
            a = out[pr][m]
            same = (a32 > 0) == (a > 0)
            r = res[pr]
            r["agree"] += int(same.sum())
            r["conf_agree"] += int(same[confident].sum())
            r["conf"] += int(confident.sum())
            r["err"] += int(P.count_bit_errors(out[pr], bits, data).sum())
    return res, err32, err_ls, nbits


@pytest.mark.gpu
def test_trained_fp16_meets_the_decision_bar():
    """North star: hard-decision bits >= 99.99 % identical to the reference's (the fp32 plan is bit-exact
    with it) over ALL data bits, on >= 8M bits, and the same BER within Monte-Carlo confidence.  The
    CNRX_FP16 plan (fp16 tensor-core operands, fp32 head) is the mixed-precision option that meets it;
    bf16 cannot (tools/ablate_bf16.py: bf16 conv operands alone cap agreement at ~99.97-99.99 %)."""
    res, e32, e_ls, n = _decision_run(("fp16", "bf16", "bf16x3"))
    assert n >= 8_000_000
    r16, rb, rx = res["fp16"], res["bf16"], res["bf16x3"]
    a16, ab = r16["agree"] / n, rb["agree"] / n
    ber32, ber16 = e32 / n, r16["err"] / n
    sigma = np.sqrt(ber32 * (1 - ber32) / n)  # binomial std of the BER estimate
    print(f"bits {n}: fp16 agree {a16:.6f} (confident {r16['conf_agree'] / r16['conf']:.6f}), bf16 agree {ab:.6f}; "
          f"BER fp32 {ber32:.5f} fp16 {ber16:.5f} bf16 {rb['err'] / n:.5f} LS-LMMSE {e_ls / n:.5f}")
    print(f"bf16x3 agree {rx['agree'] / n:.7f} BER {rx['err'] / n:.5f}")
    assert a16 >= 0.9999
    assert rx["agree"] / n >= 0.9999 and abs(rx["err"] / n - ber32) <= 3 * sigma  # split-precision plan
    assert abs(ber16 - ber32) <= 3 * sigma      # the same BER within Monte-Carlo confidence
    assert e32 < e_ls                           # the trained receiver beats LS-LMMSE on the same slots
    # bf16: recorded ceiling, not the north-star bar
    assert ab >= 0.999 and abs(rb["err"] / n - ber32) <= 3 * sigma


@pytest.mark.skipif(not os.path.exists(CKPT3), reason="cfg3 checkpoint not generated")
def test_cfg3_checkpoint_loads():
    g = _graph("cfg3")
    assert all(g.bn_ready) and g.learnable_count() == G.CONFIGS["cfg3"].graph_fn().learnable_count()


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(CKPT3), reason="cfg3 checkpoint not generated")
def test_trained_cfg3_fp32_bit_exact_and_16bit_decisions():
    """cfg3 (4 subnets x 6 MRB @ 96, dilation 2, 64-QAM + interferer) with TRAINED weights
    (tools/train_cfg.py, 8000 steps; profiles/r02_train_cfg3.json: BER 0.170 vs LS-LMMSE 0.202):
      * the fp32 plan is bit-exact with the oracle (the reference restated with dilation) on crops
        with the receptive-radius margin, at the full 3276-subcarrier grid;
      * fp16 / bf16 hard decisions vs fp32 over >= 8 M data bits, same BER within 3 sigma.  The recorded
        agreement is below the 99.99 % bar that fp16 meets on cfg2: this network sits at BER 0.17, so
        many more bits are near the decision boundary, and the ablation (tools/ablate_bf16.py CFG=cfg3)
        shows no single fp32 rounding point closes the gap (fp16 operands alone cap it at ~99.99 %);
        the fp32 plan is the exact mode."""
    import oracle
    import torch
    from paper_2510_12739_b200 import plan as P
    g = _graph("cfg3")
    cfg = G.CONFIGS["cfg3"]
    b = slots.generate(cfg.link, 1, 5)
    feat = oracle.featurize(b.y, b.pilots, b.pilot_mask)
    got = P.Plan(g, "fp32").forward(feat)
    R = 25
    for a, e in ((0, 96), (1600, 1696), (3180, 3276)):
        lo, hi = max(0, a - R), min(3276, e + R)
        ref = oracle.forward(g, np.ascontiguousarray(feat[:, :, lo:hi]))
        assert np.array_equal(got[:, :, a:e], ref[:, :, a - lo:e - lo]), a
    res, e32, e_ls, n = _decision_run(("fp16", "bf16", "bf16x3"), n_batches=16, B=4, name="cfg3")
    assert n >= 8_000_000
    ber32 = e32 / n
    sigma = np.sqrt(ber32 * (1 - ber32) / n)
    r16, rb, rx = res["fp16"], res["bf16"], res["bf16x3"]
    print(f"cfg3 bf16x3 agree {rx['agree'] / n:.7f} BER {rx['err'] / n:.5f}")
    # the split-precision plan meets the north-star bar on cfg3 too
    assert rx["agree"] / n >= 0.9999 and abs(rx["err"] / n - ber32) <= 3 * sigma
    print(f"cfg3 bits {n}: fp16 agree {r16['agree'] / n:.6f} (confident {r16['conf_agree'] / r16['conf']:.6f}), "
          f"bf16 agree {rb['agree'] / n:.6f}; BER fp32 {ber32:.5f} fp16 {r16['err'] / n:.5f} bf16 {rb['err'] / n:.5f} "
          f"LS-LMMSE {e_ls / n:.5f}")
    assert r16["agree"] / n >= 0.9998 and rb["agree"] / n >= 0.998
    assert r16["conf_agree"] == r16["conf"]          # every |LLR| >= 1 decision identical
    for r in (r16, rb):
        assert abs(r["err"] / n - ber32) <= 3 * sigma
    assert e32 < e_ls
