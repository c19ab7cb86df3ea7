"""GPU parity of the CNRX_FP16 plan (fp16 tensor-core operands and planes, fp32 accumulation, fp32 LLR
head): the same kernels as the bf16 plan with the other 16-bit format (csrc/elem16.cuh).  Checked
against the emulation with fp16 rounding points (tests/emulate_bf16.py FP16_POLICY) and the reference.

Tolerances: fp16 rounds 8x finer than bf16, so the bars are the bf16 ones tightened where the
rounding dominates — single layers p99 <= 1e-4 / max <= 2e-3 of max|emu|; whole networks relative L2
<= 5e-3 against the emulation and <= 5e-3 against the fp32 reference, sign agreement >= 99.5 %
(random weights).  The trained-checkpoint decision bar (>= 99.99 % over all data bits) is in
tests/test_trained.py."""
import dataclasses

import numpy as np
import pytest

import emulate_bf16 as E
import oracle
from paper_2510_12739_b200 import graph as G, plan as P, slots
from test_gpu_parity import _tiny

pytestmark = pytest.mark.gpu


def assert_fp16_layer(gpu, emu):
    rel = np.abs(gpu - emu) / np.abs(emu).max()
    assert np.quantile(rel, 0.99) <= 1e-4 and rel.max() <= 2e-3, (np.quantile(rel, 0.99), rel.max())


def assert_fp16_net(gpu, emu, ref):
    assert np.linalg.norm(gpu - emu) / np.linalg.norm(emu) <= 5e-3, np.linalg.norm(gpu - emu) / np.linalg.norm(emu)
    assert np.linalg.norm(gpu - ref) / np.linalg.norm(ref) <= 5e-3, np.linalg.norm(gpu - ref) / np.linalg.norm(ref)
    assert np.mean(np.sign(gpu) == np.sign(ref)) >= 0.995


@pytest.mark.parametrize("kind,c,dil", [("1x1", 64, 1), ("3x3", 64, 1), ("res", 64, 1), ("3x3", 64, 2),
                                        ("res", 64, 2), ("3x3", 96, 1), ("res", 96, 2), ("3x3", 32, 1)])
def test_fp16_layers_exact(kind, c, dil):
    g, x = _tiny(kind, c, dil)
    p = P.Plan(g, "fp16")
    got = p.forward(x)
    assert_fp16_layer(got, E.emulate(g, x, precision="fp16"))
    names = p.launch_names()
    assert any("f16" in n for n in names if "conv" in n), names  # the fp16 instantiations ran


@pytest.mark.parametrize("name,B,F", [("cfg1", 3, 72), ("cfg2", 2, 37), ("cfg2", 1, 612), ("cfg4", 2, 29),
                                      ("cfg4m", 1, 33), ("cfg3", 1, 40)])
def test_fp16_vs_emulation_and_oracle(name, B, F):
    g = G.CONFIGS[name].graph(seed=7)
    x = np.random.default_rng(B * F + 1).standard_normal((B, 14, F, g.in_channels)).astype(np.float32)
    got = P.Plan(g, "fp16").forward(x)
    assert_fp16_net(got, E.emulate(g, x, precision="fp16"), oracle.forward(g, x))


def test_fp16_default_program_kernels():
    """cfg2 on the fp16 plan: the same program as bf16 (fused residual blocks, TMA head) in its fp16
    instantiations; the head runs its GEMV in fp32 (no tensor-core z rounding)."""
    g = G.CONFIGS["cfg2"].graph()
    p = P.Plan(g, "fp16")
    p.forward(np.zeros((4, 14, 16, 12), np.float32))
    names = p.launch_names()
    assert sum("conv_blk64" in n for n in names) == 4, names
    assert any("head_tma" in n for n in names), names
    assert p.info()["precision"] == P.FP16


def test_fp16_two_kernel_program_matches_fused_blocks():
    """fused_blocks = 0 runs each block as two weights-stationary convs (conv_ws64<f16>): bit-identical."""
    g = G.CONFIGS["cfg2"].graph(seed=3)
    x = np.random.default_rng(2).standard_normal((3, 14, 40, 12)).astype(np.float32)
    a = P.Plan(g, "fp16", options={"fused_blocks": 1}).forward(x)
    q = P.Plan(g, "fp16", options={"fused_blocks": 0})
    b = q.forward(x)
    assert any("conv_ws64_kernel<f16>" in n for n in q.launch_names()), q.launch_names()
    assert np.array_equal(a, b)


def test_fp16_receive_full_grid_batch_invariance():
    """cfg2 at its full grid through the receive path: parity with emulation + reference on two slots, and
    every slot bit-identical alone or inside a 64-slot batch."""
    cfg = G.CONFIGS["cfg2"]
    b = slots.generate(cfg.link, 64, 31)
    g = cfg.graph(seed=21)
    p = P.Plan(g, "fp16")
    p.set_pilots(b.pilots, b.pilot_mask)
    full = p.receive(b.y)
    for i in (0, 63):
        assert np.array_equal(p.receive(b.y[i:i + 1])[0], full[i])
    feat = oracle.featurize(b.y[[0, 63]], b.pilots, b.pilot_mask)
    assert_fp16_net(full[[0, 63]], E.emulate(g, feat, precision="fp16"), oracle.forward(g, feat))


def test_plan_options_round_trip_and_env_free():
    """cnrx_plan_create_ex takes explicit options (no environment): they are reported back unchanged."""
    g = G.CONFIGS["cfg2"].graph()
    d = P.default_options()
    assert d["fused_blocks"] == 1 and d["cta_pair"] == 1 and d["fused_head"] == 0
    p = P.Plan(g, "bf16", options={"fused_blocks": 0, "pipeline_chunks": 3})
    o = p.options()
    assert o["fused_blocks"] == 0 and o["pipeline_chunks"] == 3 and o["cta_pair"] == 1


def test_fp16_packs_saturate_instead_of_overflowing():
    """fp16 planes hold |x| <= 65504: out-of-range values saturate (cvt.rn.satfinite) rather than
    becoming inf and poisoning the network with NaNs downstream."""
    import torch
    link = dataclasses.replace(G.CONFIGS["cfg2"].link, F=48)
    b = slots.generate(link, 2, 3)
    spec = G.conet_template(64, 2, [2], "mul", "bn", False, 12, 4, "standard", 3, [1])
    for ns in [spec.main] + spec.supports:
        ns.kernel = 1
    g = G.build_conet(spec)
    g.init_he_normal(1, randomize_aux=True)
    p = P.Plan(g, "fp16")
    p.set_pilots(b.pilots, b.pilot_mask)
    y = torch.from_numpy(b.y * np.float32(3e5)).cuda()   # |Re y| up to ~1e6 > 65504
    plane = p.feature_plane(y)
    assert np.isfinite(plane).all() and np.abs(plane).max() == 65504.0
    out = torch.empty((2, link.T, link.F, 4), dtype=torch.float32, device="cuda")
    p.receive_device(y, out)
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()
