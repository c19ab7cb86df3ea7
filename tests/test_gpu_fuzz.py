"""Randomised builder graphs (the reference's conet_template / deeprx_template, netspec.cpp:53-81, with
random widths, depths, fusion ops and points, stem/head kernels, input channels and bit counts) through
every plan precision, against the oracle on random inputs (seeded, so a failure reproduces):
  * fp32: bit-exact;
  * bf16x3 / fp16x3: rel L2 <= 1e-4 and max |d| / max |ref| <= 1e-4 (fp16x3, inside its fp16 value range)
    / 2e-4 (bf16x3; tests/test_gpu_x3.py keeps 1e-4 on the BASELINE configs), and the split plans lower
    every graph the bf16 plan lowers;
  * bf16 / fp16: within the emulation bound of tests/test_gpu_parity.py (rel L2 <= 2e-2 / 5e-3).
Graphs a 16-bit plan cannot express must be rejected loudly (CnrxUnsupported), never computed wrong.
Since round 2 the tensor-core plans also lower 3x3 LLR heads (NetSpec.kernel = 3: a conv whose epilogue
writes the fp32 LLRs), LN fusion norms (a row-wise program with double statistics), concat fusion at
widths <= 64 (the planes side by side, then the 1x1 restore conv) and depthwise-separable convs (the
depthwise stage on CUDA cores over the plane, the pointwise stage on the tensor cores)."""
import dataclasses
import os

import numpy as np
import pytest

import oracle
import emulate_bf16 as E
from paper_2510_12739_b200 import graph as G, plan as P

pytestmark = pytest.mark.gpu


def _random_graph(seed):
    r = np.random.default_rng(seed)
    in_ch = int(r.choice([6, 12, 24]))
    bits = int(r.choice([2, 4, 6]))
    width = int(r.choice([32, 64, 96]))
    kernel = int(r.choice([1, 1, 1, 3]))  # stem / head kernel (the 16-bit plans lower 1x1 heads only)
    if r.random() < 0.25:
        spec = dataclasses.replace(G.deeprx_template(width, int(r.integers(1, 4)), in_ch, bits), kernel=kernel)
        g = G.build_net(spec)
    else:
        main = int(r.integers(1, 4))
        sups = [int(x) for x in r.integers(1, 4, size=int(r.integers(1, 4)))]
        op = str(r.choice(["mul", "add", "concat"] if width <= 64 else ["mul", "add"]))
        pts = sorted(set(int(x) for x in r.integers(0, main, size=int(r.integers(1, main + 1)))))
        bidir = bool(r.random() < 0.3)  # feedback fusion (network.hpp:518-522)
        norm = str(r.choice(["bn", "bn", "ln"]))  # fusion norm (network.hpp:550)
        conv = str(r.choice(["standard", "standard", "depthwise"]))  # conv_stage kinds (network.hpp:443-449)
        spec = G.conet_template(width, main, sups, op, norm, bidir, in_ch, bits, conv=conv, kernel=kernel,
                                fusion_points=pts)
        g = G.build_conet(spec)
    g.init_he_normal(seed, randomize_aux=True)
    B, F = int(r.integers(1, 4)), int(r.integers(3, 40))
    x = r.standard_normal((B, 14, F, in_ch)).astype(np.float32)
    return g, x


# CNRX_FUZZ_SEEDS widens the soak (profiles/r02n_fuzz_soak.log: 600 seeds); the default keeps the suite short
@pytest.mark.parametrize("seed", range(int(os.environ.get("CNRX_FUZZ_SEEDS", "48"))))
def test_random_builder_graphs_all_precisions(seed):
    g, x = _random_graph(1000 + seed)
    ref = oracle.forward(g, x)
    assert np.array_equal(P.Plan(g, "fp32").forward(x), ref)
    lowered = {}
    for prec in ("bf16", "fp16", "bf16x3", "fp16x3"):
        try:
            lowered[prec] = P.Plan(g, prec).forward(x)
        except P.CnrxUnsupported:
            lowered[prec] = None
    if lowered["bf16"] is not None:  # the split plans lower whatever the 16-bit plans lower
        assert lowered["bf16x3"] is not None and lowered["fp16x3"] is not None
    # norms in double: random fusion norms can make |LLR| ~ 1e30 and a float32 norm overflows to inf / inf
    ref64 = ref.astype(np.float64)
    scale = np.abs(ref64).max()
    # the fp16 split plan's documented domain is |value| <= 65504 (DESIGN 4): multiplicative fusion chains with
    # random norm parameters leave it on ~2 % of the seeds (600-seed soak, profiles/r02n_fuzz_soak.log: every
    # fp16x3 miss had max |activation| > 2.6e4, up to 1e30) -- those graphs are checked on bf16x3 only
    amax = [0.0]

    def rec(t):
        amax[0] = max(amax[0], float(t.abs().max()))
        return t
    E.emulate(g, x, policy={k: rec for k in E.BF16_POLICY})
    # max-norm bar: 1e-4 for fp16x3 (22 significant bits); 2e-4 for bf16x3 on these random graphs -- 16 significant
    # bits per value reach 0.8e-4 on a 25-conv, 6-product graph already in the CPU emulation of the split
    # (seed 125: GPU 1.2e-4), the BASELINE configs keep 1e-4 (tests/test_gpu_x3.py)
    for prec, mx_bar in (("bf16x3", 2e-4), ("fp16x3", 1e-4)):
        got = lowered[prec]
        if got is None or (prec == "fp16x3" and amax[0] > 3e4):
            continue
        d = got.astype(np.float64) - ref64
        l2 = np.linalg.norm(d) / np.linalg.norm(ref64)
        mx = np.abs(d).max() / scale
        assert l2 <= 1e-4 and mx <= mx_bar, (prec, l2, mx)
    for prec, bound in (("bf16", 2e-2), ("fp16", 5e-3)):
        got = lowered[prec]
        if got is None or (prec == "fp16" and amax[0] > 3e4):  # outside fp16's range the packs saturate (documented)
            continue
        emu = E.emulate(g, x, precision=prec).astype(np.float64)
        assert np.linalg.norm(got.astype(np.float64) - emu) / np.linalg.norm(emu) <= bound, prec
