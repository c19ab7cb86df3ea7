"""Kernel programs against each other, bit for bit, selected per plan with cnrx_plan_options
(cnrx_plan_create_ex; no environment switches):
  * the CTA-pair 96 -> 96 3x3 conv (csrc/conv_pair.cu, default) vs the single-CTA kernel (cta_pair = 0):
    same UMMA K order per output element, same epilogue -> identical LLRs;
  * the fused residual-block kernel (csrc/conv_blk.cu, default) vs the two-kernel program
    (fused_blocks = 0): conv1's output is rounded to 16 bits at the same point in both -> identical LLRs;
  * the CoNet interaction + LLR head folded into the last fused blocks (conv_blk.cu BlkFold: one launch per
    subnetwork, fp32 partial folds, fp32 head GEMV in head.cu's summation order; fused_head = 1) vs the
    separate head kernel: identical LLRs, bf16 and fp16, 2 / 3 / 4 subnetworks;
  * the two-kernel program's fused head (conv_ws.cu kWsHead: clusters of one CTA per subnetwork exchanging
    tiles through distributed shared memory, tensor-core head) vs the separate tensor-core head kernel."""
import numpy as np
import pytest

from paper_2510_12739_b200 import graph as G, plan as P

pytestmark = pytest.mark.gpu


def _graph(which):
    if which == "cfg2":
        g = G.CONFIGS["cfg2"].graph()
        x = np.random.default_rng(7).standard_normal((5, 14, 101, 12)).astype(np.float32)
    elif which == "cfg4":  # 96-channel RB net; 3 slots x 15 x 105 rows -> an odd number of 128-row tiles
        g = G.CONFIGS["cfg4"].graph()
        x = np.random.default_rng(9).standard_normal((3, 14, 101, 12)).astype(np.float32)
    elif which == "dilated96":
        g = G.Graph()
        xi = g.add_input(24)
        s = g.add_relu(g.add_conv(xi, "s", 1, 24, 96, True))
        for k in range(2):
            h1 = g.add_relu(g.add_norm(g.add_conv(g.add_relu(s), f"a{k}", 3, 96, 96, False, dilation_f=2), "bn", f"n{k}", 96))
            s = g.add_binary(G.OP_ADD, g.add_conv(h1, f"b{k}", 3, 96, 96, True, dilation_f=2), s)
        g.set_output(g.add_conv(s, "out", 1, 96, 6, True))
        g.init_he_normal(4, randomize_aux=True)
        x = np.random.default_rng(10).standard_normal((2, 14, 133, 24)).astype(np.float32)
    elif which in ("conet2", "conet4"):  # 2 / 4 MRB subnetworks @ 64, fusion at the last block
        sup = [2] if which == "conet2" else [2, 2, 2]
        spec = G.conet_template(64, 2, sup, "mul", "bn", False, 12, 6, "standard", 3, [1])
        for ns in [spec.main] + spec.supports:
            ns.kernel = 1
        g = G.build_conet(spec)
        g.init_he_normal(6, randomize_aux=True)
        x = np.random.default_rng(11).standard_normal((3, 14, 57, 12)).astype(np.float32)
    else:  # MRB-style blocks with dilation 2 in F, ragged grid
        g = G.Graph()
        xi = g.add_input(12)
        s = g.add_relu(g.add_conv(xi, "s", 1, 12, 64, True))
        for k in range(2):
            h1 = g.add_relu(g.add_norm(g.add_conv(g.add_relu(s), f"a{k}", 3, 64, 64, False, dilation_f=2), "bn", f"n{k}", 64))
            s = g.add_binary(G.OP_ADD, g.add_conv(h1, f"b{k}", 3, 64, 64, True, dilation_f=2), s)
        g.set_output(g.add_conv(s, "out", 1, 64, 4, True))
        g.init_he_normal(3, randomize_aux=True)
        x = np.random.default_rng(8).standard_normal((3, 14, 77, 12)).astype(np.float32)
    return g, x


def _run(which, prec="bf16", **opts):
    g, x = _graph(which)
    p = P.Plan(g, prec, options=opts)
    y = p.forward(x)
    return y, p.launch_names()


def _same(a, b):
    assert np.isfinite(a).all()
    assert np.array_equal(a, b), (np.abs(a - b).max(), int((a != b).sum()))


@pytest.mark.parametrize("which", ["cfg2", "dilated"])
def test_fused_block_kernel_is_bit_exact(which):
    yf, lf = _run(which, fused_blocks=1)
    yu, lu = _run(which, fused_blocks=0)
    assert any("conv_blk64" in n for n in lf), lf
    assert not any("conv_blk64" in n for n in lu), lu
    _same(yf, yu)


@pytest.mark.parametrize("which", ["cfg4", "dilated96"])
def test_cta_pair_conv_is_bit_exact_with_single_cta(which):
    yp, lp = _run(which, cta_pair=1)
    ys, ls = _run(which, cta_pair=0)
    assert any("conv_pair96" in n for n in lp), lp
    assert not any("conv_pair96" in n for n in ls), ls
    _same(yp, ys)


@pytest.mark.parametrize("prec", ["bf16", "fp16"])
@pytest.mark.parametrize("which", ["dilated96", "cfg3"])
def test_pair_relu_on_load_is_bit_exact(which, prec):
    """96-channel MRB blocks: conv1 applies the input ReLU to its window in shared memory (two ReLU warps
    per CTA of the pair) instead of reading a pre-activated plane the previous conv2 wrote."""
    if which == "cfg3":
        g = G.CONFIGS["cfg3"].graph(seed=5)
        x = np.random.default_rng(5).standard_normal((1, 14, 70, g.in_channels)).astype(np.float32)
        q = P.Plan(g, prec, options={"relu_on_load": 1})
        yo = q.forward(x)
        lo = q.launch_names()
        r = P.Plan(g, prec, options={"relu_on_load": 0})
        yp, lp = r.forward(x), r.launch_names()
    else:
        yo, lo = _run(which, prec, relu_on_load=1)
        yp, lp = _run(which, prec, relu_on_load=0)
    assert any("relu_in" in n for n in lo), lo
    assert not any("relu_in" in n for n in lp), lp
    assert len(lo) <= len(lp)
    _same(yo, yp)


@pytest.mark.parametrize("prec", ["bf16", "fp16"])
@pytest.mark.parametrize("which", ["cfg2", "conet2", "conet4"])
def test_fused_block_head_is_bit_exact_with_head_kernel(which, prec):
    yh, lh = _run(which, prec, fused_head=1)
    yk, lk = _run(which, prec, fused_head=0)
    assert any("<fold+head>" in n for n in lh) and not any("head_tma" in n for n in lh), lh
    if which != "conet2":
        assert any("<fold>" in n for n in lh), lh  # mid launches with an fp32 partial-fold plane
    assert any("head_tma" in n for n in lk), lk
    _same(yh, yk)


@pytest.mark.parametrize("which", ["cfg2", "dilated"])
def test_ws_fused_head_is_bit_exact_with_tc_head_kernel(which):
    # two-kernel program in both arms, tensor-core head, head fused into the last convs or not
    yh, lh = _run(which, fused_blocks=0, fused_head=1, tensor_core_head=1)
    yk, lk = _run(which, fused_blocks=0, fused_head=0, tensor_core_head=1)
    assert any("<head>" in n for n in lh) and not any("head_tma" in n for n in lh), lh
    assert not any("<head>" in n for n in lk) and any("head_tma" in n for n in lk), lk
    _same(yh, yk)
