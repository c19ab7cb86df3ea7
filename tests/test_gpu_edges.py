"""Edge cases of the drop-in boundary on the GPU: empty / degenerate shapes rejected exactly as the
reference rejects them (tensor.hpp checked_numel -> std::invalid_argument "tensor dimensions must be
positive"), the one-plane row limit, recovery after a failed workspace build, the smallest grids, and
the largest batch the bench sweeps (per-slot results identical to running the slot alone)."""
import ctypes as C

import numpy as np
import pytest

import oracle
import emulate_bf16 as E
from paper_2510_12739_b200 import graph as G, plan as P, slots

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_empty_and_degenerate_shapes_are_rejected_like_the_reference(prec):
    p = P.Plan(G.CONFIGS["cfg1"].graph(), prec)
    for shape in [(0, 14, 72, 6), (2, 0, 72, 6), (2, 14, 0, 6)]:
        with pytest.raises(P.CnrxInvalidArgument, match="dimensions must be positive"):
            p.forward(np.zeros(shape, np.float32))
    # the plan is still usable afterwards
    x = np.random.default_rng(0).standard_normal((1, 14, 72, 6)).astype(np.float32)
    y = p.forward(x)
    assert y.shape == (1, 14, 72, 2) and np.isfinite(y).all()


def test_batch_beyond_one_plane_is_an_error_and_the_plan_recovers(monkeypatch):
    """Batches whose workspace exceeds the plan's memory budget run in slot chunks (test_gpu_x3.py); with the
    budget lifted, a chunk beyond 2^31 plane rows is rejected before any allocation or access."""
    import torch
    monkeypatch.setenv("CNRX_MEM_BUDGET_MB", "1e12")
    g = G.CONFIGS["cfg2"].graph()
    p = P.Plan(g, "bf16")
    x = torch.zeros((1, 14, 612, 12), dtype=torch.float32, device="cuda")
    out = torch.zeros((1, 14, 612, 4), dtype=torch.float32, device="cuda")
    huge = 240_000  # 240000 slots x 9195 rows > 2^31 plane rows: rejected before any allocation or access
    for _ in range(2):  # twice: a failed build must not leave a stale workspace for the same shape
        rc = P.lib().cnrx_forward_device(p.h, C.c_void_p(x.data_ptr()), huge, 14, 612, 12, P.MODE_EVAL,
                                         C.c_void_p(out.data_ptr()), None)
        assert rc == P.ERR_INVALID_ARGUMENT
        assert "too large" in P.lib().cnrx_last_error().decode()
    xs = np.random.default_rng(1).standard_normal((2, 14, 612, 12)).astype(np.float32)
    assert np.isfinite(p.forward(xs)).all()


@pytest.mark.parametrize("F", [1, 2, 3])
def test_smallest_grids_fp32_bit_exact_bf16_vs_emulation(F):
    g = G.CONFIGS["cfg2"].graph(seed=5)
    x = np.random.default_rng(F).standard_normal((2, 14, F, 12)).astype(np.float32)
    ref = oracle.RefNet.from_graph(g).forward(x)
    assert np.array_equal(P.Plan(g, "fp32").forward(x), ref)
    got = P.Plan(g, "bf16").forward(x)
    emu = E.emulate(g, x)
    assert np.linalg.norm(got - emu) / np.linalg.norm(emu) <= 2e-2


def test_largest_bench_batch_slots_match_single_slot_runs():
    """B = 4096 cfg2 slots through the device receive path (30 GB of activation planes): sampled slots
    are bit-identical to the same slot received alone."""
    import torch
    cfg = G.CONFIGS["cfg2"]
    link = cfg.link
    g = cfg.graph(seed=9)
    p = P.Plan(g, "bf16")
    pmask, pvals = slots.pilot_pattern(link.T, link.F, link.pilot_symbols, link.pilot_spacing)
    p.set_pilots(pvals.astype(np.complex64), pmask)
    B = 4096
    y, _bits = P.generate_slots_device(link, B, 77, slot0=0)
    out = torch.empty((B, link.T, link.F, link.bits), dtype=torch.float32, device="cuda")
    p.receive_device(y, out, torch.cuda.current_stream().cuda_stream)
    one = torch.empty((1, link.T, link.F, link.bits), dtype=torch.float32, device="cuda")
    for i in (0, 1234, B - 1):
        p.receive_device(y[i:i + 1].contiguous(), one, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert torch.equal(one[0], out[i]), i
    assert torch.isfinite(out).all()


@pytest.mark.parametrize("k,dil,cin,cout,T,F", [
    (3, 1, 6, 32, 14, 72),     # cfg1's first conv: narrow input, tile kernel <1,8,2>
    (1, 1, 1, 1, 1, 1),        # smallest everything
    (5, 3, 33, 17, 7, 40),     # 5x5 dilated, odd channel counts, partial output-channel group
    (3, 2, 64, 24, 12, 37),    # wide input: two pixels per thread <2,8,2>, ragged F tiles
    (3, 1, 96, 16, 14, 20),    # 96 channels: one pixel per thread, weights streamed per tap (ws)
    (3, 2, 128, 8, 14, 19),    # 128 channels, dilated: ws
    (3, 1, 320, 8, 14, 9),     # window too large for shared memory: direct-conv fallback
    (3, 1, 8, 8, 64, 5),       # T = 64: two columns per tile
    (3, 1, 8, 8, 65, 5),       # T > 64: direct-conv fallback
])
def test_fp32_conv_tiles_bit_exact(k, dil, cin, cout, T, F):
    """The fp32 direct conv over its tiling corners (conv_f32_tile_kernel variants and the conv_f32_px
    fallback) inside a conv -> BN -> ReLU -> conv -> add block: bit-exact with the reference arithmetic."""
    g = G.Graph()
    xi = g.add_input(cin)
    s = g.add_conv(xi, "s", k, cin, cout, True, dilation_f=dil)
    h = g.add_relu(g.add_norm(g.add_conv(s, "a", k, cout, cout, False, dilation_f=dil), "bn", "n", cout))
    g.set_output(g.add_binary(G.OP_ADD, g.add_conv(h, "b", k, cout, cout, True, dilation_f=dil), s))
    g.init_he_normal(k * 100 + cin, randomize_aux=True)
    x = np.random.default_rng(cin + T).standard_normal((3, T, F, cin)).astype(np.float32)
    p = P.Plan(g, "fp32")
    got = p.forward(x)
    assert np.array_equal(got, oracle.forward(g, x)), "fp32 conv differs from the reference arithmetic"
    names = p.launch_names()
    fallback = cin == 320 or T > 64  # conv_f32_px_kernel, or conv_f32_kernel on small grids
    assert any(("conv_f32_px" in n or n == "conv_f32_kernel") if fallback else "conv_f32_tile" in n for n in names), names
    if cin in (96, 128):
        assert any(n.endswith(",ws>") for n in names), names
