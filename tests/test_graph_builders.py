"""paper_2510_12739_b200.graph builds the same networks as the reference builders (network.hpp:470-600,
netspec.cpp:42-81): node records, parameter names/shapes/learnability, reports."""
import numpy as np
import pytest

import oracle
from paper_2510_12739_b200 import graph as G


def _same(g, r):
    assert np.array_equal(r.nodes(), g.node_array()[:, :11])
    assert [(p.name, p.value.shape, p.learnable) for p in g.params] == r.params()
    assert g.learnable_count() == r.learnable_count()
    assert g.conv_depth() == r.conv_depth()


@pytest.mark.parametrize("blocks,sup,fp", [(4, [4, 4], [3]), (2, [1], []), (3, [2, 3], [0, 2])])
def test_build_conet_matches_reference(ref, blocks, sup, fp):
    spec = G.conet_template(24, blocks, sup, "mul", "bn", False, 12, 4, "standard", 3, fp)
    spec.main.kernel = 1
    for s in spec.supports:
        s.kernel = 1
    r = oracle.RefNet.conet(24, blocks, sup, 12, 4, fusion_points=fp)
    _same(G.build_conet(spec), r)


def test_build_deeprx_matches_reference(ref):
    spec = G.deeprx_template(32, 3, 12, 4)
    spec.kernel = 1
    _same(G.build_net(spec), oracle.RefNet.deeprx(32, 3, 12, 4))


def test_config_graphs_replay_into_reference(ref):
    for name in ("cfg1", "cfg2", "cfg4"):
        g = G.CONFIGS[name].graph()
        _same(g, oracle.RefNet.from_graph(g))


def test_config_sizes():
    assert G.CONFIGS["cfg2"].graph().macs_per_re() == 887296
    assert G.CONFIGS["cfg1"].graph().macs_per_re() == 58816
    assert G.CONFIGS["cfg4"].graph().macs_per_re() == 1328640
    g3 = G.CONFIGS["cfg3"].graph()
    assert g3.max_dilation() == 2 and g3.output_channels() == 6 and g3.in_channels == 24


def test_param_count_kat(ref):
    """a single 3x3 conv 6->8 with bias has 440 parameters."""
    g = G.Graph()
    x = g.add_input(6)
    g.set_output(g.add_conv(x, "c", 3, 6, 8, True))
    assert g.learnable_count() == 440


def test_depth_14_vs_24(ref):
    """PAPER.md:210 / SPEC.md:387: CoNet with 14 sequential convs vs DeepRx with 24 (41.7% shallower)."""
    conet = oracle.RefNet.conet(64, 6, [6], 6, 6, block_kernel=3, io_kernel=3)
    deeprx = oracle.RefNet.deeprx(64, 11, 6, 6, block_kernel=3, io_kernel=3)
    assert conet.conv_depth() == 14 and deeprx.conv_depth() == 24


def test_validation_errors():
    with pytest.raises(ValueError, match="equal channel counts"):
        spec = G.conet_template(16, 2, [2], "mul", "bn", False, 6, 2)
        spec.supports[0].blocks[1].filters = 8
        G.build_conet(spec)
    g = G.Graph()
    x = g.add_input(6)
    with pytest.raises(ValueError, match="expects 5 input channels"):
        g.add_conv(x, "c", 3, 5, 8, True)
