"""The bf16 emulator used by the GPU tests tracks the reference within bf16 accuracy."""
import numpy as np

import oracle
import emulate_bf16 as E
from paper_2510_12739_b200 import graph as G


def test_emulator_tracks_reference(oracle_lib):
    for name in ("cfg1", "cfg2", "cfg4"):
        g = G.CONFIGS[name].graph(seed=2)
        x = np.random.default_rng(1).standard_normal((1, 14, 24, g.in_channels)).astype(np.float32)
        r = oracle.forward(g, x)
        e = E.emulate(g, x)
        assert np.linalg.norm(e - r) / np.linalg.norm(r) < 0.02
        assert np.mean(np.sign(e) == np.sign(r)) > 0.99
