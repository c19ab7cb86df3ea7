"""Opt-in fused residual-block kernel (csrc/conv_blk.cu, CNRX_BLK=1) against the default two-kernel
path: bit-identical LLRs (conv1's output is rounded to bf16 at the same point in both, and both
accumulate the same UMMA sequence).  The switch is read at plan compile, so each arm runs in its own
process."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

ARM = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2510_12739_b200 import graph as G, plan as P
which, out = sys.argv[2], sys.argv[3]
if which == "cfg2":
    g = G.CONFIGS["cfg2"].graph()
    x = np.random.default_rng(7).standard_normal((5, 14, 101, 12)).astype(np.float32)
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
p = P.Plan(g, "bf16")
y = p.forward(x)
np.save(out, y)
print(json.dumps({"launches": p.launch_names()}))
"""


def _run(which, fused, tmp_path):
    out = str(tmp_path / f"{which}_{int(fused)}.npy")
    env = {**os.environ, "CNRX_BLK": "1" if fused else "0"}
    r = subprocess.run([sys.executable, "-c", ARM, ROOT, which, out], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out), json.loads(r.stdout.strip().splitlines()[-1])["launches"]


@pytest.mark.parametrize("which", ["cfg2", "dilated"])
def test_fused_block_kernel_is_bit_exact(which, tmp_path):
    yf, lf = _run(which, True, tmp_path)
    yu, lu = _run(which, False, tmp_path)
    assert any("conv_blk64" in n for n in lf), lf
    assert not any("conv_blk64" in n for n in lu), lu
    assert np.isfinite(yf).all()
    assert np.array_equal(yf, yu), (np.abs(yf - yu).max(), int((yf != yu).sum()))
