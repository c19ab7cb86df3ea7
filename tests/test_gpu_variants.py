"""Kernel variants against each other, bit for bit (each arm in its own process: the switches are read
when a plan is built):
  * the CTA-pair 96 -> 96 3x3 conv (csrc/conv_pair.cu, default) vs the single-CTA kernel
    (CNRX_NO_PAIR=1): same UMMA K order per output element, same epilogue -> identical LLRs;
  * the opt-in fused residual-block kernel (csrc/conv_blk.cu, CNRX_BLK=1) vs the default two-kernel
    path: conv1's output is rounded to bf16 at the same point in both -> identical LLRs;
  * the CoNet interaction + LLR head fused into the last convs' epilogue (conv_ws.cu kWsHead: clusters
    of one CTA per subnetwork exchanging tiles through distributed shared memory) vs the separate head
    kernel (CNRX_NO_HEADFUSE=1): same fold arithmetic, same bf16 z, same head UMMAs -> identical LLRs."""
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


def _run(which, fused, tmp_path, var="CNRX_BLK"):
    out = str(tmp_path / f"{which}_{var}_{int(fused)}.npy")
    env = {**os.environ, var: "1" if fused else "0"}
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


@pytest.mark.parametrize("which", ["cfg4", "dilated96"])
def test_cta_pair_conv_is_bit_exact_with_single_cta(which, tmp_path):
    yp, lp = _run(which, False, tmp_path, "CNRX_NO_PAIR")
    ys, ls = _run(which, True, tmp_path, "CNRX_NO_PAIR")
    assert any("conv_pair96" in n for n in lp), lp
    assert not any("conv_pair96" in n for n in ls), ls
    assert np.isfinite(yp).all()
    assert np.array_equal(yp, ys), (np.abs(yp - ys).max(), int((yp != ys).sum()))


@pytest.mark.parametrize("which", ["cfg2", "dilated"])
def test_fused_head_is_bit_exact_with_head_kernel(which, tmp_path):
    # two-kernel program in both arms (CNRX_BLK=0 is set by _run's "fused=False"), head fused or not
    out = {}
    for nohf in (False, True):
        o = str(tmp_path / f"{which}_hf{int(nohf)}.npy")
        env = {**os.environ, "CNRX_BLK": "0", "CNRX_HEADFUSE": "1"}
        if nohf:
            env["CNRX_NO_HEADFUSE"] = "1"
        r = subprocess.run([sys.executable, "-c", ARM, ROOT, which, o], env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        out[nohf] = (np.load(o), json.loads(r.stdout.strip().splitlines()[-1])["launches"])
    (yh, lh), (yk, lk) = out[False], out[True]
    assert any("<head>" in n for n in lh) and not any("head_tma" in n for n in lh), lh
    assert not any("<head>" in n for n in lk) and any("head_tma" in n for n in lk), lk
    assert np.isfinite(yh).all()
    assert np.array_equal(yh, yk), (np.abs(yh - yk).max(), int((yh != yk).sum()))
