"""Diagnostics: isolate bf16 conv accuracy on tiny graphs and time cfg2 on the right stream."""
import os
import sys

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import emulate_bf16 as E  # noqa: E402
from paper_2510_12739_b200 import graph as G, plan as P, slots  # noqa: E402


def stats(a, b):
    d = np.abs(a - b)
    s = np.abs(b).max()
    return f"max {d.max()/s:.2e} p99 {np.quantile(d, 0.99)/s:.2e} med {np.median(d)/s:.2e} argmax {np.unravel_index(d.argmax(), d.shape)}"


def tiny(kind, cin=12, c=64, F=40, B=2, dil=1):
    g = G.Graph()
    x = g.add_input(cin)
    if kind == "1x1":
        h = g.add_relu(g.add_conv(x, "a", 1, cin, c, True))
    elif kind == "3x3":
        s = g.add_relu(g.add_conv(x, "s", 1, cin, c, True))
        h = g.add_relu(g.add_conv(s, "a", 3, c, c, True, dilation_f=dil))
    elif kind == "res":
        s = g.add_relu(g.add_conv(x, "s", 1, cin, c, True))
        h1 = g.add_relu(g.add_conv(s, "a", 3, c, c, True, dilation_f=dil))
        h = g.add_binary(G.OP_ADD, g.add_conv(h1, "b", 3, c, c, True, dilation_f=dil), s)
    g.set_output(g.add_conv(h, "out", 1, c, 4, True))
    g.init_he_normal(3, randomize_aux=True)
    xin = np.random.default_rng(1).standard_normal((B, 14, F, cin)).astype(np.float32)
    return g, xin


def main():
    import torch
    for kind, dil, c in [("1x1", 1, 64), ("3x3", 1, 64), ("res", 1, 64), ("3x3", 2, 64), ("3x3", 1, 96), ("res", 2, 96)]:
        g, x = tiny(kind, c=c, dil=dil)
        pb = P.Plan(g, "bf16")
        yb = pb.forward(x)
        em = E.emulate(g, x)
        print(f"{kind} dil{dil} c{c}: gpu vs emu {stats(yb, em)}")
    # timing on torch's stream
    cfg = G.CONFIGS["cfg2"]
    link = cfg.link
    g = cfg.graph()
    B = 256
    full = slots.generate(link, B, 1)
    pb = P.Plan(g, "bf16")
    pb.set_pilots(full.pilots, full.pilot_mask)
    yd = torch.from_numpy(full.y).cuda()
    out = torch.empty((B, 14, link.F, 4), dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        pb.receive_device(yd, out, st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    e0.record()
    for _ in range(n):
        pb.receive_device(yd, out, st)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    flop = 2.0 * g.macs_per_re() * 14 * link.F * B
    print(f"cfg2 B=256 bf16 receive: {ms:.3f} ms/batch  {B/ms*1e3:.0f} slots/s  {flop/ms/1e9:.1f} TFLOP/s")


if __name__ == "__main__":
    main()
