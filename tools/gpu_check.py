"""Diagnostics run on a B200 (not a test): parity numbers of every path + a first timing of cfg2."""
import os
import sys
import time

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import emulate_bf16 as E  # noqa: E402
from paper_2510_12739_b200 import graph as G, plan as P, slots  # noqa: E402


def rel(a, b):
    return float(np.abs(a - b).max() / max(1e-12, np.abs(b).max()))


def main():
    rng = np.random.default_rng(0)
    for name, shape in [("cfg1", (4, 14, 72, 6)), ("cfg2", (2, 14, 40, 12)), ("cfg4", (1, 14, 24, 12))]:
        g = G.CONFIGS[name].graph()
        x = rng.standard_normal(shape).astype(np.float32)
        ref = oracle.forward(g, x)
        t = time.time()
        pf = P.Plan(g, "fp32")
        y32 = pf.forward(x)
        print(f"{name} fp32: rel max err {rel(y32, ref):.3e}  launches {len(pf.launch_names())}  ({time.time()-t:.2f}s)")
        try:
            pb = P.Plan(g, "bf16")
            yb = pb.forward(x)
            em = E.emulate(g, x)
            print(f"{name} bf16: vs emu {rel(yb, em):.3e}  vs ref {rel(yb, ref):.3e}  sign agree vs ref "
                  f"{np.mean(np.sign(yb) == np.sign(ref)):.5f}  launches {pb.launch_names()}")
        except P.CnrxError as e:
            print(f"{name} bf16: {type(e).__name__}: {e}")
    # receive path
    cfg = G.CONFIGS["cfg2"]
    link = cfg.link
    g = cfg.graph()
    import dataclasses
    small = dataclasses.replace(link, F=48)
    batch = slots.generate(small, 3, 7)
    feat = oracle.featurize(batch.y, batch.pilots, batch.pilot_mask)
    ref = oracle.forward(g, feat)
    for prec in ("fp32", "bf16"):
        p = P.Plan(g, prec)
        p.set_pilots(batch.pilots, batch.pilot_mask)
        y = p.receive(batch.y)
        print(f"receive {prec}: rel err vs ref(featurize_oracle) {rel(y, ref):.3e}  sign agree {np.mean(np.sign(y)==np.sign(ref)):.5f}")
    # featurize alone
    import torch
    p = P.Plan(g, "fp32")
    p.set_pilots(batch.pilots, batch.pilot_mask)
    yd = torch.from_numpy(batch.y).cuda()
    fd = torch.empty(feat.shape, dtype=torch.float32, device="cuda")
    p.featurize_device(yd, fd)
    torch.cuda.synchronize()
    print(f"featurize: max abs err {np.abs(fd.cpu().numpy() - feat).max():.3e}")
    # timing cfg2 full size
    B = 256
    full = slots.generate(link, B, 1)
    pb = P.Plan(g, "bf16")
    pb.set_pilots(full.pilots, full.pilot_mask)
    yd = torch.from_numpy(full.y).cuda()
    out = torch.empty((B, 14, link.F, 4), dtype=torch.float32, device="cuda")
    for _ in range(3):
        pb.receive_device(yd, out, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 10
    for _ in range(n):
        pb.receive_device(yd, out, torch.cuda.current_stream().cuda_stream)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    flop = 2.0 * g.macs_per_re() * 14 * link.F * B
    print(f"cfg2 B=256 bf16 receive: {ms:.3f} ms/batch  {B/ms*1e3:.0f} slots/s  {flop/ms/1e9:.1f} TFLOP/s")
    print("launches:", pb.launch_names())
    # per-kernel timing via a graph-free loop per launch type is done by ncu; here a quick check of
    # parity at full size vs emulation on a few slots
    feat = oracle.featurize(full.y[:2], full.pilots, full.pilot_mask)
    em = E.emulate(g, feat)
    print(f"cfg2 full-F bf16 vs emu rel {rel(out[:2].cpu().numpy(), em):.3e}")


if __name__ == "__main__":
    main()
