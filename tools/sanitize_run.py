"""Small pass over every kernel family, meant to run under compute-sanitizer ("use
compute-sanitizer (racecheck/memcheck) on our kernels"):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_run.py [case ...]

Shapes are tiny (the sanitizer slows kernels 10-100x) but chosen so every launch has partial tiles, halo
rows on both sides and more than one CTA.  Each case also checks its LLRs against the oracle, so a run that
only "passes" because a kernel was skipped fails here.  Not a test and not a measurement.
"""
import dataclasses
import os
import sys

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
from paper_2510_12739_b200 import graph as G, plan as P, slots  # noqa: E402


def rel(a, b):
    return float(np.abs(a - b).max() / max(1e-12, np.abs(b).max()))


def receive_case(name, F, B, precs, opts=None):
    cfg = G.CONFIGS[name]
    link = dataclasses.replace(cfg.link, F=F)
    batch = slots.generate(link, B, seed=3)
    g = cfg.graph(seed=2)
    feat = oracle.featurize(batch.y, batch.pilots, batch.pilot_mask)
    ref = oracle.forward(g, feat)
    for prec in precs:
        p = P.Plan(g, prec, device=0, options=opts or {})
        p.set_pilots(batch.pilots, batch.pilot_mask)
        llr = p.receive(batch.y)
        r = rel(llr, ref)
        tol = {"fp32": 0.0, "bf16x3": 1e-4, "fp16x3": 1e-4, "fp16": 2e-2, "bf16": 1e-1}[prec]
        kinds = sorted({n.split("<")[0] for n in p.launch_names()})
        print(f"{name} F={F} B={B} {prec} {opts or ''}: rel {r:.2e} (tol {tol:g}) kernels {kinds}", flush=True)
        assert r <= tol, (name, prec, r)
        del p


CASES = {
    # fused-block program (conv_blk64), stem conv_tc, TMA head
    "cfg2": lambda: receive_case("cfg2", 40, 3, ["bf16", "fp16"]),
    # two-kernel program (conv_ws64)
    "cfg2_ws": lambda: receive_case("cfg2", 40, 2, ["bf16"], {"fused_blocks": 0}),
    # fused interaction + head epilogues
    "cfg2_fh": lambda: receive_case("cfg2", 40, 2, ["bf16"], {"fused_head": 1}),
    # split-precision kernels (conv_x3) and the fp32 CUDA-core plan
    "cfg2_x3": lambda: receive_case("cfg2", 40, 2, ["bf16x3", "fp32"]),
    # cfg1: narrow fp32 tile kernels, 32-ch conv_x3
    "cfg1": lambda: receive_case("cfg1", 72, 3, ["fp32", "bf16x3", "bf16"]),
    # 96-channel CTA-pair kernel (RB blocks, second pre-activated plane), 96-ch head
    "cfg4": lambda: receive_case("cfg4", 29, 2, ["bf16", "bf16x3"]),
    # cfg3: 4 subnets, dilation 2, 24 features, 6 bits
    "cfg3": lambda: receive_case("cfg3", 40, 1, ["bf16", "fp16"]),
}


def main():
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
    print("sanitize_run OK", flush=True)


if __name__ == "__main__":
    main()
