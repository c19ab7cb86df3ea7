"""Bounds check of every kernel family ("use compute-sanitizer (racecheck/memcheck) on our
kernels").  compute-sanitizer is closed on this GPU pool, so the plans run with their own guard bands
(cnrx_plan_set_guard_bands: 256 KB canaries either side of every workspace buffer) and the caller's input /
output buffers sit inside canary-filled torch allocations:

    python tools/sanitize_run.py [case ...]          (tools/sanitize.sh adds compute-sanitizer where open)

Shapes are small but chosen so every launch has partial tiles, halo rows on both sides and more than one
CTA.  Each case also checks its LLRs against the oracle, so a run that only "passes" because a kernel was
skipped fails here.  Not a measurement; tests/test_gpu_guard.py runs the same cases in the GPU suite.
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
    import torch
    results = []
    for prec in precs:
        p = P.Plan(g, prec, device=0, options=opts or {})
        p.set_guard_bands(True)
        p.set_pilots(batch.pilots, batch.pilot_mask)
        # caller buffers inside canary-filled allocations (device entry point)
        pad = 1 << 16
        yin = torch.from_numpy(np.ascontiguousarray(batch.y))
        if yin.is_complex():
            yin = torch.view_as_real(yin)  # [B,T,F,N,2] fp32
        ybuf = torch.full((yin.numel() + 2 * pad,), float("nan"), dtype=torch.float32, device="cuda")
        ybuf[pad:pad + yin.numel()] = yin.reshape(-1).cuda()
        n_out = int(np.prod(ref.shape))
        obuf = torch.full((n_out + 2 * pad,), 12345.0, dtype=torch.float32, device="cuda")
        yv = ybuf[pad:pad + yin.numel()].view(yin.shape)
        ov = obuf[pad:pad + n_out].view(ref.shape)
        for b in (B, 1, B):  # regrow / shrink / reuse of the workspace
            p.receive_device(yv[:b], ov[:b], torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        llr = ov.cpu().numpy()
        assert bool((obuf[:pad] == 12345.0).all()) and bool((obuf[pad + n_out:] == 12345.0).all()), "write outside llr"
        llr_host = p.receive(batch.y)  # host entry point: staging buffers are guarded too
        assert np.array_equal(llr_host, llr), "host / device entry points differ"
        nbuf, bad = p.check_guard_bands()
        r = rel(llr, ref)
        # fp32: the GPU featurizer is within 1e-5 of the restated one (tests/test_gpu_featurize.py); the
        # forward itself is bit-exact on equal features
        tol = {"fp32": 1e-5, "bf16x3": 1e-4, "fp16x3": 1e-4, "fp16": 2e-2, "bf16": 1e-1}[prec]
        kinds = sorted({n.split("<")[0] for n in p.launch_names()})
        print(f"{name} F={F} B={B} {prec} {opts or ''}: rel {r:.2e} (tol {tol:g}) guarded buffers {nbuf} "
              f"bad canary bytes {bad} kernels {kinds}", flush=True)
        assert r <= tol, (name, prec, r)
        assert nbuf > 0 and bad == 0, (name, prec, nbuf, bad)
        results.append((prec, nbuf, bad, kinds))
        del p
    return results


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
    # cfg2 at its full 612-subcarrier grid, odd batch (multi-wave grids, partial last tiles)
    "cfg2_full": lambda: receive_case("cfg2", 612, 3, ["bf16"]),
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
