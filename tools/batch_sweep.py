"""cfg5: cfg2 shapes over batch sizes, bf16 and fp32 — device time per batch (median of
reps, inputs resident in HBM, CUDA events on the launching stream), slots/s and per-slot cost.
usage: python tools/batch_sweep.py [max_B_bf16=8192] [max_B_fp32=512]"""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch

from paper_2510_12739_b200 import graph as G, plan as P, slots

max16 = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
max32 = int(sys.argv[2]) if len(sys.argv) > 2 else 512
cfg = G.CONFIGS["cfg2"]
link = cfg.link
g = cfg.graph(seed=1)
pmask, pvals = slots.pilot_pattern(link.T, link.F, link.pilot_symbols, link.pilot_spacing)
rows = []
for prec, maxb in (("bf16", max16), ("fp32", max32)):
    p = P.Plan(g, prec)
    p.set_pilots(pvals.astype(np.complex64), pmask)
    B = 1
    while B <= maxb:
        y, _ = P.generate_slots_device(link, B, 3)
        out = torch.empty((B, link.T, link.F, p.out_channels), device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        p.set_graph_capture(B <= 16)  # launch-bound small batches replay a CUDA graph
        for _ in range(3):
            p.receive_device(y, out, st)
        torch.cuda.synchronize()
        reps = 20 if B <= 1024 else 5
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            p.receive_device(y, out, st)
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        ms = float(np.median(ts))
        rows.append({"precision": prec, "B": B, "ms_per_batch": ms, "slots_per_s": B / ms * 1e3,
                     "us_per_slot": ms * 1e3 / B})
        print(json.dumps(rows[-1]), flush=True)
        del y, out
        B *= 4 if B < 4096 else 2
    p.close()
    torch.cuda.empty_cache()
print(json.dumps({"config": "cfg5 (cfg2 shapes)", "sweep": rows}))
