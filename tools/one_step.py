"""Minimal profiling target: a few cfg2 receive steps (B slots, default 256) on the given precision."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
from paper_2510_12739_b200 import graph as G, plan as P, slots
prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = G.CONFIGS["cfg2"]
b = slots.generate(cfg.link, B, 1)
p = P.Plan(cfg.graph(seed=1), prec, options={})
p.set_pilots(b.pilots, b.pilot_mask)
y = torch.from_numpy(b.y).cuda()
out = torch.empty((B, 14, cfg.link.F, 4), device="cuda")
for _ in range(steps):
    p.receive_device(y, out, 0)
torch.cuda.synchronize()
print("ok", p.launch_names())
