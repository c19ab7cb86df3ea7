"""Minimal profiling target: a few forward steps of one BASELINE config at its batch (features input)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
from paper_2510_12739_b200 import graph as G, plan as P
name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
prec = sys.argv[2] if len(sys.argv) > 2 else G.CONFIGS[name].precision
B = int(sys.argv[3]) if len(sys.argv) > 3 else G.CONFIGS[name].batch
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
cfg = G.CONFIGS[name]
g = cfg.graph(seed=1)
p = P.Plan(g, prec, options={})
x = torch.randn((B, cfg.link.T, cfg.link.F, g.in_channels), device="cuda")
out = torch.empty((B, cfg.link.T, cfg.link.F, g.output_channels()), device="cuda")
for _ in range(steps):
    p.forward_device(x, out, 0)
torch.cuda.synchronize()
print("ok", p.launch_names())
