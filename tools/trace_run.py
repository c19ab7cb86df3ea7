"""Run one cfg2 forward with CNRX_TRACE=1 to print per-role cycle budgets of every conv launch."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
from paper_2510_12739_b200 import graph as G, plan as P, slots
cfg = G.CONFIGS["cfg2"]; g = cfg.graph(); B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
b = slots.generate(cfg.link, B, 1)
p = P.Plan(g, "bf16"); p.set_pilots(b.pilots, b.pilot_mask)
y = torch.from_numpy(b.y).cuda(); out = torch.empty((B, 14, cfg.link.F, 4), device="cuda")
p.receive_device(y, out, 0); torch.cuda.synchronize()
print("second run", file=sys.stderr)
p.receive_device(y, out, 0); torch.cuda.synchronize()
