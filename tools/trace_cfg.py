"""CNRX_TRACE=1 python tools/trace_cfg.py cfg3 [B]: one receive of a config with per-role conv traces."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
from paper_2510_12739_b200 import graph as G, plan as P, slots
cfg = G.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
B = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.batch
b = slots.generate(cfg.link, B, 1)
p = P.Plan(cfg.graph(), cfg.precision); p.set_pilots(b.pilots, b.pilot_mask)
y = torch.from_numpy(b.y).cuda(); out = torch.empty((B, cfg.link.T, cfg.link.F, p.out_channels), device="cuda")
p.receive_device(y, out, 0); torch.cuda.synchronize()
print("second run", file=sys.stderr)
p.receive_device(y, out, 0); torch.cuda.synchronize()
