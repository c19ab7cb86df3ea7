"""Two receive passes of one config at batch B on cuda:0 (a fixed workload for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
from paper_2510_12739_b200 import graph as G, plan as P, slots
name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
cfg = G.CONFIGS[name]
B = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.batch
b = slots.generate(cfg.link, B, 1)
p = P.Plan(cfg.graph(), "bf16")
p.set_pilots(b.pilots, b.pilot_mask)
y = torch.from_numpy(b.y).cuda()
out = torch.empty((B, cfg.link.T, cfg.link.F, p.out_channels), device="cuda")
for _ in range(2):
    p.receive_device(y, out, 0)
torch.cuda.synchronize()
print("ok", name, B)
