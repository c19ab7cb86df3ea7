"""fp32 (bit-exact CUDA-core) plan: device time per cfg2 batch, for A/B of the fp32 conv kernel."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import numpy as np
import torch
from paper_2510_12739_b200 import graph as G, plan as P, slots
cfg = G.CONFIGS["cfg2"]; B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
b = slots.generate(cfg.link, B, 1)
p = P.Plan(cfg.graph(seed=1), "fp32"); p.set_pilots(b.pilots, b.pilot_mask)
y = torch.from_numpy(b.y).cuda(); out = torch.empty((B, cfg.link.T, cfg.link.F, p.out_channels), device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(2): p.receive_device(y, out, st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); [p.receive_device(y, out, st) for _ in range(3)]; e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1) / 3
np.save(os.environ.get("F32_OUT", "/tmp/f32.npy"), out[:4].cpu().numpy())
print(f"fp32 B={B}: {ms:.2f} ms/batch, {B / ms * 1e3:.0f} slots/s, names={sorted(set(p.launch_names()))[:4]}")
