"""B=1 cfg2 receive through a captured CUDA graph (the latency_b1 path), a few replays: a profiling target."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
from paper_2510_12739_b200 import graph as G, plan as P, slots
prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = G.CONFIGS["cfg2"]
b = slots.generate(cfg.link, 1, 1)
p = P.Plan(cfg.graph(seed=1), prec, options={})
p.set_pilots(b.pilots, b.pilot_mask)
p.set_graph_capture(True)
y = torch.from_numpy(b.y).cuda(); out = torch.empty((1, 14, cfg.link.F, 4), device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(reps):
    p.receive_device(y, out, s)
torch.cuda.synchronize()
a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
p.receive_device(y, out, s)
e.record(); e.synchronize()
print("graph replay ms", a.elapsed_time(e), p.launch_names())
