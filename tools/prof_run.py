"""Per-launch device times (CUDA events inside the library) for one config, averaged over a few runs."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
from paper_2510_12739_b200 import graph as G, plan as P, slots
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = G.CONFIGS[name]; g = cfg.graph(); B = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.batch
b = slots.generate(cfg.link, B, 1)
prec = os.environ.get("PREC") or (cfg.precision if hasattr(cfg, "precision") else "bf16")
p = P.Plan(g, prec); p.set_pilots(b.pilots, b.pilot_mask)
y = torch.from_numpy(b.y).cuda(); out = torch.empty((B, cfg.link.T, cfg.link.F, p.out_channels), device="cuda")
for _ in range(3):
    p.receive_device(y, out, 0)
torch.cuda.synchronize()
# whole-step time without per-kernel events (those would break programmatic dependent launches)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    p.receive_device(y, out, 0)
b.record()
b.synchronize()
step_ms = a.elapsed_time(b) / 10
p.set_profiling(True)
reps = 10
for _ in range(reps):
    p.receive_device(y, out, 0)
torch.cuda.synchronize()
tot = 0.0
for n, ms, c in p.read_profile():
    tot += ms / reps
    print(f"{n:40s} {ms / reps * 1e3:9.1f} us")
print(f"{'total (sum of kernels)':40s} {tot * 1e3:9.1f} us")
print(f"{'step':40s} {step_ms * 1e3:9.1f} us")
