"""Minimal fused-block head run (debug target)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from paper_2510_12739_b200 import graph as G, plan as P
prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
F = int(sys.argv[2]) if len(sys.argv) > 2 else 37
g = G.CONFIGS["cfg2"].graph()
x = np.random.default_rng(7).standard_normal((2, 14, F, 12)).astype(np.float32)
p = P.Plan(g, prec, options={"fused_head": 1})
y = p.forward(x)
print("ok", p.launch_names(), float(np.abs(y).max()))
q = P.Plan(g, prec, options={"fused_head": 0})
print("same", np.array_equal(y, q.forward(x)))
