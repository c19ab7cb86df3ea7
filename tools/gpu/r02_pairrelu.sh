#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest tests/test_gpu_variants.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02_variants2.log 2>&1
echo "rc=$?" >> gpurun_out/r02_variants2.log
tail -3 gpurun_out/r02_variants2.log; grep -E "^E |FAILED" gpurun_out/r02_variants2.log | head -5
for o in 1 0; do
  echo "== relu_on_load=$o"
  for c in cfg3 cfg4; do
    OPTS="{\"relu_on_load\": $o}" timeout 300 python - $c <<'PY'
import os, sys, json, time
sys.path.insert(0, "."); import torch
from paper_2510_12739_b200 import graph as G, plan as P, slots
name = sys.argv[1]; cfg = G.CONFIGS[name]; g = cfg.graph(seed=1); B = cfg.batch
b = slots.generate(cfg.link, B, 1)
p = P.Plan(g, cfg.precision, options=json.loads(os.environ["OPTS"])); p.set_pilots(b.pilots, b.pilot_mask)
y = torch.from_numpy(b.y).cuda(); out = torch.empty((B, cfg.link.T, cfg.link.F, g.output_channels()), device="cuda")
for _ in range(3): p.receive_device(y, out, 0)
torch.cuda.synchronize(); ts = []
for _ in range(5):
    time.sleep(0.3); a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); p.receive_device(y, out, 0); e.record(); e.synchronize(); ts.append(a.elapsed_time(e))
p.set_profiling(True); p.read_profile(); p.receive_device(y, out, 0); torch.cuda.synchronize()
prof = p.read_profile()
pair = [round(ms * 1e3) for n, ms, c in prof if "pair" in n]
print(name, "ms/step", round(sorted(ts)[2], 3), "pair launches us", pair[:4], "...", len(pair))
PY
  done
done
