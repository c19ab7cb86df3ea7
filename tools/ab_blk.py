"""A/B of library builds on one GPU (kernel experiments): each lib (path; 'default' = in-tree) runs in a
fresh process, interleaved `reps` times: cfg2 B=256 receive, 5 warm-up steps, then bursts of 20 steps
(CUDA events; 0.3 s apart so the clock starts each burst at boost) -> median ms/step, and the mean
per-launch time of each kernel from the library's profiling events.
usage: python tools/ab_blk.py reps lib1 [lib2 ...]   (env PREC=bf16|fp16, B=256)"""
import json
import os
import statistics
import subprocess
import sys

CHILD = r'''
import os, sys, time, json
sys.path.insert(0, os.environ["ROOT"])
import torch
from paper_2510_12739_b200 import graph as G, plan as P, slots
B = int(os.environ.get("B", "256")); prec = os.environ.get("PREC", "bf16")
cfg = G.CONFIGS["cfg2"]; b = slots.generate(cfg.link, B, 1)
opts = json.loads(os.environ.get("OPTS", "{}"))
p = P.Plan(cfg.graph(seed=1), prec, options=opts); p.set_pilots(b.pilots, b.pilot_mask)
y = torch.from_numpy(b.y).cuda(); out = torch.empty((B, 14, cfg.link.F, 4), device="cuda")
s = torch.cuda.Stream()
for _ in range(5): p.receive_device(y, out, s.cuda_stream)
torch.cuda.synchronize()
bursts = []
for k in range(5):
    time.sleep(0.3)
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(20): p.receive_device(y, out, s.cuda_stream)
    e.record(s); e.synchronize()
    bursts.append(a.elapsed_time(e) / 20)
time.sleep(0.3)
p.set_profiling(True); p.read_profile()
for _ in range(10): p.receive_device(y, out, s.cuda_stream)
torch.cuda.synchronize()
agg = {}
for n, ms, c in p.read_profile():
    a_ = agg.setdefault(n, [0.0, 0]); a_[0] += ms; a_[1] += c
import hashlib
sha = hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:12]
print(json.dumps({"ms_per_step": sorted(bursts)[len(bursts)//2], "min": min(bursts), "sha": sha,
                  "per_launch_us": {n: round(v[0] / v[1] * 1e3, 1) for n, v in agg.items()}}))
'''

reps = int(sys.argv[1])
libs = sys.argv[2:]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
res = {l: [] for l in libs}
for _ in range(reps):
    for l in libs:
        env = dict(os.environ, ROOT=root)
        lib, _, opt = l.partition("+")  # "lib+opt=1,opt2=0": plan options for this arm
        if lib != "default":
            env["CNRX_LIB"] = os.path.abspath(lib)
        env["OPTS"] = json.dumps({k: float(v) if "." in v else int(v) for k, v in (kv.split("=") for kv in opt.split(",") if kv)})
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        try:
            res[l].append(json.loads(r.stdout.strip().splitlines()[-1]))
        except Exception:
            print(l, "FAILED", r.stderr[-2000:], flush=True)
for l, rs in res.items():
    if not rs:
        continue
    ms = [r["ms_per_step"] for r in rs]
    blk = [r["per_launch_us"].get("conv_blk64_kernel") for r in rs]
    print(json.dumps({"lib": l, "ms_per_step_median": round(statistics.median(ms), 4), "ms_min": round(min(r["min"] for r in rs), 4),
                      "conv_blk_us_median": statistics.median([x for x in blk if x]) if any(blk) else None,
                      "llr_sha": sorted({r["sha"] for r in rs}),
                      "last": rs[-1]["per_launch_us"]}), flush=True)
