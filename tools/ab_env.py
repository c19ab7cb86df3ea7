"""A/B timing of environment-variable variants of the plan on one GPU: each variant's whole receive step
is timed in a fresh process (plans read their env switches at build time), interleaved, reps times;
prints min / median ms.  usage: python tools/ab_env.py reps 'A=' 'CNRX_NO_RELU_IN=1' ..."""
import os
import statistics
import subprocess
import sys

reps = int(sys.argv[1])
variants = sys.argv[2:]
here = os.path.dirname(os.path.abspath(__file__))
res = {v: [] for v in variants}
for _ in range(reps):
    for v in variants:
        env = dict(os.environ)
        for kv in v.split():
            k, _, val = kv.partition("=")
            if val:
                env[k] = val
        out = subprocess.run([sys.executable, os.path.join(here, "prof_run.py")], env=env, capture_output=True,
                             text=True).stdout
        tot = [l for l in out.splitlines() if l.startswith("step")]
        res[v].append(float(tot[-1].split()[1]) / 1e3)
for v, xs in res.items():
    print(f"{v:40s} min {min(xs):.3f} ms  median {statistics.median(xs):.3f} ms  ({len(xs)} runs)")
