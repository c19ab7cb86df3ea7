"""A/B of the fp32 conv kernels (CNRX_F32_TILE=0|1 is read once per process): per config, median
forward_device time over 30 runs and a sha256 of the LLRs (the two kernels must agree bit for bit).

    python tools/f32_ab.py [arm ...]   # CNRX_F32_TILE values (default 0 1); runs the arms in subprocesses, prints one JSON line per arm
"""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
CASES = [("cfg1", 64), ("cfg1", 1), ("cfg2", 16), ("cfg4", 8)]


def arm():
    sys.path.insert(0, ROOT)
    import torch
    from paper_2510_12739_b200 import graph as G, plan as P
    res = {}
    for name, B in CASES:
        cfg = G.CONFIGS[name]
        g = cfg.graph(seed=1)
        p = P.Plan(g, "fp32", options={})
        gen = torch.Generator(device="cuda").manual_seed(5)
        x = torch.randn((B, cfg.link.T, cfg.link.F, g.in_channels), device="cuda", generator=gen)
        out = torch.empty((B, cfg.link.T, cfg.link.F, g.output_channels()), device="cuda")
        for _ in range(3):
            p.forward_device(x, out, 0)
        torch.cuda.synchronize()
        ts = []
        for _ in range(30):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            p.forward_device(x, out, 0)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        names = sorted(set(n for n in p.launch_names() if "conv" in n))
        res[f"{name}_b{B}"] = {"ms": ts[len(ts) // 2], "sha": hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()[:16],
                               "kernels": names}
    print(json.dumps({"tile": os.environ.get("CNRX_F32_TILE", "1"), **res}))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "arm":
        arm()
    else:
        outs = []
        arms = sys.argv[1:] or ["0", "1"]
        for t in arms:
            r = subprocess.run([sys.executable, __file__, "arm"], env={**os.environ, "CNRX_F32_TILE": t},
                               capture_output=True, text=True)
            print(r.stdout.strip() or r.stderr[-2000:])
            outs.append(json.loads(r.stdout) if r.returncode == 0 else None)
        if all(outs):
            for k in outs[0]:
                if k != "tile":
                    same = all(o[k]["sha"] == outs[0][k]["sha"] for o in outs)
                    print(k, "same" if same else "DIFFERENT", " / ".join(f"{o['tile']}: {o[k]['ms']:.3f}" for o in outs), "ms")
