"""Fused residual-block kernel (conv_blk.cu, CNRX_BLK=1) vs the default two-kernel path: bit-for-bit LLRs
and step time, one config.  Runs each arm in a subprocess (the env switch is read at plan compile).

    python tools/blk_check.py [cfg2] [B]
"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.join(HERE, "..")


def arm(name, B, out):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    from paper_2510_12739_b200 import graph as G, plan as P, slots
    cfg = G.CONFIGS[name]
    g = cfg.graph()
    b = slots.generate(cfg.link, B, 1)
    p = P.Plan(g, "bf16")
    p.set_pilots(b.pilots, b.pilot_mask)
    y = torch.from_numpy(b.y).cuda()
    o = torch.empty((B, cfg.link.T, cfg.link.F, p.out_channels), device="cuda")
    for _ in range(3):
        p.receive_device(y, o, 0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        p.receive_device(y, o, 0)
    e1.record()
    e1.synchronize()
    np.save(out, o.cpu().numpy())
    p.set_profiling(True)
    p.receive_device(y, o, 0)
    torch.cuda.synchronize()
    prof = [(n, ms) for n, ms, c in p.read_profile()]
    print(json.dumps({"step_ms": e0.elapsed_time(e1) / 10, "launches": prof}))


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--arm":
        arm(sys.argv[2], int(sys.argv[3]), sys.argv[4])
        return
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    import numpy as np
    res = {}
    reps = int(os.environ.get("BLK_REPS", "1"))
    steps = {"fused": [], "unfused": []}
    for tag, env in [a for _ in range(reps) for a in (("fused", {"CNRX_BLK": "1"}), ("unfused", {"CNRX_BLK": "0"}))]:
        out = f"/tmp/blk_{tag}.npy"
        r = subprocess.run([sys.executable, __file__, "--arm", name, str(B), out], env={**os.environ, **env},
                           capture_output=True, text=True, timeout=900)
        if r.returncode != 0:
            print(tag, "FAILED", r.stdout[-3000:], r.stderr[-3000:])
            sys.exit(1)
        res[tag] = json.loads(r.stdout.strip().splitlines()[-1])
        res[tag]["out"] = np.load(out)
        print(tag, f"step {res[tag]['step_ms']:.3f} ms")
        steps[tag].append(res[tag]["step_ms"])
        for n, ms in res[tag]["launches"]:
            print(f"   {n:40s} {ms * 1e3:8.1f} us")
    print("step ms (all reps):", {k: [round(x, 3) for x in v] for k, v in steps.items()})
    a, b = res["fused"]["out"], res["unfused"]["out"]
    same = np.array_equal(a, b)
    d = np.abs(a - b)
    print(f"bit-exact: {same}  max|diff| {d.max():.3e}  mismatches {(d > 0).sum()} / {d.size}  finite {np.isfinite(a).all()}")
    sys.exit(0 if same else 2)


if __name__ == "__main__":
    main()
