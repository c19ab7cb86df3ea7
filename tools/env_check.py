"""Two environment variants of the bf16 plan on one config: bit-for-bit LLRs and whole-step time,
arms alternated `reps` times, each arm in its own process (plans read their switches when built).

    python tools/env_check.py cfg4 256 'CNRX_NO_PAIR=0' 'CNRX_NO_PAIR=1' [reps]
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
    print(json.dumps({"step_ms": e0.elapsed_time(e1) / 10, "launches": [(n, ms) for n, ms, c in p.read_profile()]}))


def main():
    if sys.argv[1] == "--arm":
        arm(sys.argv[2], int(sys.argv[3]), sys.argv[4])
        return
    name, B, ea, eb = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4]
    reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
    import numpy as np
    outs, steps = {}, {ea: [], eb: []}
    for _ in range(reps):
        for spec in (ea, eb):
            env = dict(os.environ)
            for kv in spec.split():
                k, _, v = kv.partition("=")
                env[k] = v
            out = f"/tmp/envchk_{abs(hash(spec))}.npy"
            r = subprocess.run([sys.executable, __file__, "--arm", name, str(B), out], env=env, capture_output=True,
                               text=True, timeout=900)
            if r.returncode != 0:
                print(spec, "FAILED\n", r.stdout[-2000:], r.stderr[-4000:])
                sys.exit(1)
            res = json.loads(r.stdout.strip().splitlines()[-1])
            steps[spec].append(res["step_ms"])
            outs[spec] = np.load(out)
            if len(steps[spec]) == 1:
                print(spec)
                for n, ms in res["launches"]:
                    print(f"   {n:40s} {ms * 1e3:8.1f} us")
    print("step ms:", {k: [round(x, 3) for x in v] for k, v in steps.items()})
    a, b = outs[ea], outs[eb]
    d = np.abs(a - b)
    print(f"bit-exact: {np.array_equal(a, b)}  max|diff| {d.max():.3e}  mismatches {(d > 0).sum()} / {d.size}  "
          f"finite {np.isfinite(a).all()}")


if __name__ == "__main__":
    main()
