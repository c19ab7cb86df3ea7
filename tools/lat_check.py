"""B=1 device latency (CUDA-graph replay, p50 of 200) and small-batch step times for env variants of the
cfg2 bf16 plan, each variant in its own process.   python tools/lat_check.py 'A=' 'CNRX_BLK=1'"""
import json, os, statistics, subprocess, sys
HERE = os.path.dirname(os.path.abspath(__file__))


def arm():
    sys.path.insert(0, os.path.join(HERE, ".."))
    import torch
    from paper_2510_12739_b200 import graph as G, plan as P, slots
    cfg = G.CONFIGS["cfg2"]
    link = cfg.link
    b = slots.generate(link, 64, 1)
    res = {}
    for B in (1, 4, 16, 64):
        p = P.Plan(cfg.graph(seed=1), "bf16")
        p.set_pilots(b.pilots, b.pilot_mask)
        p.set_graph_capture(True)
        y = torch.from_numpy(b.y[:B].copy()).cuda()
        o = torch.empty((B, link.T, link.F, 4), device="cuda")
        s = torch.cuda.current_stream().cuda_stream
        for _ in range(5):
            p.receive_device(y, o, s)
        torch.cuda.synchronize()
        ts = []
        for _ in range(200 if B == 1 else 50):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            p.receive_device(y, o, s)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[B] = round(statistics.median(ts) * 1e3, 1)
        del p
    print(json.dumps(res))


if __name__ == "__main__":
    if sys.argv[1] == "--arm":
        arm()
    else:
        for rep in range(2):
            for spec in sys.argv[1:]:
                env = dict(os.environ)
                for kv in spec.split():
                    k, _, v = kv.partition("=")
                    if v:
                        env[k] = v
                r = subprocess.run([sys.executable, __file__, "--arm"], env=env, capture_output=True, text=True)
                print(f"{spec:20s} median us by B:", r.stdout.strip().splitlines()[-1] if r.returncode == 0 else r.stderr[-2000:])
