"""Depth / latency study (SPEC.md:485-493 `bench_depth_latency`): CoNet-14 vs
DeepRx-24 at a matched parameter budget, solved with the reference's width solver (files.py), on the
GPU plan.

Reports param counts, sequential conv depths (network.hpp:320-330), the depth ratio, and the measured
single-slot (B=1, one TTI) forward latency — median and interquartile range over >= 100 runs, device
time of a CUDA-graph replay, subnets of a stage executed concurrently (grouped launches) — plus batch
throughput.  usage: python tools/depth_latency.py [P=1900000] [precision=fp32|bf16|fp16|bf16x3] [runs=200] [io_kernel=3]"""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np

from paper_2510_12739_b200 import files as Fi

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1_900_000
prec = sys.argv[2] if len(sys.argv) > 2 else "fp32"
runs = int(sys.argv[3]) if len(sys.argv) > 3 else 200
# io_kernel 3 (default): the spec-file templates (3x3 stem/head, as the paper's networks); 1: 1x1 stem/head as
# in the BASELINE configs (NetSpec.kernel = 1, BlockSpec.kernel = 3).  Every plan precision lowers both.
io_kernel = int(sys.argv[4]) if len(sys.argv) > 4 else 3
T, F, C_IN, BITS = 14, 612, 12, 4  # cfg2 grid and features

SPECS = {
    # 6 MRBs per subnet: stem + 12 block convs + head = 14 sequential convs
    "CoNet-14": {"template": "conet", "main_blocks": 6, "support_blocks": [6], "fusion_op": "mul",
                 "fusion_norm": "bn", "in_channels": C_IN, "bits": BITS, "kernel": 3},
    # 11 RBs: stem + 22 block convs + head = 24 sequential convs
    "DeepRx-24": {"template": "deeprx", "blocks": 11, "in_channels": C_IN, "bits": BITS, "kernel": 3},
}


def measure(g, B, reps, graph):
    import torch
    from paper_2510_12739_b200 import plan as Pl
    p = Pl.Plan(g, prec)
    x = torch.randn((B, T, F, C_IN), device="cuda")
    out = torch.empty((B, T, F, BITS), device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    p.set_graph_capture(graph)
    for _ in range(5):
        p.forward_device(x, out, st)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        p.forward_device(x, out, st)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    measure.kernels = sorted(set(p.launch_names()))
    p.close()
    return np.array(ts)


def build(f, w, shape_only=False):
    from paper_2510_12739_b200 import graph as G
    f = f.with_width(w)
    if f.is_conet():
        spec = f.to_conet()
        for ns in [spec.main] + spec.supports:
            ns.kernel = io_kernel
        return G.build_conet(spec, shape_only=shape_only)
    spec = f.to_deeprx()
    spec.kernel = io_kernel
    return G.build_net(spec, shape_only=shape_only)


rows = {}
for name, spec in SPECS.items():
    f = Fi.parse_spec_file_json(json.dumps(spec))
    r = Fi.solve_filters(lambda w: build(f, w, True).learnable_count(), P)
    if not r.found:
        raise SystemExit(f"{name}: {r.diagnostic}")
    g = build(f, r.width)
    g.init_he_normal(1, randomize_aux=True)
    row = {"width": r.width, "params": g.learnable_count(), "conv_depth": g.conv_depth(),
           "macs_per_re": g.macs_per_re()}
    try:
        lat = measure(g, 1, runs, True)
        thr = measure(g, 64, 20, False)
        row.update({"latency_b1_ms": {"median": float(np.median(lat)), "p25": float(np.percentile(lat, 25)),
                                      "p75": float(np.percentile(lat, 75)), "runs": runs},
                    "throughput_b64_slots_per_s": float(64 / (np.median(thr) * 1e-3)),
                    "kernels_b64": measure.kernels})
    except Exception as e:  # no GPU / unsupported lowering: graph properties only
        row["measure_error"] = str(e)
    rows[name] = row
c, d = rows["CoNet-14"], rows["DeepRx-24"]
rep = {"budget_params": P, "precision": prec, "io_kernel": io_kernel, "grid": [T, F], "in_channels": C_IN, "bits": BITS, "nets": rows,
       "depth_reduction": 1 - c["conv_depth"] / d["conv_depth"]}
if "latency_b1_ms" in c and "latency_b1_ms" in d:
    rep["latency_reduction_b1"] = 1 - c["latency_b1_ms"]["median"] / d["latency_b1_ms"]["median"]
print(json.dumps(rep, indent=1))
