"""Device-resident BER sweep: slots generated on the GPU (cnrx_generate_slots), received by the plan and
scored on the GPU (cnrx_count_bit_errors) — nothing crosses PCIe but the per-slot error counts.

usage: python tools/ber_sweep.py [cfg2] [batches] [batch] [checkpoint.cnck [spec.json]]
Without a trained checkpoint the network has random weights and the BER sits near 0.5; the sweep is
then a throughput run of the whole device pipeline (generate + receive + count)."""
import dataclasses
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch

from paper_2510_12739_b200 import files as Fi, graph as G, plan as P, slots

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n_batches = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cfg = G.CONFIGS[name]
B = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.batch
if len(sys.argv) > 5:
    p = Fi.plan_from_files(sys.argv[5], sys.argv[4], cfg.precision)
elif len(sys.argv) > 4:  # a checkpoint of this config's own graph (e.g. tests/golden/cfg2_trained.cnck)
    g = cfg.graph_fn()
    Fi.load_checkpoint(g, sys.argv[4])
    p = P.Plan(g, cfg.precision)
else:
    p = P.Plan(cfg.graph(seed=1), cfg.precision)
pmask, pvals = slots.pilot_pattern(cfg.link.T, cfg.link.F, cfg.link.pilot_symbols, cfg.link.pilot_spacing)
p.set_pilots(pvals.astype(np.complex64), pmask)
data = torch.from_numpy(pmask == 0).cuda()
bins = np.linspace(cfg.link.snr_db[0], cfg.link.snr_db[1], 6)
llr = torch.empty((B, cfg.link.T, cfg.link.F, cfg.link.bits), dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
rows = []
t_total, slots_total = 0.0, 0
for lo, hi in zip(bins[:-1], bins[1:]):
    link = dataclasses.replace(cfg.link, snr_db=(float(lo), float(hi)))
    errs, nbits, e_ls, e_pc = 0, 0, 0, 0
    for k in range(n_batches + 1):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        y, bits = P.generate_slots_device(link, B, seed=2024, slot0=k * B)
        p.receive_device(y, llr, st)
        e = P.count_bit_errors(llr, bits, data)
        b.record()
        b.synchronize()
        if k == 0:
            continue  # warm-up
        t_total += a.elapsed_time(b) * 1e-3
        slots_total += B
        errs += int(e.sum().item())
        nbits += B * int(pmask.size - pmask.sum()) * cfg.link.bits
        # classical baselines on the same slots: LS-LMMSE and perfect-CSI LMMSE
        yh, _, hh = P.generate_slots_device(link, B, seed=2024, slot0=k * B, with_h=True)
        nv = P.slot_noise_var(link, B, 2024, k * B)
        e_ls += int(P.count_bit_errors(P.classical_receive_device(p, yh, nv, link.mod_order), bits, data).sum())
        e_pc += int(P.count_bit_errors(P.classical_receive_device(p, yh, nv, link.mod_order, h=hh), bits,
                                       data).sum())
    rows.append({"snr_db": [float(lo), float(hi)], "ber": errs / nbits, "ber_ls_lmmse": e_ls / nbits,
                 "ber_perfect_csi_lmmse": e_pc / nbits, "bits": nbits})
print(json.dumps({"config": name, "batch": B, "device_pipeline_slots_per_s": slots_total / t_total,
                  "note": "network: random weights unless a checkpoint is given; LMMSE baselines on the same slots", "sweep": rows}))
