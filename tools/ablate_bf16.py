"""Ablate the bf16 plan's rounding points on the TRAINED cfg2 checkpoint (CPU, torch).

For each variant, one or more roles of tests/emulate_bf16.BF16_POLICY get a different rounding
function (identity = fp32, fp16, bf16); hard decisions on data bits are compared with the fp32
forward (all roles identity) on the same host-generated slots.  Prints one JSON line per variant.

usage: python tools/ablate_bf16.py [B=32] [seed=7]"""
import json
import os
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch

import emulate_bf16 as E
import oracle
from paper_2510_12739_b200 import files as Fi, graph as G, slots

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 7
torch.set_num_threads(os.cpu_count())
g = G.CONFIGS["cfg2"].graph_fn()
Fi.load_checkpoint(g, os.path.join(ROOT, "tests", "golden", "cfg2_trained.cnck"))
link = G.CONFIGS["cfg2"].link
ident = E._ident
fp32 = {k: ident for k in E.BF16_POLICY}
variants = {
    "bf16 (shipped)": {},
    "fp32 feat": dict(feat=ident),
    "fp32 w": dict(w=ident),
    "fp32 act": dict(act=ident),
    "fp32 res": dict(res=ident),
    "fp32 leaf": dict(leaf=ident),
    "fp32 z": dict(z=ident),
    "fp32 res+leaf+z": dict(res=ident, leaf=ident, z=ident),
    "fp32 res+leaf+z+feat": dict(res=ident, leaf=ident, z=ident, feat=ident),
    "fp32 all but act": dict(res=ident, leaf=ident, z=ident, feat=ident, w=ident),
    "fp32 all but w": dict(res=ident, leaf=ident, z=ident, feat=ident, act=ident),
    "fp16 all": {k: E.fp16 for k in E.BF16_POLICY},
    "fp16 act+w, fp32 rest": dict(act=E.fp16, w=E.fp16, feat=E.fp16, res=ident, leaf=ident, z=ident),
}
only = os.environ.get("ABL_ONLY")
chunks = []
for c0 in range(0, B, 8):
    b = slots.generate(link, min(8, B - c0), seed * 1000 + c0)
    feat = oracle.featurize(b.y, b.pilots, b.pilot_mask)
    chunks.append((b, feat))
ref = [E.emulate(g, f, fp32) for _, f in chunks]
for name, pol in variants.items():
    if only and only not in name:
        continue
    agree = n = e_v = e_r = 0
    for (b, f), r in zip(chunks, ref):
        v = E.emulate(g, f, pol)
        m = b.data_mask
        rv, vv, tb = r[:, m], v[:, m], b.bits[:, m]
        agree += int(((rv > 0) == (vv > 0)).sum())
        n += rv.size
        e_v += int(((vv > 0) != tb).sum())
        e_r += int(((rv > 0) != tb).sum())
    print(json.dumps({"variant": name, "agree": agree / n, "bits": n, "flips": n - agree,
                      "ber": e_v / n, "ber_fp32": e_r / n}), flush=True)
