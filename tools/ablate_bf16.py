"""Ablate the bf16 / fp16 plans' rounding points on a TRAINED checkpoint (CPU, torch).

For each variant, one or more roles of tests/emulate_bf16.BF16_POLICY get a different rounding
function (identity = fp32, fp16, bf16); hard decisions on data bits are compared with the fp32
forward (all roles identity) on the same host-generated slots.  Prints one JSON line per variant.

usage: python tools/ablate_bf16.py [B=32] [seed=7]   (env CFG=cfg2|cfg3, FCROP=<subcarriers>: score the
interior of a subcarrier crop, margin = the receptive radius, to bound the CPU cost of cfg3)"""
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
CFG = os.environ.get("CFG", "cfg2")
FCROP = int(os.environ.get("FCROP", "0"))
g = G.CONFIGS[CFG].graph_fn()
Fi.load_checkpoint(g, os.path.join(ROOT, "tests", "golden", f"{CFG}_trained.cnck"))
link = G.CONFIGS[CFG].link
MARGIN = 2 * sum(1 for n in g.nodes if n.op == G.OP_CONV and g.params[n.w].value.shape[0] == 3) + 2
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
    "fp16 (shipped: z fp32)": dict(E.FP16_POLICY),
    "fp16, fp32 res": dict(E.FP16_POLICY, res=ident),
    "fp16, fp32 leaf": dict(E.FP16_POLICY, leaf=ident),
    "fp16, fp32 feat": dict(E.FP16_POLICY, feat=ident),
    "fp16, fp32 w": dict(E.FP16_POLICY, w=ident),
    "fp16, fp32 act": dict(E.FP16_POLICY, act=ident),
    "fp16, fp32 res+leaf": dict(E.FP16_POLICY, res=ident, leaf=ident),
    "fp16, fp32 feat+leaf": dict(E.FP16_POLICY, feat=ident, leaf=ident),
    "fp16, fp32 feat+res": dict(E.FP16_POLICY, feat=ident, res=ident),
    "fp16, fp32 feat+res+leaf": dict(E.FP16_POLICY, feat=ident, res=ident, leaf=ident),
    "fp16x2 split operands (3-pass)": dict(feat=E.fp16x2, w=E.fp16x2, act=E.fp16x2, res=E.fp16x2, leaf=E.fp16x2, z=ident),
    "bf16x2 split operands (3-pass)": dict(feat=E.bf16x2, w=E.bf16x2, act=E.bf16x2, res=E.bf16x2, leaf=E.bf16x2, z=ident),
    "bf16x2 split operands, fp32 planes": dict(feat=ident, w=E.bf16x2, act=E.bf16x2, res=ident, leaf=ident, z=ident),
    "fp16 act, fp16x2 w (2-pass), fp32 planes": dict(feat=E.fp16, w=E.fp16x2, act=E.fp16, res=ident, leaf=ident, z=ident),
    "fp16x2 act, fp16 w (2-pass), fp32 planes": dict(feat=E.fp16x2, w=E.fp16, act=E.fp16x2, res=ident, leaf=ident, z=ident),
    "fp16 act+w, fp32 planes": dict(feat=E.fp16, w=E.fp16, act=E.fp16, res=ident, leaf=ident, z=ident),
}
only = os.environ.get("ABL_ONLY")
chunks = []
for c0 in range(0, B, 8):
    b = slots.generate(link, min(8, B - c0), seed * 1000 + c0)
    feat = oracle.featurize(b.y, b.pilots, b.pilot_mask)
    if FCROP and FCROP < link.F:  # crop + score only the interior (bits outside are dropped below)
        f0 = (link.F - FCROP) // 2
        feat = np.ascontiguousarray(feat[:, :, f0:f0 + FCROP])
        keep = np.zeros(b.data_mask.shape, bool)
        keep[:, f0 + MARGIN:f0 + FCROP - MARGIN] = True
        b.bits = b.bits[:, :, f0:f0 + FCROP]
        b.data_mask = (b.data_mask & keep)[:, f0:f0 + FCROP]
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
