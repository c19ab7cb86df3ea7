"""Train a BASELINE network on GPU-generated slots to obtain TRAINED weights (a CNCK checkpoint) for the
hard-decision / BER parity claims.  Not part of the product path: PyTorch autograd interprets the same
GraphNode list the plan compiles (training is out of scope for the engine), the data come from
the device slot generator + featurizer (cnrx_generate_slots / cnrx_featurize_device), and the trained
parameters are written in the reference's checkpoint format (files.save_checkpoint).

Eval-mode BN is kept as the reference's eval affine with running statistics rm = 0, rv = 1 (the
learnable gains / shifts are trained), so the checkpoint's BN flags are all "ready".

usage: python tools/train_cfg.py [cfg2] [steps=1500] [batch=16] [out=tests/golden/cfg2_trained.cnck]
prints one JSON line: loss curve summary, BER of the trained network vs LS-LMMSE / perfect-CSI LMMSE,
and the bf16-vs-fp32 hard-decision agreement of the B200 plans on held-out slots."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch
import torch.nn.functional as Fn

from paper_2510_12739_b200 import files as Fi, graph as G, plan as P, slots

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1500
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 16
out_path = sys.argv[4] if len(sys.argv) > 4 else os.path.join("tests", "golden", f"{name}_trained.cnck")
cfg = G.CONFIGS[name]
link = cfg.link
dev = torch.device("cuda")
torch.manual_seed(0)

g = cfg.graph(seed=1)  # He-normal init
g.seed_norm_stats()
for p in g.params:  # biases / BN shifts start at zero, gains at one
    if p.name.endswith(".b") or p.name.endswith(".s"):
        p.value[:] = 0
    if p.name.endswith(".g"):
        p.value[:] = 1

# torch parameters in NCHW conv layout; BN running stats stay fixed (0 / 1)
tp = {}
for i, p in enumerate(g.params):
    v = torch.from_numpy(np.array(p.value)).to(dev)
    owner = g.weight_owner(i)
    if owner is not None and owner.op == G.OP_CONV:
        v = v.permute(3, 2, 0, 1).contiguous()  # [kh,kw,cin,cout] -> [cout,cin,kh,kw]
    tp[i] = torch.nn.Parameter(v, requires_grad=p.learnable)
lr = float(os.environ.get("LR", "2e-3"))
clip = float(os.environ.get("CLIP", "0"))  # global grad-norm clip (0: off); cfg3's 4-way product needs it
opt = torch.optim.Adam([v for v in tp.values() if v.requires_grad], lr=lr)
sched = torch.optim.lr_scheduler.CosineAnnealingLR(opt, steps)


def run(x):
    """x: [B,C,T,F] -> LLRs [B,bits,T,F] following g.nodes (network.hpp:380-420 semantics, eval BN)."""
    vals = {}
    for i, n in enumerate(g.nodes):
        a = vals.get(n.in0)
        if n.op == G.OP_INPUT:
            v = x
        elif n.op == G.OP_CONV:
            w = tp[n.w]
            kh = w.shape[2]
            v = Fn.conv2d(a, w, tp[n.b] if n.b >= 0 else None, padding=(kh // 2, (kh // 2) * n.dilation_f),
                          dilation=(1, n.dilation_f))
        elif n.op == G.OP_RELU:
            v = torch.relu(a)
        elif n.op == G.OP_BN:
            scale = tp[n.gamma] / torch.sqrt(tp[n.rvar] + 1e-5)
            v = (a - tp[n.rmean][None, :, None, None]) * scale[None, :, None, None] + tp[n.beta][None, :, None, None]
        elif n.op == G.OP_ADD:
            v = a + vals[n.in1]
        elif n.op == G.OP_MUL:
            v = a * vals[n.in1]
        else:
            raise SystemExit(f"op {n.op} not supported by the trainer")
        vals[i] = v
    return vals[g.output_node]


pmask, pvals = slots.pilot_pattern(link.T, link.F, link.pilot_symbols, link.pilot_spacing)
feat_plan = P.Plan(g, "fp32")
feat_plan.set_pilots(pvals.astype(np.complex64), pmask)
data = torch.from_numpy(pmask == 0).to(dev)
C_in = g.in_channels
losses = []
t0 = time.time()
for step in range(steps):
    y, bits = P.generate_slots_device(link, batch, seed=7, slot0=step * batch)
    feat = torch.empty((batch, link.T, link.F, C_in), dtype=torch.float32, device=dev)
    feat_plan.featurize_device(y, feat, torch.cuda.current_stream().cuda_stream)
    x = feat.permute(0, 3, 1, 2)
    with torch.autocast("cuda", dtype=torch.bfloat16):
        llr = run(x).float().permute(0, 2, 3, 1)  # [B,T,F,bits]
    loss = Fn.binary_cross_entropy_with_logits(llr[:, data], bits[:, data].float())
    opt.zero_grad(set_to_none=True)
    loss.backward()
    if clip > 0:
        torch.nn.utils.clip_grad_norm_([v for v in tp.values() if v.requires_grad], clip)
    opt.step()
    sched.step()
    if step % 50 == 0 or step == steps - 1:
        losses.append((step, float(loss.detach())))
train_s = time.time() - t0

# export -> checkpoint
for i, p in enumerate(g.params):
    v = tp[i].detach()
    owner = g.weight_owner(i)
    if owner is not None and owner.op == G.OP_CONV:
        v = v.permute(2, 3, 1, 0)
    p.value = v.float().cpu().numpy().copy()
g.bn_ready = [1] * len(g.bn_ready)
os.makedirs(os.path.dirname(out_path) or ".", exist_ok=True)
Fi.save_checkpoint(g, out_path)

# held-out evaluation on the B200 plans
p32, p16, ph = P.Plan(g, "fp32"), P.Plan(g, "bf16"), P.Plan(g, "fp16")
for p in (p32, p16, ph):
    p.set_pilots(pvals.astype(np.complex64), pmask)
n_eval, agree, agree_h, tot = max(8, 64 // batch), 0, 0, 0
err = {"net_bf16": 0, "net_fp16": 0, "net_fp32": 0, "ls_lmmse": 0, "perfect_csi_lmmse": 0}
nbits = 0
for k in range(n_eval):
    y, bits, h = P.generate_slots_device(link, batch, seed=99, slot0=k * batch, with_h=True)
    l32 = torch.empty((batch, link.T, link.F, link.bits), dtype=torch.float32, device=dev)
    l16 = torch.empty_like(l32)
    lh = torch.empty_like(l32)
    st = torch.cuda.current_stream().cuda_stream
    p32.receive_device(y, l32, st)
    p16.receive_device(y, l16, st)
    ph.receive_device(y, lh, st)
    err["net_fp16"] += int(P.count_bit_errors(lh, bits, data).sum())
    nv = P.slot_noise_var(link, batch, 99, k * batch)
    err["net_fp32"] += int(P.count_bit_errors(l32, bits, data).sum())
    err["net_bf16"] += int(P.count_bit_errors(l16, bits, data).sum())
    err["ls_lmmse"] += int(P.count_bit_errors(P.classical_receive_device(p32, y, nv, link.mod_order), bits, data).sum())
    err["perfect_csi_lmmse"] += int(P.count_bit_errors(P.classical_receive_device(p32, y, nv, link.mod_order, h=h),
                                                       bits, data).sum())
    m = data[None, :, :, None].expand_as(l32)
    agree += int(((l32 > 0) == (l16 > 0))[m].sum())
    agree_h += int(((l32 > 0) == (lh > 0))[m].sum())
    tot += int(m.sum())
    nbits += batch * int(data.sum()) * link.bits
print(json.dumps({"config": name, "steps": steps, "batch": batch, "train_s": round(train_s, 1),
                  "loss": losses[::max(1, len(losses) // 8)] + [losses[-1]], "checkpoint": out_path,
                  "ber": {k: v / nbits for k, v in err.items()}, "eval_bits": nbits,
                  "hard_decision_agreement_bf16_vs_fp32": agree / tot,
                  "hard_decision_agreement_fp16_vs_fp32": agree_h / tot}))
