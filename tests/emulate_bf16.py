"""Test helper: CPU (torch fp32) emulation of the CNRX_BF16 / CNRX_FP16 plans' arithmetic.

The bf16 tensor-core plan rounds values to bf16 exactly where it stores activation planes (input
features, every conv epilogue output, pre-activated copies, pointwise-program outputs) and folds an
eval BN that follows a conv into bf16(W * scale) and bias*scale + shift.  This emulator applies the
same rounding points with fp32 accumulation, so the GPU result can be checked tightly against it
(deviation only from accumulation order), independent of how well bf16 tracks the fp32 reference.
It mirrors the absorption rules of Bf16Compiler in paper_2510_12739_b200/csrc/api.cpp.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as Fn

from paper_2510_12739_b200 import graph as G


import os

STEM_ENABLED = os.environ.get("CNRX_STEM") is not None  # mirrors api.cpp: fused CUDA-core stem is opt-in


def bf16(t: torch.Tensor) -> torch.Tensor:
    return t.to(torch.bfloat16).to(torch.float32)


def bn_affine(g, n):
    gamma, beta = g.params[n.gamma].value, g.params[n.beta].value
    rm, rv = g.params[n.rmean].value, g.params[n.rvar].value
    istd = (1.0 / np.sqrt(rv.astype(np.float64) + 1e-5)).astype(np.float32)
    scale = (gamma * istd).astype(np.float32)
    shift = (beta - rm * scale).astype(np.float32)
    return torch.from_numpy(scale), torch.from_numpy(shift)


def _ident(t: torch.Tensor) -> torch.Tensor:
    return t


def fp16(t: torch.Tensor) -> torch.Tensor:
    return t.to(torch.float16).to(torch.float32)


def fp16x2(t: torch.Tensor) -> torch.Tensor:
    """A value carried as an fp16 (hi, lo) pair: hi = fp16(t), lo = fp16(t - hi)."""
    hi = fp16(t)
    return hi + fp16(t - hi)


def bf16x2(t: torch.Tensor) -> torch.Tensor:
    """A value carried as a bf16 (hi, lo) pair: hi = bf16(t), lo = bf16(t - hi)."""
    hi = bf16(t)
    return hi + bf16(t - hi)


# Rounding points of the bf16 plan, by role (tools/ablate_bf16.py switches them one at a time):
#   feat  - the input feature plane (the stems' tensor-core operand)
#   w     - BN-folded conv weights (tensor-core operands)
#   act   - every other conv input plane (tensor-core operands: block inputs relu(y), conv1 outputs h)
#   res   - the residual stream: a block output y as stored for the next block's skip connection
#   leaf  - the subnetworks' final planes as the interaction fold reads them
#   z     - the folded interaction z and the head weights (tensor-core head)
BF16_POLICY = dict(feat=bf16, w=bf16, act=bf16, res=bf16, leaf=bf16, z=bf16)
# CNRX_FP16 plans: the same rounding points in fp16, and the LLR head in fp32 (z not rounded)
FP16_POLICY = dict(feat=fp16, w=fp16, act=fp16, res=fp16, leaf=fp16, z=_ident)


def emulate(g: "G.Graph", x: np.ndarray, policy: dict | None = None, precision: str = "bf16") -> np.ndarray:
    """x: [B,T,F,C] fp32 features -> LLRs [B,T,F,bits] as the bf16 (or fp16) plan computes them.

    `policy` overrides the rounding function per role (see BF16_POLICY); None = the shipped plan."""
    R = dict(BF16_POLICY if precision == "bf16" else FP16_POLICY)
    if policy:
        R.update(policy)
    return _emulate(g, x, R)


def _emulate(g, x, R):
    nodes = g.nodes
    consumers = [[] for _ in nodes]
    for i, n in enumerate(nodes):
        if n.in0 >= 0:
            consumers[n.in0].append(i)
        if n.in1 >= 0:
            consumers[n.in1].append(i)
    single = lambda i: consumers[i][0] if len(consumers[i]) == 1 else -1
    planes, vals, nonneg, producer_relu = {}, {}, {}, {}
    xt = torch.from_numpy(np.ascontiguousarray(x, np.float32)).permute(0, 3, 1, 2)  # [B,C,T,F]
    planes[g.input_node] = xt  # planes hold fp32 values; rounding is applied per role at each use

    def layer_norm(xv, n):  # norms.hpp:171-184 in double over the channel dim, as the GPU's pw_ln_kernel
        xd = xv.double()
        c = xd.shape[1]
        m = xd.sum(1, keepdim=True) / c
        v = torch.clamp((xd * xd).sum(1, keepdim=True) / c - m * m, min=0.0)
        istd = 1.0 / torch.sqrt(v + 1e-5)
        gm = torch.from_numpy(g.params[n.gamma].value).double()[None, :, None, None]
        bt = torch.from_numpy(g.params[n.beta].value).double()[None, :, None, None]
        return ((xd - m) * istd * gm + bt).float()

    def chain(u):
        if u in planes:
            return R['leaf'](planes[u])
        n = nodes[u]
        if n.op == G.OP_LN:  # its own row-wise program: a materialised plane, then a leaf
            planes[u] = R['act'](layer_norm(chain(n.in0), n))
            return R['leaf'](planes[u])
        if n.op == G.OP_RELU:
            return torch.relu(chain(n.in0))
        if n.op == G.OP_BN:
            s, t = bn_affine(g, n)
            return chain(n.in0) * s[None, :, None, None] + t[None, :, None, None]
        if n.op in (G.OP_ADD, G.OP_MUL):
            for o in (n.in0, n.in1):  # a layer-norm operand is materialised as a plane first
                if o not in planes and nodes[o].op == G.OP_LN:
                    chain(o)
            if n.in1 in planes:
                leaf, rest = n.in1, n.in0
            elif n.in0 in planes:
                leaf, rest = n.in0, n.in1
            else:
                raise ValueError("not a linear chain")
            r = chain(rest)
            lv = R['leaf'](planes[leaf])
            return r * lv if n.op == G.OP_MUL else r + lv
        raise ValueError(f"op {n.op} not emulated")

    def plane_for(u):
        if u in planes:
            return planes[u]
        n = nodes[u]
        if n.op == G.OP_DWCONV:  # depthwise conv on CUDA cores (launch_dwconv_plane): fp32 weights
            xin = R['act'](plane_for(n.in0))
            wv = g.params[n.w].value  # [kh,kw,C,1]
            kh, kw = wv.shape[0], wv.shape[1]
            wk = torch.from_numpy(np.ascontiguousarray(wv[..., 0].transpose(2, 0, 1)))[:, None]  # [C,1,kh,kw]
            bias = torch.from_numpy(g.params[n.b].value) if n.b >= 0 else None
            planes[u] = Fn.conv2d(xin, wk, bias=bias, padding=(kh // 2, (kw // 2) * n.dilation_f),
                                  dilation=(1, n.dilation_f), groups=wk.shape[0])
            return planes[u]
        if n.op == G.OP_CONCAT:  # the two planes side by side (launch_concat_planes): a copy, no rounding
            planes[u] = torch.cat([plane_for(n.in0), plane_for(n.in1)], 1)
            return planes[u]
        if n.op == G.OP_RELU:
            v, bn = n.in0, None
            if v not in planes and nodes[v].op == G.OP_BN and nodes[v].in0 in planes:
                bn, v = nodes[v], nodes[v].in0
            if v in planes:
                if bn is None and nonneg.get(v, False):
                    planes[u] = planes[v]
                    return planes[u]
                if v in vals:
                    z = vals[v]
                    if bn is not None:
                        s, t = bn_affine(g, bn)
                        z = z * s[None, :, None, None] + t[None, :, None, None]
                    planes[u] = torch.relu(z)
                    return planes[u]
        planes[u] = R['act'](chain(u))  # a pointwise-program output plane
        return planes[u]

    absorbed = set()
    stem_cin = None
    n_stems = 0
    for i, n in enumerate(nodes):
        if n.op != G.OP_CONV or i in absorbed or i == g.output_node:
            continue
        w0 = g.params[n.w].value
        # 1x1 convs on the network input run on CUDA cores in fp32 (fused stem kernel): no bf16
        # rounding of the features or the weights (mirrors Bf16Compiler's stem selection)
        stem = (STEM_ENABLED and n.in0 == g.input_node and w0.shape[0] == 1 and w0.shape[2] in (6, 12, 24, 48)
                and w0.shape[3] % 8 == 0 and w0.shape[3] <= 64 and n_stems < 4
                and (stem_cin is None or stem_cin == w0.shape[2]))
        if stem:
            n_stems += 1
            stem_cin = w0.shape[2]
        inp = xt if stem else (R['feat'] if n.in0 == g.input_node else R['act'])(plane_for(n.in0))
        w = torch.from_numpy(g.params[n.w].value)  # [kh,kw,cin,cout]
        cout = w.shape[3]
        bias = torch.from_numpy(g.params[n.b].value.copy()) if n.b >= 0 else torch.zeros(cout)
        scale = None
        end, relu, res = i, False, None
        c = single(end)
        if c >= 0 and nodes[c].op == G.OP_BN and c != g.output_node:
            scale, shift = bn_affine(g, nodes[c])
            bias = bias * scale + shift
            absorbed.add(c)
            end, c = c, single(c)
        if c >= 0 and nodes[c].op == G.OP_RELU:
            relu = True
            absorbed.add(c)
            end, c = c, single(c)
        if not relu and c >= 0 and nodes[c].op == G.OP_ADD:
            other = nodes[c].in1 if nodes[c].in0 == end else nodes[c].in0
            if other != end and other < i:
                res = R['res'](plane_for(other))
                absorbed.add(c)
                end = c
        if res is not None and stem:
            raise ValueError("stem with residual is not emulated")
        wf = w * scale[None, None, None, :] if scale is not None else w
        wk = wf.permute(3, 2, 0, 1).contiguous()  # [cout,cin,kh,kw]
        if not stem:
            wk = R['w'](wk)
        kh, kw = w.shape[0], w.shape[1]
        cin_plane = inp.shape[1]
        if cin_plane > wk.shape[1]:  # zero-padded input channels
            wk = torch.cat([wk, torch.zeros(cout, cin_plane - wk.shape[1], kh, kw)], 1)
        v = Fn.conv2d(inp, wk, bias=bias, padding=(kh // 2, (kw // 2) * n.dilation_f), dilation=(1, n.dilation_f))
        if relu:
            v = torch.relu(v)
        if res is not None:
            v = v + res
        vals[end] = v
        planes[end] = v
        nonneg[end] = relu
    on = nodes[g.output_node]
    w_out = g.params[on.w].value
    if w_out.shape[0] == 3:
        # 3x3 LLR head (NetSpec.kernel = 3): the fold chain materialised as a 16-bit plane, a tensor-core conv
        # with rounded weights, fp32 LLRs (Bf16Compiler's llr_head op)
        z = R['act'](plane_for(on.in0))
        wk = R['w'](torch.from_numpy(w_out).permute(3, 2, 0, 1).contiguous())
        if z.shape[1] > wk.shape[1]:
            wk = torch.cat([wk, torch.zeros(wk.shape[0], z.shape[1] - wk.shape[1], 3, 3)], 1)
        hb = torch.from_numpy(g.params[on.b].value) if on.b >= 0 else torch.zeros(w_out.shape[3])
        v = Fn.conv2d(z, wk, bias=hb, padding=(1, on.dilation_f), dilation=(1, on.dilation_f))
        return v.permute(0, 2, 3, 1).contiguous().numpy()
    f = chain(on.in0)
    hw = torch.from_numpy(g.params[on.w].value[0, 0])  # [C,bits]
    hb = torch.from_numpy(g.params[on.b].value) if on.b >= 0 else torch.zeros(hw.shape[1])
    if hw.shape[0] == 64 and hw.shape[1] in (2, 4, 6, 8) and os.environ.get("CNRX_TC_HEAD") is not None:
        # opt-in tensor-core head (cnrx_plan_options::tensor_core_head, bf16 plans): the folded
        # interaction z and the head weights are rounded to bf16, products accumulate in fp32
        f, hw = R['z'](f), R['z'](hw)
    out = torch.einsum("bctf,cj->btfj", f, hw) + hb
    return out.numpy()
