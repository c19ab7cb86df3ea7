"""Host-side mirror of the reference's network description API.

The drop-in boundary of this package is the reference's `conetrx::Network<float>` (network.hpp:45-432):
a closed vocabulary of `LayerOp` nodes (network.hpp:17), `GraphNode` records (network.hpp:19-26) and
named parameters (network.hpp:28-33), built by `build_net` / `build_conet` (network.hpp:470-562) from
`NetSpec` / `CoNetSpec` (netspec.hpp:19-54).  This module restates that construction API so that a
graph built here is node-for-node and name-for-name identical to the one the reference builds
(pinned by tests/test_graph_builders.py against the reference compiled in oracle/_ref).

The GPU plan (`paper_2510_12739_b200.plan.Plan`) consumes exactly these node/param arrays through the
C ABI in include/conetrx_cuda.h — the same fields the reference's C++ wrapper passes from a real
`Network<float>` (include/conetrx/gpu_plan.hpp).

One extension beyond the reference: `dilation_f` on conv nodes / BlockSpec (BASELINE config 3 needs
dilation 2 along frequency; the reference's conv2d has none, kernels.hpp:70-75).  It defaults to 1,
which is the reference behaviour.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

# LayerOp (network.hpp:17)
OP_INPUT, OP_CONV, OP_DWCONV, OP_RELU, OP_BN, OP_LN, OP_ADD, OP_MUL, OP_CONCAT = range(9)
OP_NAMES = ["input", "conv", "dwconv", "relu", "batch_norm", "layer_norm", "add", "mul", "concat"]
NODE_FIELDS = 12  # op,in0,in1,w,b,gamma,beta,rmean,rvar,bn_flag,out_channels,dilation_f


def require(cond: bool, msg: str) -> None:
    """tensor.hpp:13-15 — the reference throws std::invalid_argument."""
    if not cond:
        raise ValueError(msg)


@dataclass
class Node:
    """GraphNode (network.hpp:19-26) + dilation_f extension."""
    op: int
    in0: int = -1
    in1: int = -1
    w: int = -1
    b: int = -1
    gamma: int = -1
    beta: int = -1
    rmean: int = -1
    rvar: int = -1
    bn_flag: int = -1
    out_channels: int = 0
    dilation_f: int = 1

    def as_row(self) -> List[int]:
        return [self.op, self.in0, self.in1, self.w, self.b, self.gamma, self.beta, self.rmean, self.rvar,
                self.bn_flag, self.out_channels, self.dilation_f]


@dataclass
class Param:
    """NamedParam (network.hpp:28-33)."""
    name: str
    value: np.ndarray
    learnable: bool = True


class Graph:
    """Restatement of `conetrx::Network<float>`'s construction API (network.hpp:49-112)."""

    def __init__(self, shape_only: bool = False) -> None:
        # shape_only: parameters are zero-stride views with the right shapes (parameter counting for
        # width solving without allocating; such a graph cannot be run)
        self.shape_only = shape_only
        self.nodes: List[Node] = []
        self.params: List[Param] = []
        self.bn_ready: List[int] = []
        self.bn_flag_names: List[str] = []
        self.input_node = -1
        self.output_node = -1
        self.in_channels = 0
        # CoNet metadata (network.hpp:340-353)
        self.fusion_meta: List[tuple] = []
        self.stage_ranges: List[tuple] = []

    # -- construction (network.hpp:49-112) ------------------------------------------------------
    def _push(self, n: Node) -> int:
        self.nodes.append(n)
        return len(self.nodes) - 1

    def _push_param(self, name: str, shape: tuple, learnable: bool, fill: float = 0.0) -> int:
        require(self.find_param(name) < 0, "duplicate parameter name " + name)
        if self.shape_only:
            value = np.broadcast_to(np.float32(fill), shape)
        else:
            value = np.full(shape, fill, np.float32)
        self.params.append(Param(name, value, learnable))
        return len(self.params) - 1

    def _check_in(self, inp: int, expected: int) -> None:
        require(0 <= inp < len(self.nodes), "bad input node index")
        have = self.nodes[inp].out_channels
        require(have == expected, f"layer expects {expected} input channels but upstream node provides {have}")

    def find_param(self, name: str) -> int:
        for i, p in enumerate(self.params):
            if p.name == name:
                return i
        return -1

    def add_input(self, channels: int) -> int:
        require(self.input_node < 0, "network already has an input node")
        self.input_node = self._push(Node(OP_INPUT, out_channels=channels))
        self.in_channels = channels
        return self.input_node

    def add_conv(self, inp: int, name: str, kernel: int, cin: int, cout: int, bias: bool,
                 dilation_f: int = 1) -> int:
        self._check_in(inp, cin)
        n = Node(OP_CONV, in0=inp, out_channels=cout, dilation_f=dilation_f)
        n.w = self._push_param(name + ".w", (kernel, kernel, cin, cout), True)
        if bias:
            n.b = self._push_param(name + ".b", (cout,), True)
        return self._push(n)

    def add_dwconv(self, inp: int, name: str, kernel: int, c: int, bias: bool) -> int:
        self._check_in(inp, c)
        n = Node(OP_DWCONV, in0=inp, out_channels=c)
        n.w = self._push_param(name + ".w", (kernel, kernel, c, 1), True)
        if bias:
            n.b = self._push_param(name + ".b", (c,), True)
        return self._push(n)

    def add_relu(self, inp: int) -> int:
        return self._push(Node(OP_RELU, in0=inp, out_channels=self.nodes[inp].out_channels))

    def add_norm(self, inp: int, kind: str, name: str, channels: int) -> int:
        self._check_in(inp, channels)
        n = Node(OP_BN if kind == "bn" else OP_LN, in0=inp, out_channels=channels)
        n.gamma = self._push_param(name + ".g", (channels,), True, 1.0)
        n.beta = self._push_param(name + ".s", (channels,), True)
        if kind == "bn":
            n.rmean = self._push_param(name + ".rm", (channels,), False)
            n.rvar = self._push_param(name + ".rv", (channels,), False, 1.0)
            n.bn_flag = len(self.bn_ready)
            self.bn_ready.append(0)
            self.bn_flag_names.append(name + ".rm")
        return self._push(n)

    def add_binary(self, op: int, a: int, b: int) -> int:
        require(op in (OP_ADD, OP_MUL), "add_binary takes add or mul")
        ca, cb = self.nodes[a].out_channels, self.nodes[b].out_channels
        require(ca == cb, f"elementwise fusion requires equal channel counts, got {ca} and {cb}")
        return self._push(Node(op, in0=a, in1=b, out_channels=ca))

    def add_concat(self, a: int, b: int) -> int:
        return self._push(Node(OP_CONCAT, in0=a, in1=b,
                               out_channels=self.nodes[a].out_channels + self.nodes[b].out_channels))

    def set_output(self, node: int) -> None:
        self.output_node = node

    # -- parameters ------------------------------------------------------------------------------
    def weight_owner(self, pidx: int) -> Optional[Node]:
        for n in self.nodes:
            if n.w == pidx:
                return n
        return None

    def init_he_normal(self, seed: int, randomize_aux: bool = False) -> "Graph":
        """He-normal conv weights from a seed (BASELINE: "Weights: He-normal from seed"); the reference's
        own init is He-uniform (network.hpp:115-127) — any init works for parity as both sides receive
        identical fp32 values.  With randomize_aux, biases, BN gains/shifts and running statistics are
        randomised too (so BN-folding bugs surface) and every BN is marked ready."""
        rng = np.random.default_rng(seed)
        for i, p in enumerate(self.params):
            owner = self.weight_owner(i)
            if owner is not None:
                w = p.value
                fan_in = w.shape[0] * w.shape[1] * (w.shape[2] if owner.op == OP_CONV else 1)
                p.value = (rng.standard_normal(w.shape) * np.sqrt(2.0 / fan_in)).astype(np.float32)
            elif randomize_aux:
                n = p.value.shape[0]
                if p.name.endswith(".b"):
                    p.value = rng.uniform(-0.1, 0.1, n).astype(np.float32)
                elif p.name.endswith(".g"):
                    p.value = rng.uniform(0.6, 1.4, n).astype(np.float32)
                elif p.name.endswith(".s"):
                    p.value = rng.uniform(-0.2, 0.2, n).astype(np.float32)
                elif p.name.endswith(".rm"):
                    p.value = rng.uniform(-0.2, 0.2, n).astype(np.float32)
                elif p.name.endswith(".rv"):
                    p.value = rng.uniform(0.5, 2.0, n).astype(np.float32)
        if randomize_aux:
            self.bn_ready = [1] * len(self.bn_ready)
        return self

    def seed_norm_stats(self) -> "Graph":
        """network.hpp:131-138: rm=0, rv=1, every BN ready."""
        for n in self.nodes:
            if n.op == OP_BN:
                self.params[n.rmean].value[:] = 0.0
                self.params[n.rvar].value[:] = 1.0
                self.bn_ready[n.bn_flag] = 1
        return self

    def copy_params_from(self, other: "Graph") -> None:
        """copy_params_by_name (network.hpp:591-600)."""
        for p in self.params:
            idx = other.find_param(p.name)
            require(idx >= 0, "source network lacks parameter " + p.name)
            sp = other.params[idx]
            require(sp.value.shape == p.value.shape, "parameter shape mismatch for " + p.name)
            p.value = sp.value.copy()

    # -- reports (network.hpp:305-338) -----------------------------------------------------------
    def learnable_count(self) -> int:
        return int(sum(p.value.size for p in self.params if p.learnable))

    def conv_depth(self) -> int:
        d = [0] * len(self.nodes)
        for i, n in enumerate(self.nodes):
            best = 0
            if n.in0 >= 0:
                best = max(best, d[n.in0])
            if n.in1 >= 0:
                best = max(best, d[n.in1])
            d[i] = best + (1 if n.op in (OP_CONV, OP_DWCONV) else 0)
        return d[self.output_node]

    def output_channels(self) -> int:
        return self.nodes[self.output_node].out_channels

    def node_array(self) -> np.ndarray:
        return np.asarray([n.as_row() for n in self.nodes], dtype=np.int32).reshape(-1, NODE_FIELDS)

    def max_dilation(self) -> int:
        return max([n.dilation_f for n in self.nodes if n.op == OP_CONV] + [1])

    def macs_per_re(self) -> int:
        """2*MACs/RE is the algorithmic FLOP count the roofline uses: every conv counts all
        kh*kw taps at every output RE, zero-padded borders included."""
        m = 0
        for n in self.nodes:
            if n.op == OP_CONV:
                kh, kw, cin, cout = self.params[n.w].value.shape
                m += kh * kw * cin * cout
            elif n.op == OP_DWCONV:
                kh, kw, c, _ = self.params[n.w].value.shape
                m += kh * kw * c
        return int(m)


# ---------------------------------------------------------------------------------------------
# Specs (netspec.hpp:11-54)
# ---------------------------------------------------------------------------------------------
@dataclass
class BlockSpec:
    kind: str = "rb"          # "rb" | "mrb"
    filters: int = 64
    kernel: int = 3
    conv: str = "standard"    # "standard" | "depthwise"
    dilation_f: int = 1       # extension (config 3)


@dataclass
class NetSpec:
    in_channels: int = 6
    input_filters: int = 64
    blocks: List[BlockSpec] = field(default_factory=list)
    output_bits: int = 6
    kernel: int = 3


@dataclass
class FusionPoint:
    main_block: int = 0
    support_id: int = 0
    op: str = "mul"           # "mul" | "add" | "concat"
    norm: str = "bn"          # "bn" | "ln"


@dataclass
class CoNetSpec:
    main: NetSpec
    supports: List[NetSpec]
    fusion: List[FusionPoint]
    bidirectional: bool = False

    def validate(self) -> None:
        """CoNetSpec::validate (netspec.cpp:13-40)."""
        require(len(self.supports) > 0, "conet spec needs at least one support net")
        require(len(self.main.blocks) > 0, "conet main net needs at least one block")
        for s in self.supports:
            require(len(s.blocks) > 0, "support net needs at least one block")
            require(s.in_channels == self.main.in_channels, "main and support nets share the input grid")

        def support_ch_at(i: int, stage: int) -> int:
            blocks = self.supports[i].blocks
            return blocks[min(stage, len(blocks) - 1)].filters

        for i, fp in enumerate(self.fusion):
            require(0 <= fp.main_block < len(self.main.blocks),
                    f"fusion point {i} references main block {fp.main_block} outside "
                    f"[0,{len(self.main.blocks)})")
            require(0 <= fp.support_id < len(self.supports),
                    f"fusion point {i} references unknown support net")
            if fp.op != "concat":
                mch = self.main.blocks[fp.main_block].filters
                sch = support_ch_at(fp.support_id, fp.main_block)
                require(mch == sch, f"fusion point {i} ({fp.op}) requires equal channel counts, main {mch} "
                                    f"vs support {sch}")


def deeprx_template(width: int, blocks: int, in_channels: int, bits: int, conv: str = "standard",
                    kernel: int = 3) -> NetSpec:
    """netspec.cpp:42-51"""
    require(width >= 1 and blocks >= 1, "deeprx template needs width >= 1 and blocks >= 1")
    return NetSpec(in_channels, width, [BlockSpec("rb", width, kernel, conv) for _ in range(blocks)], bits, kernel)


def conet_template(width: int, main_blocks: int, support_blocks: Sequence[int], op: str, norm: str,
                   bidirectional: bool, in_channels: int, bits: int, conv: str = "standard", kernel: int = 3,
                   fusion_points: Sequence[int] = ()) -> CoNetSpec:
    """netspec.cpp:53-81"""
    require(width >= 1 and main_blocks >= 1 and len(support_blocks) > 0, "bad conet template arguments")
    main = NetSpec(in_channels, width, [BlockSpec("mrb", width, kernel, conv) for _ in range(main_blocks)],
                   bits, kernel)
    sups = []
    for nb in support_blocks:
        require(nb >= 1, "support net needs at least one block")
        sups.append(NetSpec(in_channels, width, [BlockSpec("mrb", width, kernel, conv) for _ in range(nb)], 0,
                            kernel))
    points = list(fusion_points) if fusion_points else list(range(main_blocks))
    fusion = [FusionPoint(k, m, op, norm) for k in points for m in range(len(sups))]
    return CoNetSpec(main, sups, fusion, bidirectional)


# ---------------------------------------------------------------------------------------------
# Builders (network.hpp:438-600)
# ---------------------------------------------------------------------------------------------
def _conv_stage(g: Graph, inp: int, name: str, kernel: int, cin: int, cout: int, bias: bool, kind: str,
                dilation_f: int = 1) -> int:
    """detail::conv_stage (network.hpp:443-449)"""
    if kind == "standard":
        return g.add_conv(inp, name, kernel, cin, cout, bias, dilation_f)
    dw = g.add_dwconv(inp, name + ".dw", kernel, cin, bias)
    return g.add_conv(dw, name + ".pw", 1, cin, cout, bias)


def _append_block(g: Graph, cur: int, cur_ch: int, blk: BlockSpec, prefix: str) -> tuple:
    """detail::append_block (network.hpp:451-465): RB = BN-ReLU-C1-BN-ReLU-C2 + skip; MRB drops the
    first BN.  No ReLU after the residual add."""
    f = blk.filters
    pre = cur
    t = cur
    if blk.kind == "rb":
        t = g.add_norm(t, "bn", prefix + ".n1", cur_ch)
    t = g.add_relu(t)
    t = _conv_stage(g, t, prefix + ".c1", blk.kernel, cur_ch, f, False, blk.conv, blk.dilation_f)
    t = g.add_norm(t, "bn", prefix + ".n2", f)
    t = g.add_relu(t)
    t = _conv_stage(g, t, prefix + ".c2", blk.kernel, f, f, True, blk.conv, blk.dilation_f)
    skip = pre if cur_ch == f else g.add_conv(pre, prefix + ".proj", 1, cur_ch, f, True)
    return g.add_binary(OP_ADD, t, skip), f


def build_net(spec: NetSpec, prefix: str = "main", shape_only: bool = False) -> Graph:
    """build_net (network.hpp:470-483)"""
    require(len(spec.blocks) > 0, "net spec needs at least one block")
    g = Graph(shape_only)
    inp = g.add_input(spec.in_channels)
    cur = g.add_relu(g.add_conv(inp, prefix + ".in", spec.kernel, spec.in_channels, spec.input_filters, True))
    ch = spec.input_filters
    for k, blk in enumerate(spec.blocks):
        cur, ch = _append_block(g, cur, ch, blk, f"{prefix}.b{k}")
    require(spec.output_bits > 0, "top-level net needs an output conv (output_bits > 0)")
    g.set_output(g.add_conv(cur, prefix + ".out", spec.kernel, ch, spec.output_bits, True))
    return g


def build_conet(spec: CoNetSpec, shape_only: bool = False) -> Graph:
    """build_conet (network.hpp:490-562)"""
    spec.validate()
    m_count = len(spec.supports)
    g = Graph(shape_only)
    inp = g.add_input(spec.main.in_channels)
    mcur = g.add_relu(g.add_conv(inp, "main.in", spec.main.kernel, spec.main.in_channels,
                                 spec.main.input_filters, True))
    mch = spec.main.input_filters
    scur, sch = [], []
    for m, s in enumerate(spec.supports):
        scur.append(g.add_relu(g.add_conv(inp, f"sup{m}.in", s.kernel, s.in_channels, s.input_filters, True)))
        sch.append(s.input_filters)
    max_stages = max([len(spec.main.blocks)] + [len(s.blocks) for s in spec.supports])
    prev_main_out = -1
    for k in range(max_stages):
        a_begin = len(g.nodes)
        for m, s in enumerate(spec.supports):
            if k >= len(s.blocks):
                continue
            sin = scur[m]
            if spec.bidirectional and prev_main_out >= 0:
                require(sch[m] == mch, f"bidirectional feedback needs equal main/support channels at stage {k}")
                sin = g.add_binary(OP_ADD, sin, prev_main_out)
            scur[m], sch[m] = _append_block(g, sin, sch[m], s.blocks[k], f"sup{m}.b{k}")
        a_end = len(g.nodes)
        b_begin = a_end
        if k < len(spec.main.blocks):
            mcur, mch = _append_block(g, mcur, mch, spec.main.blocks[k], f"main.b{k}")
        b_end = len(g.nodes)
        for fi, fp in enumerate(spec.fusion):
            if fp.main_block != k:
                continue
            operand, och = scur[fp.support_id], sch[fp.support_id]
            fname = f"fuse{fi}"
            if fp.op == "concat":
                require(och > 0, "fusion with uninitialized support")
                cc = g.add_concat(mcur, operand)
                fused = g.add_conv(cc, fname + ".restore", 1, mch + och, mch, False)
            else:
                require(och == mch, f"fusion point {fi} needs equal channels, main {mch} vs support {och}")
                fused = g.add_binary(OP_MUL if fp.op == "mul" else OP_ADD, mcur, operand)
            norm = g.add_norm(fused, fp.norm, fname + ".n", mch)
            g.fusion_meta.append((fused, operand, norm))
            mcur = norm
        g.stage_ranges.append((a_begin, a_end, b_begin, b_end, len(g.nodes)))
        prev_main_out = mcur
    g.set_output(g.add_conv(mcur, "main.out", spec.main.kernel, mch, spec.main.output_bits, True))
    return g


def build_reference_main(spec: CoNetSpec) -> Graph:
    """build_reference_main (network.hpp:567-587): the main path with each fusion replaced by its norm."""
    spec.validate()
    g = Graph()
    inp = g.add_input(spec.main.in_channels)
    cur = g.add_relu(g.add_conv(inp, "main.in", spec.main.kernel, spec.main.in_channels,
                                spec.main.input_filters, True))
    ch = spec.main.input_filters
    for k, blk in enumerate(spec.main.blocks):
        cur, ch = _append_block(g, cur, ch, blk, f"main.b{k}")
        for fi, fp in enumerate(spec.fusion):
            if fp.main_block != k:
                continue
            require(fp.op != "concat", "reference network is defined for mul/add fusion only")
            cur = g.add_norm(cur, fp.norm, f"fuse{fi}.n", ch)
    g.set_output(g.add_conv(cur, "main.out", spec.main.kernel, ch, spec.main.output_bits, True))
    return g


def build_plain_cnn_conet(in_channels: int, width: int, layers: int, n_subnets: int, bits: int,
                          kernel: int = 3) -> Graph:
    """BASELINE config 1: plain-CNN subnets (conv+ReLU chains) fused by element-wise product, then a 1x1
    head.  The reference has no BlockKind for plain CNNs (netspec.hpp:11), so — as the reference's own
    tests would — it is built with the raw add_conv/add_relu/add_binary API (network.hpp:56-103).
    There is no post-fusion norm on this path."""
    g = Graph()
    inp = g.add_input(in_channels)
    outs = []
    for s in range(n_subnets):
        name = "main" if s == 0 else f"sup{s - 1}"
        cur, ch = inp, in_channels
        for l in range(layers):
            cur = g.add_relu(g.add_conv(cur, f"{name}.c{l}", kernel, ch, width, True))
            ch = width
        outs.append(cur)
    fused = outs[0]
    for o in outs[1:]:
        fused = g.add_binary(OP_MUL, fused, o)
    g.set_output(g.add_conv(fused, "main.out", 1, width, bits, True))
    return g


# ---------------------------------------------------------------------------------------------
# BASELINE.json configs
# ---------------------------------------------------------------------------------------------
@dataclass
class LinkSpec:
    """Synthetic-slot parameters for one BASELINE config (generator: paper_2510_12739_b200.slots)."""
    T: int = 14
    F: int = 72
    N: int = 1
    mod_order: int = 4
    n_taps: int = 3
    rms_delay_s: float = 0.0       # 0: exponential PDP over n_taps with unit tap spacing index
    tap_spacing_s: float = 0.0
    doppler_max_hz: float = 0.0
    snr_db: tuple = (0.0, 20.0)
    sir_db: Optional[tuple] = None  # co-channel QPSK interferer (config 3)
    pilot_symbols: tuple = (2, 11)
    pilot_spacing: int = 2
    scs_hz: float = 30e3
    fc_hz: float = 3.5e9
    cp_fraction: float = 0.07

    @property
    def bits(self) -> int:
        return {4: 2, 16: 4, 64: 6}[self.mod_order]

    @property
    def features(self) -> int:
        return 6 * self.N


@dataclass
class Config:
    name: str
    graph_fn: object
    link: LinkSpec
    batch: int
    precision: str
    description: str = ""

    def graph(self, seed: int = 1, randomize_aux: bool = True) -> Graph:
        g = self.graph_fn()
        return g.init_he_normal(seed, randomize_aux=randomize_aux)


def _conet_cfg(width: int, n_sup: int, blocks: int, in_ch: int, bits: int, dil_subnets: Sequence[int] = ()) -> Graph:
    spec = conet_template(width, blocks, [blocks] * n_sup, "mul", "bn", False, in_ch, bits, "standard", 3,
                          [blocks - 1])
    # BASELINE configs use 1x1 stems/heads (NetSpec.kernel) with 3x3 block convs (BlockSpec.kernel).
    spec.main.kernel = 1
    for s in spec.supports:
        s.kernel = 1
    for idx in dil_subnets:  # 0 = main, m+1 = support m
        net = spec.main if idx == 0 else spec.supports[idx - 1]
        for b in net.blocks:
            b.dilation_f = 2
    return build_conet(spec)


def _resnet_cfg(width: int, blocks: int, in_ch: int, bits: int) -> Graph:
    spec = deeprx_template(width, blocks, in_ch, bits, "standard", 3)
    spec.kernel = 1
    return build_net(spec)


CONFIGS = {
    "cfg1": Config("cfg1", lambda: build_plain_cnn_conet(6, 32, 4, 2, 2),
                   LinkSpec(T=14, F=72, N=1, mod_order=4, n_taps=3, rms_delay_s=0.0, doppler_max_hz=0.0,
                            snr_db=(0.0, 20.0)),
                   64, "fp32", "CoNet-small: 2 plain-CNN subnets x 4 conv3x3 @32, mul, 1x1 head -> 2 LLRs"),
    "cfg2": Config("cfg2", lambda: _conet_cfg(64, 2, 4, 12, 4),
                   LinkSpec(T=14, F=612, N=2, mod_order=16, n_taps=12, rms_delay_s=300e-9, tap_spacing_s=100e-9,
                            doppler_max_hz=200.0, snr_db=(0.0, 25.0)),
                   256, "bf16", "CoNet-ResNet: 3 MRB subnets x 4 blocks @64, mul+BN fusion, 1x1 head -> 4 LLRs"),
    "cfg3": Config("cfg3", lambda: _conet_cfg(96, 3, 6, 24, 6, dil_subnets=(2, 3)),
                   LinkSpec(T=14, F=3276, N=4, mod_order=64, n_taps=23, rms_delay_s=1e-6, tap_spacing_s=200e-9,
                            doppler_max_hz=500.0,
                            snr_db=(0.0, 25.0), sir_db=(0.0, 15.0)),
                   64, "bf16", "CoNet-ResNet-large: 4 subnets x 6 MRB @96 (sup1, sup2 dilated x2 in F), 6 LLRs"),
    "cfg4": Config("cfg4", lambda: _resnet_cfg(96, 8, 12, 4),
                   LinkSpec(T=14, F=612, N=2, mod_order=16, n_taps=12, rms_delay_s=300e-9, tap_spacing_s=100e-9,
                            doppler_max_hz=200.0, snr_db=(0.0, 25.0)),
                   256, "bf16", "plain ResNet (DeepRx-style RB x 8 @96), same inputs as cfg2"),
    # "96 ch" and "MAC-matched to cfg2" disagree; run both.  W=78 gives 877,344 MACs/RE
    # (cfg2: 887,296); the bf16 plan pads 78 channels to 96 internally.
    "cfg4m": Config("cfg4m", lambda: _resnet_cfg(78, 8, 12, 4),
                    LinkSpec(T=14, F=612, N=2, mod_order=16, n_taps=12, rms_delay_s=300e-9, tap_spacing_s=100e-9,
                             doppler_max_hz=200.0, snr_db=(0.0, 25.0)),
                    256, "bf16", "plain ResNet (DeepRx-style RB x 8 @78, MAC-matched to cfg2), same inputs as cfg2"),
}
