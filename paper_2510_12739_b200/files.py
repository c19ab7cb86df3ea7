"""Net spec files and CNCK checkpoints -> graph -> GPU plan.

Restates the reference's file formats so trained networks load straight into the B200 plan without the
reference's own C++ `Network`:

* spec file JSON (`parse_spec_file_json` / `spec_file_to_json` / `load_spec_file`,
  netspec.cpp:160-257; `SpecFile`, netspec.hpp:78-106) with the same defaults, the same error
  messages (std::invalid_argument -> ValueError, std::runtime_error -> RuntimeError) and the same
  canonical JSON text (the vendored nlohmann prints sorted keys, two-space indent, inline int arrays);
* the parameter-budget width solver (`solve_filters` / `solve_spec_width`, netspec.cpp:103-158);
* the CNCK checkpoint (`save_checkpoint` / `load_checkpoint`, checkpoint.cpp:47-99): little-endian,
  magic "CNCK", version 1, (name, rank, dims u64, fp32 data) per parameter in `params()` order, then
  (name, u8) BN-ready flags keyed by `bn_flag_names()`.

tests/test_files.py pins all of it against the reference built in place (oracle/_ref): canonical JSON
text, graphs, solved widths, and checkpoints written by either side and read by the other.
"""
from __future__ import annotations

import json
import struct
from dataclasses import dataclass, field, replace
from typing import Callable, List, Optional

import numpy as np

from . import graph as G
from .graph import require

_FUSION_OPS = ("mul", "add", "concat")
_NORMS = ("bn", "ln")
_CONVS = ("standard", "depthwise")


@dataclass
class SpecFile:
    """netspec.hpp:78-102 (defaults included)."""
    family: str = "deeprx"
    width: int = 64
    blocks: int = 4
    main_blocks: int = 4
    support_blocks: List[int] = field(default_factory=lambda: [4])
    conv: str = "standard"
    kernel: int = 3
    fusion_op: str = "mul"
    fusion_norm: str = "bn"
    fusion_points: List[int] = field(default_factory=list)
    bidirectional: bool = False
    in_channels: int = 6
    bits: int = 6
    target_params: int = 0

    def is_conet(self) -> bool:
        return self.family == "conet"

    def to_deeprx(self) -> G.NetSpec:
        return G.deeprx_template(self.width, self.blocks, self.in_channels, self.bits, self.conv, self.kernel)

    def to_conet(self) -> G.CoNetSpec:
        return G.conet_template(self.width, self.main_blocks, self.support_blocks, self.fusion_op, self.fusion_norm,
                                self.bidirectional, self.in_channels, self.bits, self.conv, self.kernel,
                                self.fusion_points)

    def with_width(self, w: int) -> "SpecFile":
        return replace(self, width=w, support_blocks=list(self.support_blocks),
                       fusion_points=list(self.fusion_points))

    def build(self, shape_only: bool = False) -> G.Graph:
        """The network this spec describes (build_conet / build_net at the spec's width)."""
        if self.is_conet():
            return G.build_conet(self.to_conet(), shape_only=shape_only)
        return G.build_net(self.to_deeprx(), shape_only=shape_only)


def _choice(v: str, allowed, what: str, expected: str) -> str:
    if v not in allowed:
        raise ValueError(f"unknown {what} '{v}' (expected {expected})")
    return v


def parse_spec_file_json(text: str) -> SpecFile:
    """netspec.cpp:202-228."""
    j = json.loads(text)
    f = SpecFile()
    f.family = j.get("template", "deeprx")
    require(f.family in ("deeprx", "conet"), "spec template must be deeprx or conet")
    f.width = int(j.get("width", f.width))
    f.blocks = int(j.get("blocks", f.blocks))
    f.main_blocks = int(j.get("main_blocks", f.main_blocks))
    if "support_blocks" in j:
        v = j["support_blocks"]
        f.support_blocks = [int(x) for x in v] if isinstance(v, list) else [int(v)]
    f.conv = _choice(j.get("conv", "standard"), _CONVS, "conv kind", "standard|depthwise")
    f.kernel = int(j.get("kernel", f.kernel))
    f.fusion_op = _choice(j.get("fusion_op", "mul"), _FUSION_OPS, "fusion op", "mul|add|concat")
    f.fusion_norm = _choice(j.get("fusion_norm", "bn"), _NORMS, "norm kind", "bn|ln")
    if "fusion_points" in j:
        f.fusion_points = [int(x) for x in j["fusion_points"]]
    f.bidirectional = bool(j.get("bidirectional", False))
    f.in_channels = int(j.get("in_channels", f.in_channels))
    f.bits = int(j.get("bits", f.bits))
    f.target_params = int(j.get("target_params", 0))
    return f


def load_spec_file(path: str) -> SpecFile:
    """netspec.cpp:230-236."""
    try:
        with open(path) as fh:
            text = fh.read()
    except OSError:
        raise RuntimeError("cannot open net spec file " + path) from None
    return parse_spec_file_json(text)


def spec_file_to_json(f: SpecFile) -> str:
    """netspec.cpp:238-257 (nlohmann::json keeps object keys sorted; dump(2))."""
    j = {"template": f.family, "width": f.width}
    if f.is_conet():
        j["main_blocks"] = f.main_blocks
        j["support_blocks"] = list(f.support_blocks)
        j["fusion_op"] = f.fusion_op
        j["fusion_norm"] = f.fusion_norm
        if f.fusion_points:
            j["fusion_points"] = list(f.fusion_points)
        j["bidirectional"] = f.bidirectional
    else:
        j["blocks"] = f.blocks
    j["conv"] = f.conv
    j["kernel"] = f.kernel
    j["in_channels"] = f.in_channels
    j["bits"] = f.bits
    if f.target_params > 0:
        j["target_params"] = f.target_params
    # the reference's nlohmann build prints sorted keys one per line and int arrays inline ("[4,4]")
    items = [f"  {json.dumps(k)}: " + ("[" + ",".join(str(int(x)) for x in v) + "]" if isinstance(v, list)
                                       else json.dumps(v)) for k, v in sorted(j.items())]
    return "{\n" + ",\n".join(items) + "\n}"


# ---------------------------------------------------------------------------------------------
# width solving (netspec.cpp:99-158)
# ---------------------------------------------------------------------------------------------
@dataclass
class SolveResult:
    """network.hpp:609-616."""
    found: bool = False
    width: int = 0
    params: int = 0
    lo_width: int = 0
    hi_width: int = 0
    lo_params: int = 0
    hi_params: int = 0
    diagnostic: str = ""


def solve_filters(count_at_width: Callable[[int], int], target: int, tol: float = 0.01,
                  max_width: int = 4096) -> SolveResult:
    """netspec.cpp:103-145: bisection over a monotone width -> parameter-count map."""
    require(target > 0, "target parameter count must be positive")
    at_min = count_at_width(1)
    require(target >= at_min, f"target {target} is below the minimal net ({at_min} params at width 1)")
    lo, hi = 1, max_width
    if count_at_width(hi) < target:
        return SolveResult(diagnostic=f"target {target} exceeds the count at max width {max_width}")
    while hi - lo > 1:
        mid = lo + (hi - lo) // 2
        if count_at_width(mid) < target:
            lo = mid
        else:
            hi = mid
    r = SolveResult(lo_width=lo, lo_params=count_at_width(lo), hi_width=hi, hi_params=count_at_width(hi))
    err_lo = abs(r.lo_params - target) / target
    err_hi = abs(r.hi_params - target) / target
    if min(err_lo, err_hi) <= tol:
        r.found = True
        r.width, r.params = (r.lo_width, r.lo_params) if err_lo <= err_hi else (r.hi_width, r.hi_params)
    else:
        r.diagnostic = (f"no integer width within {tol * 100:g}% of {target}: width {r.lo_width} -> {r.lo_params} "
                        f"params, width {r.hi_width} -> {r.hi_params} params")
    return r


def solve_spec_width(f: SpecFile, target: int, tol: float = 0.01) -> SolveResult:
    """netspec.cpp:147-153 (param_count(...).total_learnable at each width, without allocating weights)."""
    return solve_filters(lambda w: f.with_width(w).build(shape_only=True).learnable_count(), target, tol)


def graph_from_spec(f: SpecFile) -> G.Graph:
    """The spec's network; a positive target_params first solves the width (error if none is within 1 %)."""
    if f.target_params > 0:
        r = solve_spec_width(f, f.target_params)
        if not r.found:
            raise ValueError(r.diagnostic)
        f = f.with_width(r.width)
    return f.build()


# ---------------------------------------------------------------------------------------------
# CNCK checkpoints (checkpoint.cpp:47-99)
# ---------------------------------------------------------------------------------------------
_MAGIC = b"CNCK"
_VERSION = 1


def save_checkpoint(g: G.Graph, path: str) -> None:
    """checkpoint.cpp:47-68."""
    try:
        fh = open(path, "wb")
    except OSError:
        raise RuntimeError("cannot open checkpoint for writing: " + path) from None
    with fh:
        out = [_MAGIC, struct.pack("<IQ", _VERSION, len(g.params))]
        for p in g.params:
            nb = p.name.encode()
            v = np.ascontiguousarray(p.value, dtype="<f4")
            out.append(struct.pack("<I", len(nb)) + nb + struct.pack("<I", v.ndim) +
                       struct.pack(f"<{v.ndim}Q", *v.shape) + v.tobytes())
        out.append(struct.pack("<I", len(g.bn_flag_names)))
        for name, ready in zip(g.bn_flag_names, g.bn_ready):
            nb = name.encode()
            out.append(struct.pack("<I", len(nb)) + nb + struct.pack("<B", 1 if ready else 0))
        fh.write(b"".join(out))


class _Reader:
    def __init__(self, data: bytes):
        self.d, self.o, self.bad = data, 0, False

    def take(self, n: int) -> bytes:
        b = self.d[self.o:self.o + n]
        if len(b) < n:  # std::ifstream: a short read sets failbit, later reads yield zeros
            self.bad = True
            b = b + bytes(n - len(b))
        self.o += n
        return b

    def u8(self) -> int:
        return self.take(1)[0]

    def u32(self) -> int:
        return struct.unpack("<I", self.take(4))[0]

    def u64(self) -> int:
        return struct.unpack("<Q", self.take(8))[0]

    def string(self) -> str:
        return self.take(self.u32()).decode(errors="replace")


def load_checkpoint(g: G.Graph, path: str) -> None:
    """checkpoint.cpp:70-99: parameters by name (shape-checked), then BN-ready flags by name."""
    try:
        with open(path, "rb") as fh:
            data = fh.read()
    except OSError:
        raise RuntimeError("cannot open checkpoint: " + path) from None
    r = _Reader(data)
    if r.take(4) != _MAGIC:
        raise RuntimeError("not a checkpoint file: " + path)
    if r.u32() != _VERSION:
        raise RuntimeError("unsupported checkpoint version")
    count = r.u64()
    for _ in range(count):
        name = r.string()
        rank = r.u32()
        dims = tuple(r.u64() for _ in range(rank))
        idx = g.find_param(name)
        if idx < 0:
            raise RuntimeError("checkpoint parameter " + name + " not present in network")
        dst = g.params[idx]
        require(tuple(dst.value.shape) == dims, "checkpoint shape mismatch for " + name)
        n = int(np.prod(dims)) if dims else 1
        dst.value = np.frombuffer(r.take(4 * n), dtype="<f4").astype(np.float32).reshape(dims)
    nflags = r.u32()
    for _ in range(nflags):
        name = r.string()
        v = r.u8()
        for k, nm in enumerate(g.bn_flag_names):
            if nm == name:
                g.bn_ready[k] = v
    if r.bad:
        raise RuntimeError("truncated checkpoint: " + path)


def plan_from_files(spec_path: str, checkpoint_path: Optional[str], precision: str = "bf16", device: int = 0):
    """Spec file (+ CNCK checkpoint) -> graph -> GPU plan.  Without a checkpoint the graph keeps its
    build-time values (zero weights), which is only useful for shape checks."""
    from .plan import Plan
    g = graph_from_spec(load_spec_file(spec_path))
    if checkpoint_path:
        load_checkpoint(g, checkpoint_path)
    return Plan(g, precision, device)
