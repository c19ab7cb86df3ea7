"""oracle — TEST INFRASTRUCTURE ONLY (the checker, never the product).

Two CPU implementations of the CoNet-Rx inference path, used by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, and by nothing else:

* `RefNet` — the UNMODIFIED reference (`conetrx::Network<float>`, proj/core of arxiv/paper_2510_12739)
  compiled in place by oracle/Makefile into oracle/_ref/libconetrx_ref.so, driven through the C shim
  oracle/ref_driver.cpp.  Graphs built with paper_2510_12739_b200.graph are replayed into the reference
  with its own add_* API (network.hpp:49-112), so the reference computes with its own code.
* `forward` / `featurize` / `pilot_pattern` — the plain-C restatement oracle/oracle.c (liboracle.so),
  pinned bit-for-bit against RefNet (tests/test_oracle_pin.py) and against tests/golden/ fixtures.
  It also covers what the reference snapshot lacks: the featurizer (SPEC.md:221-229, :272-289 — the
  reference's format_nn_input/classic.cpp are missing) and conv dilation (config 3).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_REF = None

_f32p = C.POINTER(C.c_float)
_i32p = C.POINTER(C.c_int32)
_u8p = C.POINTER(C.c_uint8)
_f64p = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def build(reference: bool = True) -> None:
    """Compile liboracle.so (always) and oracle/_ref (only where /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if reference and os.path.isdir(os.environ.get("CNRX_REFERENCE", "/root/reference")):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)
        # reference-side C++ integration example (needs libconetrx_cuda.so built first)
        integ = os.path.join(os.path.dirname(HERE), "tools", "integration")
        if os.path.exists(os.path.join(os.path.dirname(HERE), "paper_2510_12739_b200", "libconetrx_cuda.so")):
            subprocess.run(["make", "-s", "-C", integ], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build(reference=False)
        L = C.CDLL(path)
        L.orc_forward.restype = C.c_int
        L.orc_forward.argtypes = [_i32p, C.c_int, C.c_int, C.c_int, C.POINTER(_f32p), _i64p, _u8p, _f32p,
                                  C.c_int64, C.c_int64, C.c_int64, C.c_int64, _f32p]
        L.orc_last_error.restype = C.c_char_p
        L.orc_featurize.restype = C.c_int
        L.orc_featurize.argtypes = [_f32p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, _f32p, _u8p, _f32p]
        L.orc_pilot_pattern.restype = C.c_int
        L.orc_pilot_pattern.argtypes = [C.c_int, C.c_int, _i32p, C.c_int, C.c_int, _u8p, _f64p]
        L.orc_qam_map.restype = C.c_int
        L.orc_qam_map.argtypes = [_u8p, C.c_int, _f64p, _f64p]
        L.orc_rng_derive.restype = C.c_uint64
        L.orc_rng_derive.argtypes = [C.c_uint64, C.c_uint64]
        _LIB = L
    return _LIB


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libconetrx_ref.so"))


def ref():
    """The reference library (oracle/_ref), or raise if it was never built."""
    global _REF
    if _REF is None:
        path = os.path.join(HERE, "_ref", "libconetrx_ref.so")
        if not os.path.exists(path):
            raise RuntimeError("oracle/_ref/libconetrx_ref.so missing: run `make -C oracle ref` where "
                               "/root/reference exists")
        R = C.CDLL(path)
        vp = C.c_void_p
        R.ref_last_error.restype = C.c_char_p
        R.ref_net_new.restype = vp
        R.ref_net_free.argtypes = [vp]
        for fn, args in [("ref_add_input", [vp, C.c_int]),
                         ("ref_add_conv", [vp, C.c_int, C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int]),
                         ("ref_add_dwconv", [vp, C.c_int, C.c_char_p, C.c_int, C.c_int, C.c_int]),
                         ("ref_add_relu", [vp, C.c_int]),
                         ("ref_add_norm", [vp, C.c_int, C.c_int, C.c_char_p, C.c_int]),
                         ("ref_add_binary", [vp, C.c_int, C.c_int, C.c_int]),
                         ("ref_add_concat", [vp, C.c_int, C.c_int])]:
            getattr(R, fn).restype = C.c_int
            getattr(R, fn).argtypes = args
        R.ref_set_output.argtypes = [vp, C.c_int]
        R.ref_build_conet_k.restype = vp
        R.ref_build_conet_k.argtypes = [C.c_int, C.c_int, _i32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.c_int, C.c_int, C.c_int, C.c_int, _i32p, C.c_int]
        R.ref_build_deeprx_k.restype = vp
        R.ref_build_deeprx_k.argtypes = [C.c_int] * 7
        R.ref_n_nodes.argtypes = [vp]
        R.ref_get_node.argtypes = [vp, C.c_int, _i32p]
        R.ref_output_node.argtypes = [vp]
        R.ref_n_params.argtypes = [vp]
        R.ref_param_name.restype = C.c_char_p
        R.ref_param_name.argtypes = [vp, C.c_int]
        R.ref_param_rank.argtypes = [vp, C.c_int]
        R.ref_param_dim.restype = C.c_int64
        R.ref_param_dim.argtypes = [vp, C.c_int, C.c_int]
        R.ref_param_learnable.argtypes = [vp, C.c_int]
        R.ref_param_data.restype = _f32p
        R.ref_param_data.argtypes = [vp, C.c_int]
        R.ref_n_bn.argtypes = [vp]
        R.ref_set_bn_ready.argtypes = [vp, C.c_int, C.c_int]
        R.ref_get_bn_ready.argtypes = [vp, C.c_int]
        R.ref_seed_norm_stats.argtypes = [vp]
        R.ref_learnable_count.restype = C.c_int64
        R.ref_learnable_count.argtypes = [vp]
        R.ref_conv_depth.argtypes = [vp]
        R.ref_forward.restype = C.c_int
        R.ref_forward.argtypes = [vp, _f32p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, _f32p, C.c_int, C.c_int]
        R.ref_forward_overrides.restype = C.c_int
        R.ref_forward_overrides.argtypes = [vp, _f32p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, _f32p, _i32p,
                                            _f32p, C.c_int]
        R.ref_time_forward.restype = C.c_double
        R.ref_time_forward.argtypes = [vp, _f32p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, _f32p, C.c_int,
                                       C.c_int]
        R.ref_threads.restype = C.c_int
        R.ref_save_checkpoint.argtypes = [vp, C.c_char_p]
        R.ref_load_checkpoint.argtypes = [vp, C.c_char_p]
        R.ref_spec_to_json.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
        R.ref_net_from_spec.restype = vp
        R.ref_net_from_spec.argtypes = [C.c_char_p]
        R.ref_solve_spec_width.argtypes = [C.c_char_p, C.c_longlong, C.c_double, _i32p, _i32p, _i64p, _i32p, _i32p]
        R.ref_rng_u64.argtypes = [C.c_uint64, C.c_int, C.POINTER(C.c_uint64)]
        R.ref_rng_uniform.argtypes = [C.c_uint64, C.c_int, _f64p]
        R.ref_rng_normal.argtypes = [C.c_uint64, C.c_int, _f64p]
        R.ref_rng_derive.restype = C.c_uint64
        R.ref_rng_derive.argtypes = [C.c_uint64, C.c_uint64]
        R.ref_qam_map.argtypes = [_u8p, C.c_int, _f64p]
        R.ref_pilot_pattern.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _u8p, _f64p]
        R.ref_tdl_channel.argtypes = [C.c_double, C.c_double, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                      C.c_double, C.c_uint64, _f64p, _f64p, _f64p]
        R.ref_tdl_tap_powers.argtypes = [C.c_double, C.c_double, C.c_int, _f64p]
        R.ref_param_count_conet.argtypes = [C.c_int, C.c_int, _i32p, C.c_int, C.c_int, C.c_int, C.c_int, _i64p,
                                            _i32p]
        _REF = R
    return _REF


class RefError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


# ---------------------------------------------------------------------------------------------
# The reference network (real conetrx::Network<float>)
# ---------------------------------------------------------------------------------------------
class RefNet:
    """A live conetrx::Network<float> inside oracle/_ref."""

    def __init__(self, handle):
        if not handle:
            raise RefError(1, ref().ref_last_error().decode())
        self.h = C.c_void_p(handle)

    def __del__(self):
        try:
            if self.h:
                ref().ref_net_free(self.h)
        except Exception:
            pass

    # -- construction ----------------------------------------------------------------------------
    @classmethod
    def from_graph(cls, g) -> "RefNet":
        """Replay a paper_2510_12739_b200.graph.Graph into the reference through its add_* API
        (network.hpp:49-112) in node order, then copy every parameter value and BN-ready flag."""
        from paper_2510_12739_b200 import graph as G
        R = ref()
        net = cls(R.ref_net_new())
        pname = lambda i: g.params[i].name
        for i, n in enumerate(g.nodes):
            if n.op == G.OP_INPUT:
                r = R.ref_add_input(net.h, n.out_channels)
            elif n.op == G.OP_CONV:
                require_dil = n.dilation_f == 1
                if not require_dil:
                    raise RefError(3, "the reference conv2d has no dilation (kernels.hpp:70-75)")
                kh, kw, cin, cout = g.params[n.w].value.shape
                r = R.ref_add_conv(net.h, n.in0, pname(n.w)[:-2].encode(), kh, cin, cout, 1 if n.b >= 0 else 0)
            elif n.op == G.OP_DWCONV:
                kh, kw, c, _ = g.params[n.w].value.shape
                r = R.ref_add_dwconv(net.h, n.in0, pname(n.w)[:-2].encode(), kh, c, 1 if n.b >= 0 else 0)
            elif n.op == G.OP_RELU:
                r = R.ref_add_relu(net.h, n.in0)
            elif n.op in (G.OP_BN, G.OP_LN):
                r = R.ref_add_norm(net.h, n.in0, 0 if n.op == G.OP_BN else 1, pname(n.gamma)[:-2].encode(),
                                   n.out_channels)
            elif n.op in (G.OP_ADD, G.OP_MUL):
                r = R.ref_add_binary(net.h, n.op, n.in0, n.in1)
            elif n.op == G.OP_CONCAT:
                r = R.ref_add_concat(net.h, n.in0, n.in1)
            else:
                raise RefError(1, f"unknown op {n.op}")
            if r != i:
                raise RefError(1, f"replay diverged at node {i}: {R.ref_last_error().decode()}")
        R.ref_set_output(net.h, g.output_node)
        net.load_params(g)
        return net

    @classmethod
    def conet(cls, width, main_blocks, support_blocks, in_ch, bits, fusion_points=(), fusion_op=0, norm=0,
              bidir=False, block_kind=1, io_kernel=1, block_kernel=3) -> "RefNet":
        sb = np.asarray(support_blocks, np.int32)
        fp = np.asarray(fusion_points, np.int32)
        return cls(ref().ref_build_conet_k(width, main_blocks, _ptr(sb, _i32p), len(sb), fusion_op, norm,
                                           int(bidir), in_ch, bits, block_kind, io_kernel, block_kernel,
                                           _ptr(fp, _i32p), len(fp)))

    @classmethod
    def deeprx(cls, width, blocks, in_ch, bits, block_kind=0, io_kernel=1, block_kernel=3) -> "RefNet":
        return cls(ref().ref_build_deeprx_k(width, blocks, in_ch, bits, block_kind, io_kernel, block_kernel))

    @classmethod
    def from_spec(cls, text: str) -> "RefNet":
        """parse_spec_file_json + build_conet / build_net (netspec.cpp:202-228, network.hpp:470-562)."""
        return cls(ref().ref_net_from_spec(text.encode()))

    # -- checkpoints (checkpoint.cpp:47-99) ------------------------------------------------------
    def save_checkpoint(self, path: str) -> None:
        if ref().ref_save_checkpoint(self.h, path.encode()):
            raise RefError(1, ref().ref_last_error().decode())

    def load_checkpoint(self, path: str) -> None:
        rc = ref().ref_load_checkpoint(self.h, path.encode())
        if rc:
            raise RefError(rc, ref().ref_last_error().decode())

    def param_values(self):
        """[(name, fp32 array)] in params() order, copied out of the reference network."""
        R = ref()
        out = []
        for i, (name, shape, _) in enumerate(self.params()):
            n = int(np.prod(shape)) if shape else 1
            ptr = R.ref_param_data(self.h, i)
            out.append((name, np.ctypeslib.as_array(ptr, shape=(n,)).copy().reshape(shape)))
        return out

    def bn_ready(self):
        R = ref()
        return [int(R.ref_get_bn_ready(self.h, k)) for k in range(R.ref_n_bn(self.h))]

    # -- parameters ------------------------------------------------------------------------------
    def load_params(self, g) -> None:
        R = ref()
        for i in range(R.ref_n_params(self.h)):
            name = R.ref_param_name(self.h, i).decode()
            j = g.find_param(name)
            if j < 0:
                raise RefError(1, "graph lacks parameter " + name)
            v = np.ascontiguousarray(g.params[j].value, np.float32).ravel()
            dst = R.ref_param_data(self.h, i)
            C.memmove(dst, v.ctypes.data, v.nbytes)
        for k, flag in enumerate(g.bn_ready):
            R.ref_set_bn_ready(self.h, k, int(flag))

    def nodes(self) -> np.ndarray:
        R = ref()
        out = np.zeros((R.ref_n_nodes(self.h), 11), np.int32)
        for i in range(out.shape[0]):
            R.ref_get_node(self.h, i, _ptr(out[i], _i32p))
        return out

    def params(self):
        R = ref()
        res = []
        for i in range(R.ref_n_params(self.h)):
            rank = R.ref_param_rank(self.h, i)
            shape = tuple(R.ref_param_dim(self.h, i, d) for d in range(rank))
            res.append((R.ref_param_name(self.h, i).decode(), shape, bool(R.ref_param_learnable(self.h, i))))
        return res

    def learnable_count(self) -> int:
        return int(ref().ref_learnable_count(self.h))

    def conv_depth(self) -> int:
        return int(ref().ref_conv_depth(self.h))

    def output_channels(self) -> int:
        return int(self.nodes()[ref().ref_output_node(self.h)][10])

    # -- the hot path ------------------------------------------------------------------------------
    def forward(self, x: np.ndarray, concurrent: bool = False, train: bool = False) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        B, T, F, Cin = x.shape
        out = np.zeros((B, T, F, self.output_channels()), np.float32)
        rc = ref().ref_forward(self.h, _ptr(x, _f32p), B, T, F, Cin, _ptr(out, _f32p), int(concurrent),
                               1 if train else 0)
        if rc:
            raise RefError(rc, ref().ref_last_error().decode())
        return out

    def forward_overrides(self, x: np.ndarray, overrides: dict) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        B, T, F, Cin = x.shape
        out = np.zeros((B, T, F, self.output_channels()), np.float32)
        ids = np.asarray(list(overrides.keys()), np.int32)
        vals = np.asarray(list(overrides.values()), np.float32)
        rc = ref().ref_forward_overrides(self.h, _ptr(x, _f32p), B, T, F, Cin, _ptr(out, _f32p), _ptr(ids, _i32p),
                                         _ptr(vals, _f32p), len(ids))
        if rc:
            raise RefError(rc, ref().ref_last_error().decode())
        return out

    def time_forward(self, x: np.ndarray, reps: int, concurrent: bool = False) -> float:
        x = np.ascontiguousarray(x, np.float32)
        B, T, F, Cin = x.shape
        out = np.zeros((B, T, F, self.output_channels()), np.float32)
        return float(ref().ref_time_forward(self.h, _ptr(x, _f32p), B, T, F, Cin, _ptr(out, _f32p),
                                            int(concurrent), reps))


def spec_to_json(text: str) -> str:
    """The reference's canonical spec JSON: spec_file_to_json(parse_spec_file_json(text))."""
    buf = C.create_string_buffer(1 << 16)
    if ref().ref_spec_to_json(text.encode(), buf, len(buf)):
        raise RefError(1, ref().ref_last_error().decode())
    return buf.value.decode()


def solve_spec_width(text: str, target: int, tol: float = 0.01):
    """solve_spec_width (netspec.cpp:147-153) -> (found, width, params, lo_width, hi_width)."""
    found, width, lo, hi = (C.c_int32() for _ in range(4))
    params = C.c_int64()
    if ref().ref_solve_spec_width(text.encode(), target, tol, C.byref(found), C.byref(width), C.byref(params),
                                  C.byref(lo), C.byref(hi)):
        raise RefError(1, ref().ref_last_error().decode())
    return bool(found.value), width.value, params.value, lo.value, hi.value


# ---------------------------------------------------------------------------------------------
# The C restatement
# ---------------------------------------------------------------------------------------------
def forward(g, x: np.ndarray) -> np.ndarray:
    """orc_forward: restated Network<float>::forward (eval) over a graph.Graph."""
    L = lib()
    x = np.ascontiguousarray(x, np.float32)
    B, T, F, Cin = x.shape
    nodes = np.ascontiguousarray(g.node_array())
    vals = [np.ascontiguousarray(p.value, np.float32) for p in g.params]
    ptrs = (_f32p * max(1, len(vals)))(*[v.ctypes.data_as(_f32p) for v in vals])
    dims = np.ones((max(1, len(vals)), 4), np.int64)
    for i, v in enumerate(vals):
        dims[i, :v.ndim] = v.shape
    ready = np.asarray(g.bn_ready if g.bn_ready else [0], np.uint8)
    out = np.zeros((B, T, F, g.output_channels()), np.float32)
    rc = L.orc_forward(_ptr(nodes, _i32p), len(g.nodes), g.input_node, g.output_node, ptrs, _ptr(dims, _i64p),
                       _ptr(ready, _u8p), _ptr(x, _f32p), B, T, F, Cin, _ptr(out, _f32p))
    if rc:
        raise RefError(rc, L.orc_last_error().decode())
    return out


def featurize(y: np.ndarray, pilots: np.ndarray, mask: np.ndarray) -> np.ndarray:
    """y: complex64 [B,T,F,N]; pilots complex [T,F]; mask uint8 [T,F] -> features fp32 [B,T,F,6N]."""
    L = lib()
    y = np.ascontiguousarray(y, np.complex64)
    B, T, F, N = y.shape
    p = np.ascontiguousarray(pilots, np.complex64)
    m = np.ascontiguousarray(mask, np.uint8)
    out = np.zeros((B, T, F, 6 * N), np.float32)
    rc = L.orc_featurize(y.view(np.float32).ctypes.data_as(_f32p), B, T, F, N, p.view(np.float32).ctypes.data_as(_f32p),
                         _ptr(m, _u8p), _ptr(out, _f32p))
    if rc:
        raise RefError(rc, L.orc_last_error().decode())
    return out


def pilot_pattern(T: int, F: int, symbols: Sequence[int], spacing: int):
    L = lib()
    syms = np.asarray(symbols, np.int32)
    mask = np.zeros((T, F), np.uint8)
    vals = np.zeros((T, F, 2), np.float64)
    rc = L.orc_pilot_pattern(T, F, _ptr(syms, _i32p), len(syms), spacing, _ptr(mask, _u8p), _ptr(vals, _f64p))
    if rc:
        raise RefError(rc, L.orc_last_error().decode())
    return mask, vals[..., 0] + 1j * vals[..., 1]


def qam_map(bits: Sequence[int], order: int) -> complex:
    b = np.asarray(bits, np.uint8)
    re, im = C.c_double(), C.c_double()
    rc = lib().orc_qam_map(_ptr(b, _u8p), order, C.byref(re), C.byref(im))
    if rc:
        raise RefError(rc, lib().orc_last_error().decode())
    return complex(re.value, im.value)
