"""ctypes binding of the C ABI (include/conetrx_cuda.h) — the Python mirror of the reference-facing
boundary.  `Plan(graph, precision)` compiles a network exactly as the reference describes it
(GraphNode list, named params, BN-ready flags; network.hpp:19-33) and `Plan.forward(x)` is the drop-in
for `Network<float>::forward(x, NormMode::eval)` (network.hpp:162): same input layout [B,T,F,C]
fp32, same output [B,T,F,bits] fp32, same error behaviour (ValueError <- std::invalid_argument,
RuntimeError <- std::runtime_error).

There is no CPU fallback: if libconetrx_cuda.so is missing or no CUDA device is present, creating a
plan raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

from . import graph as G

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CNRX_LIB") or os.path.join(HERE, "libconetrx_cuda.so")  # CNRX_LIB: A/B builds only

OK, ERR_INVALID_ARGUMENT, ERR_NOT_READY, ERR_UNSUPPORTED, ERR_CUDA = range(5)
FP32, BF16, FP16, BF16X3, FP16X3 = 0, 1, 2, 3, 4
# bf16x3 / fp16x3: split-precision tensor-core plans (fp32-grade LLRs, conv_x3.cu)
PRECISIONS = {"fp32": FP32, "bf16": BF16, "fp16": FP16, "bf16x3": BF16X3, "fp16x3": FP16X3}
MODE_TRAIN, MODE_EVAL = 0, 1


class CnrxError(RuntimeError):
    """Base class; subclasses mirror the reference's exception types."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class CnrxInvalidArgument(CnrxError, ValueError):
    pass


class CnrxNotReady(CnrxError):
    pass


class CnrxUnsupported(CnrxError):
    pass


class CnrxCudaError(CnrxError):
    pass


_ERRS = {ERR_INVALID_ARGUMENT: CnrxInvalidArgument, ERR_NOT_READY: CnrxNotReady,
         ERR_UNSUPPORTED: CnrxUnsupported, ERR_CUDA: CnrxCudaError}


class cnrx_node(C.Structure):
    _fields_ = [(n, C.c_int32) for n in
                ("op", "in0", "in1", "w", "b", "gamma", "beta", "rmean", "rvar", "bn_flag", "out_channels",
                 "dilation_f")]


class cnrx_param(C.Structure):
    _fields_ = [("name", C.c_char_p), ("rank", C.c_int32), ("learnable", C.c_int32), ("dims", C.c_int64 * 4),
                ("data", C.POINTER(C.c_float))]


class cnrx_plan_info(C.Structure):
    _fields_ = [("precision", C.c_int32), ("device", C.c_int32), ("n_launches", C.c_int32),
                ("n_tc_convs", C.c_int32), ("input_channels", C.c_int32), ("output_channels", C.c_int32),
                ("macs_per_re", C.c_int64), ("rows_per_slot", C.c_int64), ("workspace_bytes", C.c_int64)]


class cnrx_plan_options(C.Structure):
    _fields_ = [("struct_size", C.c_int32), ("fused_blocks", C.c_int32), ("fused_head", C.c_int32),
                ("tensor_core_head", C.c_int32), ("cta_pair", C.c_int32), ("weights_stationary", C.c_int32),
                ("relu_on_load", C.c_int32), ("cuda_core_stem", C.c_int32), ("pipeline_chunks", C.c_int32),
                ("pipeline_taper", C.c_float)]


OPTION_NAMES = [n for n, _ in cnrx_plan_options._fields_ if n != "struct_size"]


class cnrx_link(C.Structure):
    _fields_ = [("T", C.c_int32), ("F", C.c_int32), ("N", C.c_int32), ("mod_order", C.c_int32),
                ("n_taps", C.c_int32), ("pilot_spacing", C.c_int32), ("n_pilot_symbols", C.c_int32),
                ("has_interferer", C.c_int32), ("pilot_symbols", C.c_int32 * 8), ("rms_delay_s", C.c_double),
                ("tap_spacing_s", C.c_double), ("doppler_max_hz", C.c_double), ("scs_hz", C.c_double),
                ("cp_fraction", C.c_double), ("snr_db_lo", C.c_double), ("snr_db_hi", C.c_double),
                ("sir_db_lo", C.c_double), ("sir_db_hi", C.c_double)]


_lib = None

EXPORTED = ["cnrx_plan_create", "cnrx_plan_create_ex", "cnrx_plan_options_default", "cnrx_get_plan_options",
            "cnrx_plan_destroy", "cnrx_feature_plane_device", "cnrx_last_error", "cnrx_forward", "cnrx_forward_device",
            "cnrx_set_pilots", "cnrx_receive", "cnrx_receive_device", "cnrx_featurize_device",
            "cnrx_receive_sharded", "cnrx_forward_sharded", "cnrx_get_plan_info", "cnrx_set_graph_capture", "cnrx_launch_name",
            "cnrx_set_profiling", "cnrx_read_profile", "cnrx_launch_flops", "cnrx_generate_slots",
            "cnrx_count_bit_errors", "cnrx_slot_noise_var", "cnrx_classical_receive", "cnrx_ipc_alloc", "cnrx_ipc_open",
            "cnrx_ipc_close", "cnrx_ipc_free", "cnrx_ipc_read", "cnrx_ipc_read_async", "cnrx_plan_set_guard_bands",
            "cnrx_plan_check_guard_bands", "cnrx_plan_guard_band_ptr"]


def lib():
    """Load libconetrx_cuda.so (build it first with paper_2510_12739_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2510_12739_b200.build` "
                           "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, f32p, i64 = C.c_void_p, C.POINTER(C.c_float), C.c_int64
    L.cnrx_plan_create.restype = C.c_int
    L.cnrx_plan_create.argtypes = [C.POINTER(cnrx_node), C.c_int32, C.c_int32, C.c_int32, C.POINTER(cnrx_param),
                                   C.c_int32, C.POINTER(C.c_uint8), C.c_int32, C.c_int32, C.c_int32,
                                   C.POINTER(vp)]
    L.cnrx_plan_create_ex.argtypes = L.cnrx_plan_create.argtypes[:-1] + [C.POINTER(cnrx_plan_options), C.POINTER(vp)]
    L.cnrx_plan_options_default.argtypes = [C.POINTER(cnrx_plan_options)]
    L.cnrx_plan_options_default.restype = None
    L.cnrx_get_plan_options.argtypes = [vp, C.POINTER(cnrx_plan_options)]
    L.cnrx_feature_plane_device.argtypes = [vp, vp, i64, i64, i64, i64, vp, C.POINTER(C.c_int32)]
    L.cnrx_plan_destroy.argtypes = [vp]
    L.cnrx_plan_set_guard_bands.argtypes = [vp, C.c_int32]
    L.cnrx_plan_check_guard_bands.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    L.cnrx_plan_guard_band_ptr.argtypes = [vp, i64, C.c_int32, C.POINTER(vp)]
    L.cnrx_plan_destroy.restype = None
    L.cnrx_last_error.restype = C.c_char_p
    L.cnrx_forward.argtypes = [vp, f32p, i64, i64, i64, i64, C.c_int32, f32p]
    L.cnrx_forward_device.argtypes = [vp, vp, i64, i64, i64, i64, C.c_int32, vp, vp]
    L.cnrx_set_pilots.argtypes = [vp, i64, i64, f32p, C.POINTER(C.c_uint8)]
    L.cnrx_receive.argtypes = [vp, f32p, i64, i64, i64, i64, f32p]
    L.cnrx_receive_device.argtypes = [vp, vp, i64, i64, i64, i64, vp, vp]
    L.cnrx_ipc_alloc.argtypes = [C.c_int32, i64, C.POINTER(vp), C.c_void_p]
    L.cnrx_ipc_open.argtypes = [C.c_int32, C.c_void_p, C.POINTER(vp)]
    L.cnrx_ipc_close.argtypes = [C.c_int32, vp]
    L.cnrx_ipc_free.argtypes = [C.c_int32, vp]
    L.cnrx_ipc_read.argtypes = [C.c_int32, vp, vp, i64]
    L.cnrx_ipc_read_async.argtypes = [C.c_int32, vp, vp, i64, vp]
    L.cnrx_featurize_device.argtypes = [vp, vp, i64, i64, i64, i64, vp, vp]
    L.cnrx_receive_sharded.argtypes = [C.POINTER(vp), C.c_int32, f32p, i64, i64, i64, i64, f32p]
    L.cnrx_forward_sharded.argtypes = [C.POINTER(vp), C.c_int32, f32p, i64, i64, i64, i64, C.c_int32, f32p]
    L.cnrx_get_plan_info.argtypes = [vp, C.POINTER(cnrx_plan_info)]
    L.cnrx_set_graph_capture.argtypes = [vp, C.c_int32]
    L.cnrx_launch_name.restype = C.c_char_p
    L.cnrx_launch_name.argtypes = [vp, C.c_int32]
    L.cnrx_set_profiling.argtypes = [vp, C.c_int32]
    L.cnrx_launch_flops.argtypes = [vp, C.c_int32]
    L.cnrx_read_profile.argtypes = [vp, C.c_int32, C.POINTER(C.c_float), C.POINTER(C.c_int32),
                                    C.POINTER(C.c_int32)]
    L.cnrx_generate_slots.argtypes = [C.POINTER(cnrx_link), i64, C.c_uint64, C.c_uint64, vp, vp, vp, vp]
    L.cnrx_count_bit_errors.argtypes = [vp, vp, vp, i64, i64, i64, C.c_int32, vp, vp]
    L.cnrx_slot_noise_var.argtypes = [C.POINTER(cnrx_link), i64, C.c_uint64, C.c_uint64, f32p]
    L.cnrx_classical_receive.argtypes = [vp, vp, vp, vp, i64, i64, i64, i64, C.c_int32, vp, vp]
    for fn in EXPORTED:
        if fn not in ("cnrx_plan_destroy", "cnrx_last_error", "cnrx_launch_name", "cnrx_plan_options_default"):
            getattr(L, fn).restype = C.c_int
    L.cnrx_launch_flops.restype = C.c_int64
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc != OK:
        msg = lib().cnrx_last_error().decode()
        raise _ERRS.get(rc, CnrxError)(rc, msg)


def _f32p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _stream(stream: Optional[int]) -> C.c_void_p:
    """None -> the plan's own stream (NULL at the ABI); 0 (torch's legacy default stream handle) ->
    cudaStreamLegacy ((cudaStream_t)1); anything else is a cudaStream_t handle."""
    if stream is None:
        return C.c_void_p(0)
    return C.c_void_p(1 if stream == 0 else stream)


def default_options() -> dict:
    """cnrx_plan_options_default() as a dict (no environment overrides)."""
    o = cnrx_plan_options()
    lib().cnrx_plan_options_default(C.byref(o))
    return {n: getattr(o, n) for n in OPTION_NAMES}


class Plan:
    """A compiled CoNet-Rx network on one GPU.

    precision: "fp32" | "bf16" | "fp16".  options: None = cnrx_plan_create (defaults + the CNRX_* A/B
    environment switches); a dict = cnrx_plan_create_ex with the defaults updated by the dict (no
    environment)."""

    def __init__(self, g: "G.Graph", precision: str = "bf16", device: int = 0, options: Optional[dict] = None):
        L = lib()
        self.graph = g
        self.precision = precision
        self.device = device
        nodes = (cnrx_node * len(g.nodes))(*[cnrx_node(*n.as_row()) for n in g.nodes])
        self._keep = [np.ascontiguousarray(p.value, np.float32) for p in g.params]
        self._names = [p.name.encode() for p in g.params]
        params = (cnrx_param * max(1, len(g.params)))()
        for i, (p, v) in enumerate(zip(g.params, self._keep)):
            params[i].name = self._names[i]
            params[i].rank = v.ndim
            params[i].learnable = int(p.learnable)
            for d in range(v.ndim):
                params[i].dims[d] = v.shape[d]
            params[i].data = _f32p(v)
        ready = np.asarray(g.bn_ready if g.bn_ready else [0], np.uint8)
        h = C.c_void_p()
        prec = PRECISIONS[precision]
        args = (nodes, len(g.nodes), g.input_node, g.output_node, params, len(g.params),
                ready.ctypes.data_as(C.POINTER(C.c_uint8)), len(g.bn_ready), prec, device)
        if options is None:
            _check(L.cnrx_plan_create(*args, C.byref(h)))
        else:
            o = cnrx_plan_options()
            L.cnrx_plan_options_default(C.byref(o))
            for k, v in options.items():
                if k not in OPTION_NAMES:
                    raise ValueError(f"unknown plan option {k!r}")
                setattr(o, k, v)
            _check(L.cnrx_plan_create_ex(*args, C.byref(o), C.byref(h)))
        self.h = h
        self.out_channels = g.output_channels()
        self.in_channels = g.in_channels

    def close(self) -> None:
        if getattr(self, "h", None):
            lib().cnrx_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- Network<float>::forward ------------------------------------------------------------
    def forward(self, x: np.ndarray, mode: int = MODE_EVAL) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        if x.ndim == 3:
            x = x[None]
        if x.ndim != 4:
            raise CnrxInvalidArgument(ERR_INVALID_ARGUMENT,
                                      f"activation tensor must be [T,F,C] or [B,T,F,C], got {list(x.shape)}")
        B, T, F, Cc = x.shape
        out = np.empty((B, T, F, self.out_channels), np.float32)
        _check(lib().cnrx_forward(self.h, _f32p(x), B, T, F, Cc, mode, _f32p(out)))
        return out

    def forward_device(self, x, out, stream: Optional[int] = None, mode: int = MODE_EVAL) -> None:
        """x, out: torch CUDA tensors (fp32, contiguous)."""
        B, T, F, Cc = x.shape
        _check(lib().cnrx_forward_device(self.h, C.c_void_p(x.data_ptr()), B, T, F, Cc, mode,
                                         C.c_void_p(out.data_ptr()), _stream(stream)))

    # ---- receiver path (featurize -> subnets -> fusion -> head) --------------------------------
    def set_pilots(self, pilots: np.ndarray, mask: np.ndarray) -> None:
        p = np.ascontiguousarray(pilots, np.complex64)
        m = np.ascontiguousarray(mask, np.uint8)
        T, F = m.shape
        _check(lib().cnrx_set_pilots(self.h, T, F, p.view(np.float32).ctypes.data_as(C.POINTER(C.c_float)),
                                     m.ctypes.data_as(C.POINTER(C.c_uint8))))

    def receive(self, y: np.ndarray, out: Optional[np.ndarray] = None) -> np.ndarray:
        """y: complex64 [B,T,F,N] host array -> LLRs fp32 [B,T,F,bits] (host, synchronous)."""
        y = np.ascontiguousarray(y, np.complex64)
        B, T, F, N = y.shape
        if out is None:
            out = np.empty((B, T, F, self.out_channels), np.float32)
        _check(lib().cnrx_receive(self.h, y.view(np.float32).ctypes.data_as(C.POINTER(C.c_float)), B, T, F, N,
                                  _f32p(out)))
        return out

    def receive_host_ptr(self, y_ptr: int, shape, out_ptr: int) -> None:
        """Host-pointer variant (e.g. pinned torch tensors): y complex64 [B,T,F,N], out fp32."""
        B, T, F, N = shape
        _check(lib().cnrx_receive(self.h, C.cast(C.c_void_p(y_ptr), C.POINTER(C.c_float)), B, T, F, N,
                                  C.cast(C.c_void_p(out_ptr), C.POINTER(C.c_float))))

    def receive_device(self, y, out, stream: Optional[int] = None) -> None:
        """y: torch complex64 CUDA tensor [B,T,F,N] (or float32 [...,2]); out: fp32 CUDA tensor."""
        B, T, F, N = y.shape[:4]
        _check(lib().cnrx_receive_device(self.h, C.c_void_p(y.data_ptr()), B, T, F, N,
                                         C.c_void_p(out.data_ptr()), _stream(stream)))

    def receive_device_ptr(self, y, out_ptr: int, stream: Optional[int] = None) -> None:
        """receive_device with a raw LLR destination (e.g. a slice of a peer GPU's buffer opened with
        ipc_open: the head kernel's stores then go over NVLink)."""
        B, T, F, N = y.shape[:4]
        _check(lib().cnrx_receive_device(self.h, C.c_void_p(y.data_ptr()), B, T, F, N, C.c_void_p(out_ptr),
                                         _stream(stream)))

    def feature_plane(self, y) -> np.ndarray:
        """Test hook: the 16-bit input-feature plane of a bf16 / fp16 plan for y (torch complex64 CUDA
        tensor [B,T,F,N]) as float32 [B,T,F,cpad] (the bf16 / fp16 values, exactly)."""
        import torch
        B, T, F, N = y.shape[:4]
        cpad = C.c_int32()
        buf = torch.empty((B, T, F, 128), dtype=torch.int16, device=y.device)
        _check(lib().cnrx_feature_plane_device(self.h, C.c_void_p(y.data_ptr()), B, T, F, N,
                                               C.c_void_p(buf.data_ptr()), C.byref(cpad)))
        flat = buf.reshape(-1)[: B * T * F * cpad.value].reshape(B, T, F, cpad.value)
        dt = torch.float16 if self.precision == "fp16" else torch.bfloat16
        return flat.view(dt).float().cpu().numpy()

    def featurize_device(self, y, feat, stream: Optional[int] = None) -> None:
        B, T, F, N = y.shape[:4]
        _check(lib().cnrx_featurize_device(self.h, C.c_void_p(y.data_ptr()), B, T, F, N,
                                           C.c_void_p(feat.data_ptr()), _stream(stream)))

    # ---- debug: guard bands around every workspace buffer (include/conetrx_cuda.h) -------------------
    def set_guard_bands(self, enable: bool = True) -> None:
        _check(lib().cnrx_plan_set_guard_bands(self.h, 1 if enable else 0))

    def check_guard_bands(self):
        """(guarded buffers, canary bytes overwritten) -- the second must be 0."""
        n, bad = C.c_int64(), C.c_int64()
        _check(lib().cnrx_plan_check_guard_bands(self.h, C.byref(n), C.byref(bad)))
        return n.value, bad.value

    def guard_band_ptr(self, index: int, side: int) -> int:
        ptr = C.c_void_p()
        _check(lib().cnrx_plan_guard_band_ptr(self.h, index, side, C.byref(ptr)))
        return ptr.value

    # ---- introspection ----------------------------------------------------------------------------
    def options(self) -> dict:
        o = cnrx_plan_options()
        _check(lib().cnrx_get_plan_options(self.h, C.byref(o)))
        return {n: getattr(o, n) for n in OPTION_NAMES}

    def info(self) -> dict:
        inf = cnrx_plan_info()
        _check(lib().cnrx_get_plan_info(self.h, C.byref(inf)))
        return {f: getattr(inf, f) for f, _ in cnrx_plan_info._fields_}

    def launch_names(self):
        names, i = [], 0
        while True:
            n = lib().cnrx_launch_name(self.h, i)
            if n is None:
                return names
            names.append(n.decode())
            i += 1

    def launch_flops_per_re(self):
        return [int(lib().cnrx_launch_flops(self.h, i)) for i in range(len(self.launch_names()))]

    def set_profiling(self, enable: bool) -> None:
        _check(lib().cnrx_set_profiling(self.h, int(enable)))

    def read_profile(self, max_n: int = 4096):
        """[(kernel name, total ms, calls)] per launch position since the last read (single call: the
        library clears its accumulators on every read)."""
        n = C.c_int32()
        ms = (C.c_float * max_n)()
        cnt = (C.c_int32 * max_n)()
        _check(lib().cnrx_read_profile(self.h, max_n, ms, cnt, C.byref(n)))
        names = self.launch_names()
        k = min(n.value, max_n)
        return [(names[i] if i < len(names) else f"launch{i}", float(ms[i]), int(cnt[i])) for i in range(k)]

    def set_graph_capture(self, enable: bool) -> None:
        _check(lib().cnrx_set_graph_capture(self.h, int(enable)))


def forward_sharded(plans, x: np.ndarray, mode: int = MODE_EVAL) -> np.ndarray:
    """cnrx_forward_sharded: Network::forward over contiguous slot ranges of several single-GPU plans."""
    x = np.ascontiguousarray(x, np.float32)
    B, T, F, Cc = x.shape
    out = np.empty((B, T, F, plans[0].out_channels), np.float32)
    arr = (C.c_void_p * len(plans))(*[p.h for p in plans])
    _check(lib().cnrx_forward_sharded(arr, len(plans), _f32p(x), B, T, F, Cc, mode, _f32p(out)))
    return out


def receive_sharded(plans, y: np.ndarray) -> np.ndarray:
    """cnrx_receive_sharded: contiguous slot ranges over several single-GPU plans (one process)."""
    y = np.ascontiguousarray(y, np.complex64)
    B, T, F, N = y.shape
    out = np.empty((B, T, F, plans[0].out_channels), np.float32)
    arr = (C.c_void_p * len(plans))(*[p.h for p in plans])
    _check(lib().cnrx_receive_sharded(arr, len(plans), y.view(np.float32).ctypes.data_as(C.POINTER(C.c_float)),
                                      B, T, F, N, _f32p(out)))
    return out


# ---------------------------------------------------------------------------------------------
# On-GPU synthetic slots + BER (cnrx_generate_slots / cnrx_count_bit_errors)
# ---------------------------------------------------------------------------------------------
def link_struct(link) -> cnrx_link:
    """A paper_2510_12739_b200.graph.LinkSpec as the C ABI's cnrx_link."""
    require_ps = list(link.pilot_symbols)
    if len(require_ps) > 8:
        raise ValueError("at most 8 pilot symbols")
    ln = cnrx_link()
    ln.T, ln.F, ln.N, ln.mod_order, ln.n_taps = link.T, link.F, link.N, link.mod_order, link.n_taps
    ln.pilot_spacing, ln.n_pilot_symbols = link.pilot_spacing, len(require_ps)
    for i, t in enumerate(require_ps):
        ln.pilot_symbols[i] = t
    ln.has_interferer = 1 if link.sir_db is not None else 0
    ln.rms_delay_s, ln.tap_spacing_s, ln.doppler_max_hz = link.rms_delay_s, link.tap_spacing_s, link.doppler_max_hz
    ln.scs_hz, ln.cp_fraction = link.scs_hz, link.cp_fraction
    ln.snr_db_lo, ln.snr_db_hi = link.snr_db
    if link.sir_db is not None:
        ln.sir_db_lo, ln.sir_db_hi = link.sir_db
    return ln


def generate_slots_device(link, B: int, seed: int, slot0: int = 0, with_h: bool = False,
                          stream: Optional[int] = None):
    """Synthetic slots generated on the current CUDA device -> (y complex64 [B,T,F,N], bits uint8
    [B,T,F,b][, h complex64 [B,T,F,N]]) torch tensors.  Asynchronous on `stream` (default: torch's
    current stream)."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    y = torch.empty((B, link.T, link.F, link.N), dtype=torch.complex64, device=dev)
    bits = torch.empty((B, link.T, link.F, link.bits), dtype=torch.uint8, device=dev)
    h = torch.empty_like(y) if with_h else None
    st = torch.cuda.current_stream().cuda_stream if stream is None else stream
    ln = link_struct(link)
    _check(lib().cnrx_generate_slots(C.byref(ln), B, seed, slot0, y.data_ptr(), bits.data_ptr(),
                                     h.data_ptr() if h is not None else None, _stream(st)))
    return (y, bits, h) if with_h else (y, bits)


def count_bit_errors(llr, bits, data_mask, stream: Optional[int] = None):
    """Per-slot hard-decision bit errors over data REs, on the device: llr [B,T,F,b] fp32, bits
    [B,T,F,b] uint8, data_mask [T,F] (bool/uint8, 1 = data RE) -> int64 tensor [B]."""
    import torch
    B, T, F, nb = llr.shape
    mask = data_mask.to(device=llr.device, dtype=torch.uint8).contiguous()
    err = torch.empty((B,), dtype=torch.int64, device=llr.device)
    st = torch.cuda.current_stream().cuda_stream if stream is None else stream
    _check(lib().cnrx_count_bit_errors(llr.contiguous().data_ptr(), bits.contiguous().data_ptr(), mask.data_ptr(),
                                       B, T, F, nb, err.data_ptr(), _stream(st)))
    return err


def slot_noise_var(link, B: int, seed: int, slot0: int = 0) -> np.ndarray:
    """Per-slot noise-plus-interference variance of generate_slots_device's slots (host, fp32 [B])."""
    out = np.empty(B, np.float32)
    ln = link_struct(link)
    _check(lib().cnrx_slot_noise_var(C.byref(ln), B, seed, slot0, _f32p(out)))
    return out


def classical_receive_device(plan: "Plan", y, noise_var, mod_order: int, h=None, out=None,
                             stream: Optional[int] = None):
    """LS-LMMSE (h=None, the plan's pilot grid) or perfect-CSI LMMSE + max-log LLRs on the device:
    y / h complex64 [B,T,F,N] torch tensors, noise_var fp32 [B] -> llr fp32 [B,T,F,bits]."""
    import torch
    B, T, F, N = y.shape
    bits = {4: 2, 16: 4, 64: 6}[mod_order]
    if out is None:
        out = torch.empty((B, T, F, bits), dtype=torch.float32, device=y.device)
    nv = torch.as_tensor(noise_var, dtype=torch.float32).to(y.device).contiguous()
    st = torch.cuda.current_stream().cuda_stream if stream is None else stream
    _check(lib().cnrx_classical_receive(plan.h, y.contiguous().data_ptr(),
                                        h.contiguous().data_ptr() if h is not None else None, nv.data_ptr(), B, T, F, N,
                                        mod_order, out.data_ptr(), _stream(st)))
    return out


# ---- peer-memory LLR gather (include/conetrx_cuda.h cnrx_ipc_*) -------------------------------------------
def ipc_alloc(device: int, nbytes: int):
    """Allocate `nbytes` on `device` and export it: returns (device pointer, 64-byte handle)."""
    ptr = C.c_void_p()
    h = (C.c_uint8 * 64)()
    _check(lib().cnrx_ipc_alloc(device, nbytes, C.byref(ptr), C.cast(h, C.c_void_p)))
    return ptr.value, bytes(h)


def ipc_open(device: int, handle: bytes) -> int:
    """Map another process's exported allocation into this process (peer access enabled lazily)."""
    h = (C.c_uint8 * 64).from_buffer_copy(handle)
    ptr = C.c_void_p()
    _check(lib().cnrx_ipc_open(device, C.cast(h, C.c_void_p), C.byref(ptr)))
    return ptr.value


def ipc_close(device: int, ptr: int) -> None:
    _check(lib().cnrx_ipc_close(device, C.c_void_p(ptr)))


def ipc_read(device: int, ptr: int, host_ptr: int, nbytes: int) -> None:
    _check(lib().cnrx_ipc_read(device, C.c_void_p(ptr), C.c_void_p(host_ptr), nbytes))


def ipc_read_async(device: int, ptr: int, host_ptr: int, nbytes: int, stream: int) -> None:
    _check(lib().cnrx_ipc_read_async(device, C.c_void_p(ptr), C.c_void_p(host_ptr), nbytes, C.c_void_p(stream)))


def ipc_free(device: int, ptr: int) -> None:
    _check(lib().cnrx_ipc_free(device, C.c_void_p(ptr)))
