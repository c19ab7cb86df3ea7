"""Generate the committed golden fixtures from the REFERENCE itself (oracle/_ref, compiled in place from
/root/reference).  Run here (where /root/reference exists):   python tests/golden/make_golden.py

The reference ships no tests or golden vectors, so parity is pinned on outputs of
the reference's own code on seeded inputs:
  * forward.npz  — conetrx::Network<float>::forward (network.hpp:162) LLRs for cfg1 / cfg2 / cfg4
                   graphs (small grids) with seeded weights, BN statistics and inputs; plus the
                   build_reference_main fusion-identity case (network.hpp:567, overrides :159-178)
  * phy.npz      — Rng streams (rng.hpp:14-69), qam_map (qam.cpp:42-52) for every label of 4/16/64-QAM,
                   pilot_pattern (pilots.cpp:13-31), tdl_tap_powers (channel.cpp:37-50)
Weights are regenerated deterministically by paper_2510_12739_b200.graph (seeded numpy), so only
inputs and outputs are stored.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))

import oracle  # noqa: E402
from paper_2510_12739_b200 import graph as G  # noqa: E402

# (config, weight seed, input seed, B, F)
FORWARD_CASES = [("cfg1", 11, 101, 2, 72), ("cfg2", 12, 102, 2, 20), ("cfg4", 13, 103, 1, 16)]


def forward_cases():
    out = {}
    for name, wseed, xseed, B, F in FORWARD_CASES:
        cfg = G.CONFIGS[name]
        g = cfg.graph(seed=wseed)
        x = np.random.default_rng(xseed).standard_normal((B, 14, F, g.in_channels)).astype(np.float32)
        net = oracle.RefNet.from_graph(g)
        out[f"{name}_x"] = x
        out[f"{name}_llr"] = net.forward(x)
        out[f"{name}_llr_concurrent"] = net.forward(x, concurrent=True)
    # fusion identity: CoNet with every support activation forced to 1 at the mul
    # fusion points equals build_reference_main with the same main-path parameters
    spec = G.conet_template(16, 2, [2], "mul", "bn", False, 6, 2, "standard", 3)
    g = G.build_conet(spec).init_he_normal(21, randomize_aux=True)
    x = np.random.default_rng(121).standard_normal((1, 14, 12, 6)).astype(np.float32)
    net = oracle.RefNet.from_graph(g)
    ov = {op: 1.0 for (_, op, _) in g.fusion_meta}
    out["fusion_identity_x"] = x
    out["fusion_identity_llr"] = net.forward_overrides(x, ov)
    gm = G.build_reference_main(spec)
    gm.copy_params_from(g)
    gm.bn_ready = [1] * len(gm.bn_ready)
    out["fusion_identity_main_llr"] = oracle.RefNet.from_graph(gm).forward(x)
    return out


def phy_cases():
    import ctypes as C
    R = oracle.ref()
    out = {}
    u64 = (C.c_uint64 * 16)()
    R.ref_rng_u64(12345, 16, u64)
    out["rng_u64_seed12345"] = np.array(list(u64), dtype=np.uint64)
    uni = np.zeros(16, np.float64)
    R.ref_rng_uniform(7, 16, uni.ctypes.data_as(C.POINTER(C.c_double)))
    out["rng_uniform_seed7"] = uni
    out["rng_derive"] = np.array([R.ref_rng_derive(1, i) for i in range(8)], dtype=np.uint64)
    for order in (4, 16, 64):
        nb = {4: 2, 16: 4, 64: 6}[order]
        pts = np.zeros((order, 2), np.float64)
        for label in range(order):
            bits = np.array([(label >> (nb - 1 - i)) & 1 for i in range(nb)], np.uint8)
            v = np.zeros(2, np.float64)
            R.ref_qam_map(bits.ctypes.data_as(C.POINTER(C.c_uint8)), order, v.ctypes.data_as(C.POINTER(C.c_double)))
            pts[label] = v
        out[f"qam{order}"] = pts
    for (T, F, sym, sp) in [(14, 64, 2, 2), (14, 72, 2, 2), (14, 612, 2, 2)]:
        mask = np.zeros(T * F, np.uint8)
        vals = np.zeros(2 * T * F, np.float64)
        R.ref_pilot_pattern(T, F, sym, sp, mask.ctypes.data_as(C.POINTER(C.c_uint8)),
                            vals.ctypes.data_as(C.POINTER(C.c_double)))
        out[f"pilots_T{T}_F{F}_mask"] = mask.reshape(T, F)
        out[f"pilots_T{T}_F{F}_values"] = vals.reshape(T, F, 2)
    tp = np.zeros(16, np.float64)
    R.ref_tdl_tap_powers(300e-9, 1.0 / (64 * 30e3), 16, tp.ctypes.data_as(C.POINTER(C.c_double)))
    out["tap_powers_300ns_F64"] = tp
    return out


if __name__ == "__main__":
    np.savez_compressed(os.path.join(HERE, "forward.npz"), **forward_cases())
    np.savez_compressed(os.path.join(HERE, "phy.npz"), **phy_cases())
    for f in ("forward.npz", "phy.npz"):
        print(f, os.path.getsize(os.path.join(HERE, f)), "bytes")
