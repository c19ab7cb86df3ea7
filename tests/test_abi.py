"""The C-ABI library loads on a CPU-only host and exports every symbol include/conetrx_cuda.h declares;
without a GPU, creating a plan fails loudly (no CPU fallback)."""
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2510_12739_b200 import graph as G, plan as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "conetrx_cuda.h")).read()
    return sorted(set(re.findall(r"\b(cnrx_[a-z_]+)\s*\(", src)))


def test_library_exports_header_symbols():
    if not os.path.exists(P.LIB_PATH):
        pytest.skip("libconetrx_cuda.so not built")
    out = subprocess.run(["nm", "-D", "--defined-only", P.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (cnrx_[a-z_]+)", out))
    missing = [f for f in header_functions() if f not in exported]
    assert not missing, missing
    assert set(P.EXPORTED) <= exported
    P.lib()  # loads


def test_plan_create_without_gpu_fails_loudly():
    if not os.path.exists(P.LIB_PATH):
        pytest.skip("libconetrx_cuda.so not built")
    from conftest import gpu_available
    if gpu_available():
        pytest.skip("a GPU is present")
    g = G.CONFIGS["cfg1"].graph()
    with pytest.raises(P.CnrxError):
        P.Plan(g, "fp32")


def test_no_oracle_import_in_product():
    """The product package never imports the oracle (test infrastructure only)."""
    pkg = os.path.join(ROOT, "paper_2510_12739_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".h", ".cuh")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "liboracle" not in txt and "_ref/" not in txt, f


def test_plan_options_defaults_and_abi_check():
    """cnrx_plan_options_default (no GPU needed) and the struct_size guard of cnrx_plan_create_ex, which
    rejects a caller compiled against another header version before touching the device."""
    if not os.path.exists(P.LIB_PATH):
        pytest.skip("libconetrx_cuda.so not built")
    import ctypes as C
    d = P.default_options()
    assert d == {"fused_blocks": 1, "fused_head": 0, "tensor_core_head": 0, "cta_pair": 1, "weights_stationary": 1,
                 "relu_on_load": 1, "cuda_core_stem": 0, "pipeline_chunks": 0, "pipeline_taper": pytest.approx(0.125)}
    o = P.cnrx_plan_options()
    P.lib().cnrx_plan_options_default(C.byref(o))
    assert o.struct_size == C.sizeof(P.cnrx_plan_options)
    o.struct_size -= 4
    g = G.CONFIGS["cfg1"].graph()
    node = (P.cnrx_node * len(g.nodes))(*[P.cnrx_node(*n.as_row()) for n in g.nodes])
    h = C.c_void_p()
    rc = P.lib().cnrx_plan_create_ex(node, len(g.nodes), g.input_node, g.output_node, None, 0, None, 0, P.BF16, 0,
                                     C.byref(o), C.byref(h))
    assert rc == P.ERR_INVALID_ARGUMENT and "struct_size" in P.lib().cnrx_last_error().decode()
    with pytest.raises(ValueError, match="unknown plan option"):
        P.Plan(g, "fp32", options={"no_such_option": 1})
