"""The plan's own bounds check over every kernel family (SURVEY.md §5 asks for compute-sanitizer memcheck on
the kernels; the GPU pool has it closed, so plans run with guard bands: cnrx_plan_set_guard_bands /
cnrx_plan_check_guard_bands in include/conetrx_cuda.h).  Every case runs the receive path through the C
ABI with 256 KB canary bands around each workspace buffer and canary-filled margins around the caller's
LLR buffer, over a grow / shrink / reuse sequence of batch sizes, checks the LLRs against the oracle
(reference forward, network.hpp:162-180, on the restated features) and requires every canary intact."""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tools"))

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", ["cfg2", "cfg2_ws", "cfg2_fh", "cfg2_x3", "cfg1", "cfg4", "cfg2_full", "cfg3"])
def test_no_write_outside_buffers(case):
    import sanitize_run as S
    results = S.CASES[case]()
    assert results and all(nbuf > 0 and bad == 0 for _, nbuf, bad, _ in results)


def test_guard_bands_detect_an_overrun():
    """The check itself: a deliberate write just past a guarded plane must be counted."""
    import dataclasses

    import torch
    from paper_2510_12739_b200 import graph as G, plan as P, slots

    cfg = G.CONFIGS["cfg2"]
    batch = slots.generate(dataclasses.replace(cfg.link, F=24), 1, seed=1)
    p = P.Plan(cfg.graph(seed=1), "bf16", device=0, options={})
    with pytest.raises(P.CnrxError):
        p.check_guard_bands()  # off by default
    p.set_guard_bands(True)
    p.set_pilots(batch.pilots, batch.pilot_mask)
    llr = p.receive(batch.y)
    nbuf, bad = p.check_guard_bands()
    assert nbuf > 0 and bad == 0
    # overwrite 8 canary bytes just past the last guarded buffer and 3 just before the first
    junk = torch.zeros(8, dtype=torch.uint8, device="cuda")
    import ctypes
    rt = ctypes.CDLL("libcudart.so.12")
    for idx, side, off, n in ((nbuf - 1, 1, 0, 8), (0, 0, (256 << 10) - 3, 3)):
        dst = p.guard_band_ptr(idx, side) + off
        assert rt.cudaMemcpy(ctypes.c_void_p(dst), ctypes.c_void_p(junk.data_ptr()), ctypes.c_size_t(n), 3) == 0
    torch.cuda.synchronize()
    assert p.check_guard_bands() == (nbuf, 11)
    with pytest.raises(P.CnrxError):
        p.guard_band_ptr(nbuf, 0)
    # switching the mode off frees the guarded workspace; results are unchanged
    p.set_guard_bands(False)
    import numpy as np
    assert np.array_equal(p.receive(batch.y), llr)
