"""On-GPU synthetic slots + BER counting (csrc/slotgen.cu) against the CPU restatement oracle/slotgen.py."""
import dataclasses

import numpy as np
import pytest

import oracle.slotgen as S
from paper_2510_12739_b200 import graph as G
from paper_2510_12739_b200 import slots


# ------------------------------------------------------------------------------------------------
# CPU: the oracle itself
# ------------------------------------------------------------------------------------------------
def test_philox_known_answers():
    """Philox4x32-10 known-answer vectors published with the algorithm (Random123 kat_vectors)."""
    kat = [((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
           ((0xFFFFFFFF,) * 4, (0xFFFFFFFF, 0xFFFFFFFF), (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
           ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
            (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1))]
    for ctr, key, want in kat:
        got = S.philox4x32_10(np.array([ctr[0]]), ctr[1], ctr[2], ctr[3], *key)
        assert tuple(int(v[0]) for v in got) == want


def _small(name, F):
    return dataclasses.replace(G.CONFIGS[name].link, F=F)


def test_oracle_slots_are_independent_and_pilots_clean():
    link = _small("cfg2", 48)
    y3, b3 = S.generate(link, 3, 77, slot0=5)
    y1, b1 = S.generate(link, 1, 77, slot0=7)
    assert np.array_equal(y3[2], y1[0]) and np.array_equal(b3[2], b1[0])
    pmask, pvals = slots.pilot_pattern(link.T, link.F, link.pilot_symbols, link.pilot_spacing)
    assert not b3[:, pmask != 0].any()
    # unit average symbol energy and the SNR range show up in the noise power at pilots-free REs
    assert 0.2 < np.mean(np.abs(y3) ** 2) < 5.0


def test_oracle_bit_errors_matches_slots_ber():
    link = _small("cfg1", 72)
    y, bits = S.generate(link, 2, 3)
    pmask, _ = slots.pilot_pattern(link.T, link.F, link.pilot_symbols, link.pilot_spacing)
    llr = np.random.default_rng(0).standard_normal(bits.shape).astype(np.float32)
    err = S.bit_errors(llr, bits, pmask == 0)
    hb = (llr > 0).astype(np.uint8)
    assert err.sum() == (hb[:, pmask == 0] != bits[:, pmask == 0]).sum()


# ------------------------------------------------------------------------------------------------
# GPU: device generator and error counts
# ------------------------------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("name,F,B", [("cfg1", 72, 3), ("cfg2", 96, 3), ("cfg3", 120, 2)])
def test_device_slots_match_oracle(name, F, B):
    import torch
    from paper_2510_12739_b200 import plan as P
    link = _small(name, F)
    y, bits, h = P.generate_slots_device(link, B, 1234, slot0=9, with_h=True)
    torch.cuda.synchronize()
    yo, bo, ho = S.generate(link, B, 1234, slot0=9, with_h=True)
    assert np.array_equal(bits.cpu().numpy(), bo)  # integer work: bit-exact
    # fp32 on the device vs float64 here: phases, 20-sinusoid sums, 23-tap sums, Box-Muller
    np.testing.assert_allclose(h.cpu().numpy(), ho, rtol=0, atol=1e-4)
    np.testing.assert_allclose(y.cpu().numpy(), yo, rtol=0, atol=2e-4)


@pytest.mark.gpu
def test_device_slots_independent_of_batching():
    import torch
    from paper_2510_12739_b200 import plan as P
    link = _small("cfg2", 64)
    y4, b4 = P.generate_slots_device(link, 4, 99, slot0=100)
    for k in (0, 3):
        y1, b1 = P.generate_slots_device(link, 1, 99, slot0=100 + k)
        assert torch.equal(y4[k], y1[0]) and torch.equal(b4[k], b1[0])


@pytest.mark.gpu
def test_receive_and_count_errors_on_device_matches_host_path():
    """Generate -> receive -> count, all on the GPU, equals the host path (same y, LLRs from the same
    plan, errors counted by the oracle)."""
    import torch
    from paper_2510_12739_b200 import plan as P
    link = _small("cfg2", 96)
    g = G.CONFIGS["cfg2"].graph(seed=3)
    p = P.Plan(g, "bf16")
    pmask, pvals = slots.pilot_pattern(link.T, link.F, link.pilot_symbols, link.pilot_spacing)
    p.set_pilots(pvals.astype(np.complex64), pmask)
    y, bits = P.generate_slots_device(link, 5, 42)
    llr = torch.empty((5, link.T, link.F, link.bits), dtype=torch.float32, device="cuda")
    p.receive_device(y, llr, torch.cuda.current_stream().cuda_stream)
    err = P.count_bit_errors(llr, bits, torch.from_numpy(pmask == 0))
    torch.cuda.synchronize()
    want = S.bit_errors(llr.cpu().numpy(), bits.cpu().numpy(), pmask == 0)
    assert np.array_equal(err.cpu().numpy(), want)
    assert np.array_equal(p.receive(y.cpu().numpy()), llr.cpu().numpy())


@pytest.mark.gpu
def test_count_errors_crafted():
    import torch
    from paper_2510_12739_b200 import plan as P
    rng = np.random.default_rng(5)
    B, T, F, nb = 3, 14, 40, 4
    bits = rng.integers(0, 2, (B, T, F, nb)).astype(np.uint8)
    mask = np.ones((T, F), bool)
    mask[2, ::2] = False
    llr = np.where(bits == 1, 1.0, -1.0).astype(np.float32)
    flips = rng.random(bits.shape) < 0.01
    llr[flips] *= -1
    llr[0, 0, 0, 0] = 0.0  # LLR 0 decides bit 0
    err = P.count_bit_errors(torch.from_numpy(llr).cuda(), torch.from_numpy(bits).cuda(), torch.from_numpy(mask))
    assert np.array_equal(err.cpu().numpy(), S.bit_errors(llr, bits, mask))
