"""Spec files, width solving and CNCK checkpoints (paper_2510_12739_b200/files.py) pinned against the
reference built in place (oracle/_ref: netspec.cpp, checkpoint.cpp, network.hpp)."""
import os

import numpy as np
import pytest

from paper_2510_12739_b200 import files as Fi
from paper_2510_12739_b200 import graph as G

SPECS = [
    '{}',
    '{"template": "deeprx", "width": 48, "blocks": 3, "in_channels": 12, "bits": 4, "kernel": 1}',
    '{"template": "conet", "width": 64, "main_blocks": 4, "support_blocks": [4, 4], "fusion_points": [3],'
    ' "in_channels": 12, "bits": 4, "kernel": 1}',
    '{"template": "conet", "width": 32, "main_blocks": 3, "support_blocks": 2, "fusion_op": "concat",'
    ' "fusion_norm": "ln", "bidirectional": true, "conv": "depthwise", "in_channels": 6, "bits": 2}',
    '{"template": "conet", "width": 16, "main_blocks": 2, "support_blocks": [1, 2], "fusion_op": "add",'
    ' "target_params": 50000}',
]


@pytest.fixture(scope="module")
def R(ref):
    if ref is None:
        pytest.skip("reference build (oracle/_ref) not available")
    import oracle
    return oracle


@pytest.mark.parametrize("text", SPECS)
def test_spec_json_canonical_text_matches_reference(R, text):
    assert Fi.spec_file_to_json(Fi.parse_spec_file_json(text)) == R.spec_to_json(text)


@pytest.mark.parametrize("text", SPECS[:4])
def test_graph_from_spec_matches_reference(R, text):
    g = Fi.graph_from_spec(Fi.parse_spec_file_json(text))
    rn = R.RefNet.from_spec(text)
    assert np.array_equal(g.node_array()[:, :11], rn.nodes())
    assert [(p.name, tuple(p.value.shape), p.learnable) for p in g.params] == rn.params()
    assert g.learnable_count() == rn.learnable_count()


@pytest.mark.parametrize("text,target", [(SPECS[2], 891588), (SPECS[1], 200000), (SPECS[4], 50000),
                                         (SPECS[3], 123456)])
def test_width_solver_matches_reference(R, text, target):
    f = Fi.parse_spec_file_json(text)
    r = Fi.solve_spec_width(f, target)
    assert (r.found, r.width, r.params if r.found else 0, r.lo_width, r.hi_width) == \
        tuple(v if i != 2 or r.found else 0 for i, v in enumerate(R.solve_spec_width(text, target)))


@pytest.mark.parametrize("text,msg", [
    ('{"template": "resnet"}', "spec template must be deeprx or conet"),
    ('{"fusion_op": "max"}', "unknown fusion op 'max' (expected mul|add|concat)"),
    ('{"fusion_norm": "gn"}', "unknown norm kind 'gn' (expected bn|ln)"),
    ('{"conv": "grouped"}', "unknown conv kind 'grouped' (expected standard|depthwise)"),
])
def test_spec_errors_match_reference(R, text, msg):
    with pytest.raises(ValueError) as e:
        Fi.parse_spec_file_json(text)
    assert str(e.value) == msg
    with pytest.raises(R.RefError) as e2:
        R.spec_to_json(text)
    assert str(e2.value) == msg


def _random_graph(text, seed):
    g = Fi.graph_from_spec(Fi.parse_spec_file_json(text))
    g.init_he_normal(seed, randomize_aux=True)
    g.bn_ready[::2] = [0] * len(g.bn_ready[::2])  # a mix of ready / not-ready flags
    return g


@pytest.mark.parametrize("text", SPECS[1:4])
def test_checkpoint_written_by_reference_loads_bitwise(R, tmp_path, text):
    g = _random_graph(text, 3)
    rn = R.RefNet.from_spec(text)
    rn.load_params(g)
    path = str(tmp_path / "ref.cnck")
    rn.save_checkpoint(path)
    h = Fi.graph_from_spec(Fi.parse_spec_file_json(text))
    Fi.load_checkpoint(h, path)
    for p, q in zip(g.params, h.params):
        assert p.name == q.name and np.array_equal(p.value, q.value)
    assert h.bn_ready == g.bn_ready == rn.bn_ready()


@pytest.mark.parametrize("text", SPECS[1:4])
def test_checkpoint_written_here_is_byte_identical_and_loads_in_reference(R, tmp_path, text):
    g = _random_graph(text, 4)
    ours, theirs = str(tmp_path / "ours.cnck"), str(tmp_path / "theirs.cnck")
    Fi.save_checkpoint(g, ours)
    rn = R.RefNet.from_spec(text)
    rn.load_params(g)
    rn.save_checkpoint(theirs)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    fresh = R.RefNet.from_spec(text)
    fresh.load_checkpoint(ours)
    for (name, v), p in zip(fresh.param_values(), g.params):
        assert name == p.name and np.array_equal(v, p.value)
    assert fresh.bn_ready() == g.bn_ready


def test_checkpoint_errors_match_reference(R, tmp_path):
    text = SPECS[1]
    g = _random_graph(text, 5)
    good = str(tmp_path / "good.cnck")
    Fi.save_checkpoint(g, good)
    data = open(good, "rb").read()
    cases = {
        "magic.cnck": b"XNCK" + data[4:],
        "version.cnck": data[:4] + (2).to_bytes(4, "little") + data[8:],
        "truncated.cnck": data[:len(data) // 2],
    }
    other = _random_graph(SPECS[2], 5)  # a checkpoint of a different network
    Fi.save_checkpoint(other, str(tmp_path / "other.cnck"))
    paths = {k: str(tmp_path / k) for k in cases}
    for k, v in cases.items():
        open(paths[k], "wb").write(v)
    paths["other.cnck"] = str(tmp_path / "other.cnck")
    paths["missing.cnck"] = str(tmp_path / "does_not_exist.cnck")
    for k, path in paths.items():
        h = Fi.graph_from_spec(Fi.parse_spec_file_json(text))
        with pytest.raises((RuntimeError, ValueError)) as e:
            Fi.load_checkpoint(h, path)
        rn = R.RefNet.from_spec(text)
        with pytest.raises(R.RefError) as e2:
            rn.load_checkpoint(path)
        assert str(e.value) == str(e2.value), k


def test_spec_file_round_trip_and_load(tmp_path):
    f = Fi.parse_spec_file_json(SPECS[2])
    path = str(tmp_path / "net.json")
    open(path, "w").write(Fi.spec_file_to_json(f))
    assert Fi.load_spec_file(path) == f
    with pytest.raises(RuntimeError, match="cannot open net spec file"):
        Fi.load_spec_file(str(tmp_path / "nope.json"))
    # cfg2's network is exactly this spec file (the bench config as a file a user could ship)
    g = Fi.graph_from_spec(f)
    c = G.CONFIGS["cfg2"].graph_fn()
    assert np.array_equal(g.node_array(), c.node_array())
    assert [p.name for p in g.params] == [p.name for p in c.params]


@pytest.mark.gpu
def test_plan_from_files_runs_reference_checkpoint(R, tmp_path):
    """Spec file + a CNCK checkpoint written by the reference -> GPU plan: fp32 bit-exact with the
    reference's own forward of the same loaded network."""
    from paper_2510_12739_b200 import plan as P
    text = SPECS[2]
    g = _random_graph(text, 7)
    g.bn_ready = [1] * len(g.bn_ready)
    rn = R.RefNet.from_spec(text)
    rn.load_params(g)
    ck, sp = str(tmp_path / "w.cnck"), str(tmp_path / "net.json")
    rn.save_checkpoint(ck)
    open(sp, "w").write(text)
    x = np.random.default_rng(1).standard_normal((2, 14, 24, 12)).astype(np.float32)
    p = Fi.plan_from_files(sp, ck, "fp32")
    assert np.array_equal(p.forward(x), rn.forward(x))
