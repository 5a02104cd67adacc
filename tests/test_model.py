"""Model files + transform against the reference's own bytes
(tests/golden/formats.npz, written by axemu.transform + axemu.save_model)."""

import json

import numpy as np
import pytest

from cases import model_graph_spec
from golden_io import load_golden
from paper_2002_09481_b200 import model as Mo
from paper_2002_09481_b200 import types as T
from paper_2002_09481_b200.formats import FormatError


def _float_graph():
    return [Mo.node(i, k, ins, **a) for i, k, ins, a in model_graph_spec()]


def test_transform_report_and_structure():
    tg, rep = Mo.transform(_float_graph(), T.truncated_lut(T.Signedness.SIGNED, 2))
    g = load_golden("formats")
    assert [rep.replaced_count, rep.inserted_min_max] == g["model_transform_report"].tolist()
    assert rep.untouched_kinds == ["Add", "AvgPool", "Input", "ReLU"]
    ax = [n for n in tg if n["kind"] == "AxConv2D"]
    assert [n["inputs"] for n in ax][0] == ["in", "c1.in_min", "c1.in_max"]
    assert all(n["attrs"]["f_min"] == float(n["attrs"]["filters"].min()) for n in ax)


def test_save_model_bytes_match_reference(tmp_path):
    """Same JSON document, same float32 sidecar, same .axm as the reference's save_model."""
    import hashlib

    tg, _ = Mo.transform(_float_graph(), T.truncated_lut(T.Signedness.SIGNED, 2))
    Mo.save_model(tg, tmp_path / "ax.json")
    g = load_golden("formats")
    assert (tmp_path / "ax.json").read_bytes() == g["model_json"].tobytes()
    assert (tmp_path / "ax.weights.bin").read_bytes() == g["model_weights"].tobytes()
    assert hashlib.sha256((tmp_path / "ax.axm").read_bytes()).digest() == g["model_axm_sha"].tobytes()


def test_load_reference_model(tmp_path):
    g = load_golden("formats")
    (tmp_path / "ax.json").write_bytes(g["model_json"].tobytes())
    (tmp_path / "ax.weights.bin").write_bytes(g["model_weights"].tobytes())
    T_lut = T.truncated_lut(T.Signedness.SIGNED, 2)
    from paper_2002_09481_b200.formats import save_lut

    save_lut(T_lut, tmp_path / "ax.axm")
    nodes = Mo.load_model(tmp_path / "ax.json")
    want, _ = Mo.transform(_float_graph(), T_lut)
    assert [(n["id"], n["kind"], n["inputs"]) for n in nodes] == [(n["id"], n["kind"], n["inputs"]) for n in want]
    for a, b in zip(nodes, want):
        for k, v in b["attrs"].items():
            if isinstance(v, np.ndarray):
                assert np.array_equal(a["attrs"][k], v)
            elif k == "lut":
                assert np.array_equal(a["attrs"][k].entries, v.entries)
            else:
                assert a["attrs"][k] == (list(v) if isinstance(v, tuple) else v)


def test_validation_messages():
    g = _float_graph()
    with pytest.raises(ValueError, match="duplicate node id"):
        Mo.validate(g + [g[1]])
    with pytest.raises(ValueError, match="does not precede"):
        Mo.validate([Mo.node("a", "ReLU", ["b"])])
    with pytest.raises(ValueError, match="needs data, min, and max"):
        Mo.validate([Mo.node("in", "Input"), Mo.node("c", "AxConv2D", ["in"])])
    clash = [Mo.node("in", "Input"), Mo.node("c1.in_min", "ReLU", ["in"]),
             Mo.node("c1", "Conv2D", ["in"], filters=np.zeros((1, 1, 3, 1), np.float32))]
    with pytest.raises(ValueError, match="already taken"):
        Mo.transform(clash, T.exact_lut(T.Signedness.SIGNED))


def test_model_file_errors(tmp_path):
    Mo.save_model(_float_graph(), tmp_path / "m.json")
    doc = json.loads((tmp_path / "m.json").read_text())
    doc["nodes"][0]["kind"] = "BatchNorm"
    (tmp_path / "m.json").write_text(json.dumps(doc))
    with pytest.raises(FormatError, match="BatchNorm"):
        Mo.load_model(tmp_path / "m.json")
    (tmp_path / "m.json").write_text('{"format": "something-else"}')
    with pytest.raises(FormatError, match="not a model"):
        Mo.load_model(tmp_path / "m.json")
    (tmp_path / "m.json").write_text("{oops")
    with pytest.raises(FormatError, match="malformed"):
        Mo.load_model(tmp_path / "m.json")
