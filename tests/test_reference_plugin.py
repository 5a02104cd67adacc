"""The reference's own executor driving the B200 engine: INTEGRATION.md section 1 applied to the real
``axemu`` package (installed into baseline/_ref), then ``axemu.graph.run(...,
engine="b200")`` on the acceptance criterion-1 stream and a calibrated ResNet-8, bit-exact with the
reference's own outputs (tests/golden).  The patch is the three-line change of graph.py:221-226."""

import os
import sys
import types
from pathlib import Path

import numpy as np
import pytest

from conftest import cuda_ok
from golden_io import bits_equal, load_golden

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device"),
              pytest.mark.skipif(not (REF / "axemu").is_dir(), reason="reference not installed in baseline/_ref")]

ENGINE_CHECK = '''    if engine not in ("gemm", "direct"):
        raise ValueError(f"engine must be 'gemm' or 'direct', got {engine!r}")'''
ENGINE_CHECK_B200 = '''    if engine not in ("gemm", "direct", "b200"):
        raise ValueError(f"engine must be 'gemm', 'direct' or 'b200', got {engine!r}")'''
CONV_FN = '''    conv_fn = axconv2d if engine == "gemm" else direct_conv'''
CONV_FN_B200 = '''    if engine == "b200":
        from paper_2002_09481_b200 import axconv2d as conv_fn  # CUDA, no CPU fallback
    else:
        conv_fn = axconv2d if engine == "gemm" else direct_conv'''


def patched_graph():
    """axemu.graph with INTEGRATION.md's engine patch, loaded from the installed reference's source."""
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/axemu_numba_cache")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import axemu  # noqa: F401  (the package the patched module's relative imports resolve against)

    src = (REF / "axemu" / "graph.py").read_text()
    assert src.count(ENGINE_CHECK) == 1 and src.count(CONV_FN) == 1, "reference graph.py changed"
    src = src.replace(ENGINE_CHECK, ENGINE_CHECK_B200).replace(CONV_FN, CONV_FN_B200)
    mod = types.ModuleType("axemu.graph_b200")
    mod.__package__ = "axemu"
    mod.__file__ = str(REF / "axemu" / "graph_b200.py")
    sys.modules[mod.__name__] = mod  # dataclasses resolve annotations through sys.modules
    exec(compile(src, mod.__file__, "exec"), mod.__dict__)
    return mod


def test_patch_leaves_reference_engines_alone():
    g = patched_graph()
    with pytest.raises(ValueError, match="engine must be"):
        g.run(g.LayerGraph([]), None, engine="cuda")


def test_c1_stream_through_reference_graph_run():
    """The reference's 100 criterion-1 cases (seed 2026, its own generator), each as a one-conv graph
    (Input -> Min/Max -> AxConv2D, graph.py:107-141's shape) through the patched graph.run, engine b200."""
    g = patched_graph()
    from axemu import Layout, Tensor4

    gold = load_golden("c1")
    rng = np.random.default_rng(2026)
    import cases as my_cases

    for i in range(100):
        c = my_cases.random_conv_case(rng)
        from axemu import MultLut, Signedness

        nodes = [g.Node("in", g.NodeKind.INPUT, [], {}),
                 g.Node("c.in_min", g.NodeKind.MIN, ["in"], {}),
                 g.Node("c.in_max", g.NodeKind.MAX, ["in"], {}),
                 g.Node("c", g.NodeKind.AXCONV2D, ["in", "c.in_min", "c.in_max"],
                        {"filters": c["f"], "strides": c["strides"], "dilations": c["dilations"],
                         "padding": c["padding"], "f_min": c["f_range"][0], "f_max": c["f_range"][1],
                         "lut": MultLut(Signedness(c["mode"]), c["lut"])})]
        from axemu import Accumulator, RoundMode

        y = g.run(g.LayerGraph(nodes), Tensor4(c["x"], Layout.NHWC), engine="b200",
                  accumulator=Accumulator(c["accumulator"]), round_mode=RoundMode(c["round_mode"])).data
        assert bits_equal(y, gold[f"out_{i}"]), i


def test_resnet8_through_reference_graph_run():
    """A calibrated ResNet-8 (reference Node objects) through the patched graph.run: engine b200 for
    every AxConv2D, the reference's numpy for pools / Add / ReLU -- logits == the golden from engine gemm."""
    g = patched_graph()
    from axemu import Layout, MultLut, Signedness, Tensor4

    from paper_2002_09481_b200 import resnet
    from paper_2002_09481_b200 import types as T

    gold = load_golden("nets")
    nodes = []
    for n in resnet.cifar_resnet(1, T.truncated_lut(T.Signedness.SIGNED, 2), seed=0):
        a = dict(n["attrs"])
        if "lut" in a:
            a["lut"] = MultLut(Signedness(a["lut"].mode.value), a["lut"].entries)
        nodes.append(g.Node(n["id"], g.NodeKind(n["kind"]), list(n["inputs"]), a))
    trace = {}
    y = g.run(g.LayerGraph(nodes), Tensor4(gold["r8_trunc2_x"], Layout.NHWC), engine="b200", trace=trace).data
    assert bits_equal(y, gold["r8_trunc2_logits"])
    assert np.array_equal(y.reshape(y.shape[0], -1).argmax(1), gold["r8_trunc2_argmax"])
