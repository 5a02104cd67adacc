"""Pin the CPU oracle (oracle/axemu_oracle.py) to the real reference's golden vectors."""

import hashlib

import numpy as np
import pytest

from cases import oracle_conv, random_conv_case
from golden_io import bits_equal, load_golden
from oracle import axemu_oracle as O


def test_c1_cases_bit_identical_to_reference():
    g = load_golden("c1")
    rng = np.random.default_rng(2026)
    for i in range(100):
        case = random_conv_case(rng)
        y, acc = oracle_conv(case, return_acc=True)
        assert bits_equal(y, g[f"out_{i}"]), i
        assert np.array_equal(acc, g[f"acc_{i}"]), i
        if i % 10 == 0:  # the nested-loop restatement agrees too
            assert bits_equal(oracle_conv(case, engine="direct"), g[f"out_{i}"]), i


def test_extreme_ranges_and_accumulators():
    g = load_golden("kat")
    extremes = [((-1e6, 1e6), (-1e3, 1e3), O.SIGNED), ((0.0, 1e-9), (-1e-12, 1e-12), O.SIGNED),
                ((-1e-3, 1e5), (-7.0, 0.0), O.UNSIGNED), ((-9.0, -1.0), (-5.0, -0.1), O.UNSIGNED),
                ((0.0, 0.0), (3.0, 3.0), O.SIGNED)]
    for e, (ir, fr, mode) in enumerate(extremes):
        for rm in (O.HALF_AWAY, O.HALF_EVEN, O.TOWARD_ZERO):
            for acc in (O.EXACT64, O.WRAP32, O.SATURATE32):
                y = O.axconv2d(g[f"ext{e}_x"], g[f"ext{e}_f"], ir, fr, O.exact_lut(mode), mode, padding="same",
                               accumulator=acc, round_mode=rm)
                assert bits_equal(y, g[f"ext{e}_{rm}_{acc}"]), (e, rm, acc)


def test_overflow_kat_wrap_and_saturate():
    g = load_golden("kat")
    x = np.ones((1, 33, 33, 31), np.float32)
    f = np.ones((33, 33, 31, 1), np.float32)
    lut = np.full(65536, 65535, np.uint16)
    for acc in (O.EXACT64, O.WRAP32, O.SATURATE32):
        y = O.axconv2d(x, f, (0.0, 1.0), (0.0, 1.0), lut, O.UNSIGNED, accumulator=acc)
        assert bits_equal(y, g[f"ovf_{acc}"]), acc
    depth = 33 * 33 * 31
    total = depth * 65535
    s = O.compute_coeffs(0.0, 1.0, O.UNSIGNED)[0]
    assert g["ovf_wrap32"][0, 0, 0, 0] == np.float32(s * s * (((total + 2**31) % 2**32) - 2**31))
    assert g["ovf_saturate32"][0, 0, 0, 0] == np.float32(s * s * (2**31 - 1))


def test_small_kats():
    g = load_golden("kat")
    y = O.direct_conv(np.zeros((1, 2, 2, 1), np.float32), np.array([0.4, -0.2, 0.7, -0.9], np.float32).reshape(2, 2, 1, 1),
                      (0.0, 0.0), (-0.9, 0.7), g["zero_in_entries"], O.SIGNED)
    assert bits_equal(y, g["zero_in_out"])
    y = O.axconv2d(g["asym_x"], g["asym_f"], (0, 1), (-2, 2), O.exact_lut(O.UNSIGNED), O.UNSIGNED, padding="same")
    assert bits_equal(y, g["asym_out"])
    x1, f1 = g["cfg1_x"], g["cfg1_f"]
    for tag, lut in (("exact", O.exact_lut(O.SIGNED)), ("random", g["cfg1_rlut"])):
        y = O.axconv2d(x1, f1, (float(x1.min()), float(x1.max())), (float(f1.min()), float(f1.max())), lut,
                       O.SIGNED, padding="same")
        assert bits_equal(y, g[f"cfg1_{tag}"])
        assert bits_equal(g[f"cfg1_{tag}_direct"], g[f"cfg1_{tag}"])


def test_hand_worked_two_tap_case():
    """test_axconv.py:77-95: A = 110, S_p = 30, S_f = 7, zp 5 / 1 -> 0.01 * 55."""
    lut = O.exact_lut(O.UNSIGNED)
    out = O.approx_gemm(np.array([[10, 20]], np.uint8), np.array([30], np.int32), np.array([[3], [4]], np.uint8),
                        np.array([7], np.int32), 0.1, 5, 0.1, 1, lut)
    assert out[0, 0] == pytest.approx(0.55, rel=1e-6)


def test_quantizer_codes_match_reference():
    g = load_golden("kat")
    rounds = [O.HALF_AWAY, O.HALF_EVEN, O.TOWARD_ZERO]
    for i in range(int(g["q_count"])):
        mn, mx = g[f"q{i}_range"]
        sgn, rm = g[f"q{i}_mode"]
        mode = O.SIGNED if sgn else O.UNSIGNED
        s, zp = O.compute_coeffs(float(mn), float(mx), mode, rounds[rm])
        assert (s, zp) == (g[f"q{i}_coeffs"][0], int(g[f"q{i}_coeffs"][1])), i
        assert np.array_equal(O.quantize_values(g[f"q{i}_vals"], s, zp, mode, rounds[rm]), g[f"q{i}_codes"]), i


def test_at_scale_first_layer_sha():
    g = load_golden("kat")
    rng = np.random.default_rng(8)
    xs = rng.uniform(0, 1, (1000, 32, 32, 3)).astype(np.float32)
    fs = rng.normal(0, 0.4, (3, 3, 3, 16)).astype(np.float32)
    ys = O.axconv2d(xs, fs, (0.0, 1.0), (-2.0, 2.0), O.exact_lut(O.SIGNED), O.SIGNED, padding="same")
    assert hashlib.sha256(ys.tobytes()).digest() == g["scale_sha"].tobytes()


@pytest.mark.parametrize("tag,depth,seed,kind", [("r8_trunc2", 1, 0, ("t", 2)), ("r8_random", 1, 0, ("r",)),
                                                 ("r8_unsigned", 1, 3, ("tu", 1)), ("r62_trunc3", 10, 1, ("t", 3))])
def test_resnet_graphs_match_reference(tag, depth, seed, kind):
    from paper_2002_09481_b200 import resnet
    from paper_2002_09481_b200 import types as T

    g = load_golden("nets")
    if kind[0] == "t":
        lut = T.truncated_lut(T.Signedness.SIGNED, kind[1])
    elif kind[0] == "tu":
        lut = T.truncated_lut(T.Signedness.UNSIGNED, kind[1])
    else:
        lut = T.MultLut(T.Signedness.SIGNED, g["random_lut_seed123"])
    nodes = oracle_nodes(resnet.cifar_resnet(depth, lut, seed=seed))
    y = O.run_graph(nodes, g[f"{tag}_x"])
    assert bits_equal(y, g[f"{tag}_logits"])


def oracle_nodes(nodes):
    out = []
    for n in nodes:
        a = dict(n["attrs"])
        if "lut" in a:
            a["mode"] = a["lut"].mode.value
            a["lut"] = a["lut"].entries
        out.append({"id": n["id"], "kind": n["kind"], "inputs": n["inputs"], "attrs": a})
    return out


def test_mac_counts():
    from paper_2002_09481_b200 import resnet
    from paper_2002_09481_b200 import types as T

    lut = T.exact_lut(T.Signedness.SIGNED)
    assert resnet.macs_per_image(resnet.cifar_resnet(1, lut)) == 12_500_992 + 640
    assert resnet.macs_per_image(resnet.cifar_resnet(10, lut)) == 139_902_976 + 640
    assert resnet.macs_per_image(resnet.resnet50(lut)) == 4_087_136_256 + 2_048_000
    nodes = oracle_nodes(resnet.cifar_resnet(1, lut))
    assert O.graph_mac_count(nodes, (3, 32, 32, 3)) == 3 * (12_500_992 + 640)


@pytest.mark.parametrize("tag,classes", [("r8_trunc2", 5), ("r8_random", 5), ("r8_unsigned", 3), ("r62_trunc3", 3),
                                         ("r50_exact", 3)])
def test_golden_networks_are_not_degenerate(tag, classes):
    """Calibrated networks (resnet.apply_calibration) predict different classes for different images, so
    argmax parity means something: >= 5 distinct classes among 16 images; >= 3 for the 8-image and
    4-image nets and for the 63-conv ResNet-62 under the 3-bit-truncating table (its calibration batch
    has 1000 images; ranges are per batch, so 32 images shift every layer's quantization)."""
    g = load_golden("nets")
    am = g[f"{tag}_argmax"]
    assert len(set(am.tolist())) >= classes, (tag, am)
    rows = g[f"{tag}_logits"].reshape(len(am), -1)
    assert len({r.tobytes() for r in rows}) == len(rows)  # no two images share a logits row


def test_bench_goldens_are_not_degenerate():
    """The benchmarked batches (ResNet-8 b1024, ResNet-50 b256, MobileNet-v1-shaped b256): several classes
    predicted (the 27-conv MobileNet with 9-tap depthwise layers is the least diverse)."""
    g = load_golden("bench")
    assert len(set(g["r8_argmax"].tolist())) >= 8
    assert len(set(g["r50_argmax"].tolist())) >= 20
    assert len(set(g["mbv1_argmax"].tolist())) >= 4
    assert len(g["r8_conv_ids"]) == 10 and len(g["r50_conv_ids"]) == 54 and len(g["mbv1_conv_ids"]) == 28


def test_depthwise_oracle_is_per_channel_axconv2d():
    """Config 5's depthwise conv in the oracle graph: a node with depthwise=True and (kh, kw, C, 1) filters
    equals the per-channel reference decomposition (axconv2d per channel, shared ranges); both engines."""
    rng = np.random.default_rng(55)
    x = np.maximum(rng.standard_normal((2, 9, 11, 5)), 0).astype(np.float32)
    f = (rng.standard_normal((3, 3, 5, 1)) * 0.4).astype(np.float32)
    lut = O.random_lut(rng, O.SIGNED)
    nodes = [{"id": "in", "kind": "Input", "inputs": [], "attrs": {}},
             {"id": "d.in_min", "kind": "Min", "inputs": ["in"], "attrs": {}},
             {"id": "d.in_max", "kind": "Max", "inputs": ["in"], "attrs": {}},
             {"id": "d", "kind": "AxConv2D", "inputs": ["in", "d.in_min", "d.in_max"],
              "attrs": dict(filters=f, lut=lut, mode=O.SIGNED, f_min=float(f.min()), f_max=float(f.max()),
                            strides=(2, 1), dilations=(1, 1), padding="same", depthwise=True)}]
    ir, fr = (float(x.min()), float(x.max())), (float(f.min()), float(f.max()))
    want = np.concatenate([O.axconv2d(x[..., c:c + 1], f[:, :, c:c + 1, :], ir, fr, lut, O.SIGNED, padding="same",
                                      strides=(2, 1)) for c in range(5)], axis=3)
    for engine in ("gemm", "direct"):
        assert bits_equal(O.run_graph(nodes, x, engine=engine), want)
    assert O.graph_mac_count(nodes, x.shape) == 2 * 5 * 11 * 9 * 5
    with pytest.raises(ValueError, match="depthwise filters"):
        O.depthwise_conv(x, np.zeros((3, 3, 5, 2), np.float32), ir, fr, lut, O.SIGNED)


def test_mobilenet_shapes_and_macs():
    """The MobileNet-v1-shaped net (config 5 in context): 13 depthwise + 14 dense convs, 568.7 M MACs per
    image (the architecture's published 569 M mult-adds), depthwise layers at (112,112,32) and (56,56,128)
    at stride 1 and 2, calibrated per output channel."""
    from paper_2002_09481_b200 import resnet
    from paper_2002_09481_b200 import types as T

    nodes = resnet.mobilenet_v1(T.truncated_lut(T.Signedness.SIGNED, 2))
    convs = [n for n in nodes if n["kind"] == "AxConv2D"]
    dws = [n for n in convs if n["attrs"].get("depthwise")]
    assert len(convs) == 28 and len(dws) == 13
    assert resnet.macs_per_image(nodes) == 568_740_352
    assert O.graph_mac_count(oracle_nodes(nodes), (1, 224, 224, 3)) == 568_740_352
    shapes = [(n["attrs"]["filters"].shape, n["attrs"]["strides"]) for n in dws[:4]]
    assert shapes == [((3, 3, 32, 1), (1, 1)), ((3, 3, 64, 1), (2, 2)), ((3, 3, 128, 1), (1, 1)),
                      ((3, 3, 128, 1), (2, 2))]
