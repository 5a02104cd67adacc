"""Generate golden vectors from the REAL reference package (run in the build container).

    python tests/golden/make_golden.py

Imports ``axemu`` from /root/reference/pkg/src (read-only; numba cache and
bytecode redirected away from the mount) and writes compressed fixtures into
tests/golden/.  The GPU box never runs this -- it only reads the .npz files.

Fixtures:
  c1.npz     100 seeded random cases (reference acceptance criterion 1,
             test_acceptance.py:51-63, seed 2026): outputs + raw emulated
             accumulators; our tests/cases.py replay is asserted identical.
  kat.npz    known-answer cases from the reference tests: extreme ranges x
             round modes x accumulators (test_axconv.py:286-310), the K=33,759
             wrap/saturate case (:250-283), zero-input/random-LUT scalar case
             (:131-152), asymmetric same padding (:331-342), config 1, the
             1000-image first layer (sha256 of the output, :225-237),
             quantizer coefficients/codes.
  nets.npz   end-to-end logits (and per-conv output sha256) of our calibrated
             ResNet-8 / ResNet-62 / ResNet-50 graphs run through the reference
             ``graph.run`` (engine "gemm") on small batches (``--nets``).
  bench.npz  the benchmarked configurations at full batch, rank 0's bench.py
             batch: ResNet-8 b1024 and ResNet-50 224x224 b256 with
             truncated_lut(signed, 2); logits + argmax + per-conv sha256, inputs
             regenerated from seeds (``--bench [r8] [r50]``, ~7 min).
  formats.npz  bytes the reference's axemu.formats writes / decodes: .axm sha256s,
             a .axt file, a 6-record CIFAR-10 file + its decoded images/labels,
             a report CSV (``--formats`` regenerates only this one).
"""

from __future__ import annotations

import hashlib
import importlib.util
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/axemu_numba_cache")
sys.dont_write_bytecode = True

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402

import axemu  # noqa: E402
from axemu import (  # noqa: E402
    Accumulator, ConvConfig, ConvGeometry, Layout, MultLut, Range, RoundMode, Signedness, Tensor4,
    axconv2d, compute_coeffs, direct_conv, exact_lut, im2cols, quantize_filters, quantize_values,
    truncated_lut,
)
from axemu.axconv import _emulate_accumulator, _lut_matmul  # noqa: E402

import cases as my_cases  # noqa: E402  (tests/cases.py -- the replay)


def _load_ref_cases():
    spec = importlib.util.spec_from_file_location("ref_cases", REF / "tests" / "cases.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


ref_cases = _load_ref_cases()


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_acc(case) -> np.ndarray:
    """Raw emulated accumulators exactly as approx_gemm computes them (axconv.py:236-243)."""
    x, f, cfg, lut = case["inputs"], case["filters"], case["cfg"], case["lut"]
    p1 = compute_coeffs(case["in_range"], lut.mode, cfg.round_mode)
    p2 = compute_coeffs(case["f_range"], lut.mode, cfg.round_mode)
    kh, kw, cin, cout = f.shape
    pm = im2cols(x, p1, cfg.geometry, (kh, kw))
    qf = quantize_filters(f, p2)
    acc = np.empty((pm.rows, cout), np.int64)
    _lut_matmul(pm.codes.view(np.uint8), np.ascontiguousarray(qf.codes.T).view(np.uint8), lut.entries, acc)
    acc = _emulate_accumulator(acc, cfg.accumulator)
    n = x.shape[0]
    return acc.reshape(n, -1, cout)


def make_c1() -> dict:
    rng_ref = np.random.default_rng(2026)
    rng_me = np.random.default_rng(2026)
    out = {}
    for i in range(100):
        rc = ref_cases.random_conv_case(rng_ref)
        mc = my_cases.random_conv_case(rng_me)
        # replay check: identical inputs
        assert np.array_equal(rc["inputs"].data, mc["x"]), i
        assert np.array_equal(rc["filters"].data, mc["f"]), i
        assert np.array_equal(rc["lut"].entries, mc["lut"]), i
        assert rc["lut"].mode.value == mc["mode"]
        g = rc["cfg"].geometry
        assert tuple(g.strides) == mc["strides"] and tuple(g.dilations) == mc["dilations"]
        assert (g.padding if isinstance(g.padding, str) else tuple(g.padding)) == mc["padding"]
        assert rc["cfg"].accumulator.value == mc["accumulator"] and rc["cfg"].round_mode.value == mc["round_mode"]
        y = axconv2d(rc["inputs"], rc["filters"], rc["in_range"], rc["f_range"], rc["lut"], rc["cfg"]).data
        d = direct_conv(rc["inputs"], rc["filters"], rc["in_range"], rc["f_range"], rc["lut"], rc["cfg"]).data
        assert np.array_equal(y.view(np.uint32), d.view(np.uint32)), i
        out[f"out_{i}"] = y
        out[f"acc_{i}"] = ref_acc(rc).reshape(y.shape)
    return out


def make_kat() -> dict:
    out = {}
    # extreme ranges (test_axconv.py:286-310)
    extremes = [
        ((-1e6, 1e6), (-1e3, 1e3), Signedness.SIGNED),
        ((0.0, 1e-9), (-1e-12, 1e-12), Signedness.SIGNED),
        ((-1e-3, 1e5), (-7.0, 0.0), Signedness.UNSIGNED),
        ((-9.0, -1.0), (-5.0, -0.1), Signedness.UNSIGNED),
        ((0.0, 0.0), (3.0, 3.0), Signedness.SIGNED),
    ]
    for e, (ir, fr, mode) in enumerate(extremes):
        rng = np.random.default_rng(0)
        x = rng.uniform(ir[0], ir[1], (2, 6, 6, 2)).astype(np.float32)
        x[0, 0, 0, 0], x[0, 0, 0, 1] = ir[0], ir[1]
        f = rng.uniform(fr[0], fr[1], (3, 3, 2, 3)).astype(np.float32)
        f[0, 0, 0, 0], f[0, 0, 1, 0] = fr[0], fr[1]
        out[f"ext{e}_x"], out[f"ext{e}_f"] = x, f
        for rm in RoundMode:
            for acc in Accumulator:
                cfg = ConvConfig(geometry=ConvGeometry(padding="same"), round_mode=rm, accumulator=acc)
                y = axconv2d(Tensor4(x), Tensor4(f, Layout.HWCN), Range(*ir), Range(*fr), exact_lut(mode), cfg)
                out[f"ext{e}_{rm.value}_{acc.value}"] = y.data
    # overflow case K = 33*33*31 (test_axconv.py:250-283)
    k, cin = 33, 31
    x = Tensor4(np.ones((1, k, k, cin), np.float32))
    f = Tensor4(np.ones((k, k, cin, 1), np.float32), Layout.HWCN)
    lut = MultLut(Signedness.UNSIGNED, np.full(65536, 65535, np.uint16))
    for acc in Accumulator:
        y = axconv2d(x, f, Range(0.0, 1.0), Range(0.0, 1.0), lut, ConvConfig(accumulator=acc))
        out[f"ovf_{acc.value}"] = y.data
    # zero input x random LUT (test_axconv.py:131-152)
    rng = np.random.default_rng(1)
    entries = rng.integers(-(1 << 15), 1 << 15, 65536).astype(np.int16)
    fvals = np.array([0.4, -0.2, 0.7, -0.9], np.float32).reshape(2, 2, 1, 1)
    y = direct_conv(Tensor4(np.zeros((1, 2, 2, 1), np.float32)), Tensor4(fvals, Layout.HWCN), Range(0.0, 0.0),
                    Range(-0.9, 0.7), MultLut(Signedness.SIGNED, entries), ConvConfig())
    out["zero_in_entries"], out["zero_in_out"] = entries, y.data
    # asymmetric same padding (test_axconv.py:331-342)
    rng = np.random.default_rng(5)
    xa = rng.uniform(0, 1, (1, 3, 3, 1)).astype(np.float32)
    fa = rng.normal(0, 1, (2, 2, 1, 1)).astype(np.float32)
    y = axconv2d(Tensor4(xa), Tensor4(fa, Layout.HWCN), Range(0, 1), Range(-2, 2), exact_lut(Signedness.UNSIGNED),
                 ConvConfig(geometry=ConvGeometry(padding="same")))
    out["asym_x"], out["asym_f"], out["asym_out"] = xa, fa, y.data
    # config 1: 1x32x32x3, 3x3x3->16, same; exact signed + one random LUT
    rng = np.random.default_rng(11)
    x1 = rng.uniform(0, 1, (1, 32, 32, 3)).astype(np.float32)
    f1 = rng.normal(0, 0.4, (3, 3, 3, 16)).astype(np.float32)
    rl = MultLut(Signedness.SIGNED, rng.integers(-(1 << 15), 1 << 15, 65536).astype(np.int16))
    out["cfg1_x"], out["cfg1_f"], out["cfg1_rlut"] = x1, f1, rl.entries
    for tag, lt in (("exact", exact_lut(Signedness.SIGNED)), ("random", rl)):
        cfg = ConvConfig(geometry=ConvGeometry(padding="same"))
        ir, fr = Range(float(x1.min()), float(x1.max())), Range(float(f1.min()), float(f1.max()))
        out[f"cfg1_{tag}"] = axconv2d(Tensor4(x1), Tensor4(f1, Layout.HWCN), ir, fr, lt, cfg).data
        out[f"cfg1_{tag}_direct"] = direct_conv(Tensor4(x1), Tensor4(f1, Layout.HWCN), ir, fr, lt, cfg).data
    # 1000-image first layer (test_axconv.py:225-237): sha256 of the full output
    rng = np.random.default_rng(8)
    xs = rng.uniform(0, 1, (1000, 32, 32, 3)).astype(np.float32)
    fs = rng.normal(0, 0.4, (3, 3, 3, 16)).astype(np.float32)
    ys = axconv2d(Tensor4(xs), Tensor4(fs, Layout.HWCN), Range(0.0, 1.0), Range(-2.0, 2.0),
                  exact_lut(Signedness.SIGNED), ConvConfig(geometry=ConvGeometry(padding="same"))).data
    out["scale_sha"] = np.frombuffer(bytes.fromhex(sha(ys)), np.uint8)
    out["scale_head"] = ys[:2]
    # quantizer: coefficients and codes over tricky values
    ranges = [(0.0, 2.55), (0.0, 0.0), (-1.0, 1.0), (2.0, 4.0), (-9.0, -1.0), (-2.3, 5.9), (0.0, 5e-324),
              (-1e6, 1e6), (-1e-3, 1e5), (-3.0, 3.0), (0.1, 0.7)]
    rng = np.random.default_rng(77)
    qi = 0
    for mode in Signedness:
        for rm in RoundMode:
            for r in ranges:
                p = compute_coeffs(Range(*r), mode, rm)
                lo, hi = r
                vals = np.concatenate([
                    rng.uniform(lo - 0.1 * abs(hi - lo) - 1e-3, hi + 0.1 * abs(hi - lo) + 1e-3, 400),
                    (np.arange(-140, 140) + 0.5) * p.scale,          # exact half steps
                    (np.arange(-140, 140) + 0.5 + 2e-6) * p.scale,   # near-half (snap region)
                    np.arange(-140, 140) * p.scale * (1 + 1e-9),     # near grid points
                ]).astype(np.float32)
                out[f"q{qi}_range"] = np.array(r, np.float64)
                out[f"q{qi}_mode"] = np.array([mode is Signedness.SIGNED, list(RoundMode).index(rm)], np.int32)
                out[f"q{qi}_coeffs"] = np.array([p.scale, p.zero_point], np.float64)
                out[f"q{qi}_vals"] = vals
                out[f"q{qi}_codes"] = quantize_values(vals, p)
                qi += 1
    out["q_count"] = np.array(qi)
    return out


def to_reference_graph(nodes):
    from axemu import LayerGraph, Node, NodeKind

    ref_nodes = []
    for n in nodes:
        attrs = dict(n["attrs"])
        if "lut" in attrs:
            lt = attrs["lut"]
            attrs["lut"] = MultLut(Signedness(lt.mode.value), lt.entries)
        ref_nodes.append(Node(n["id"], NodeKind(n["kind"]), list(n["inputs"]), attrs))
    return LayerGraph(ref_nodes)


def make_nets() -> dict:
    from paper_2002_09481_b200 import resnet
    from paper_2002_09481_b200 import types as T

    out = {}
    rl = T.random_lut(np.random.default_rng(123), T.Signedness.SIGNED)
    runs = [
        ("r8_trunc2", resnet.cifar_resnet(1, T.truncated_lut(T.Signedness.SIGNED, 2), seed=0), "cifar", 16),
        ("r8_random", resnet.cifar_resnet(1, rl, seed=0), "cifar", 16),
        ("r8_unsigned", resnet.cifar_resnet(1, T.truncated_lut(T.Signedness.UNSIGNED, 1), seed=3), "cifar", 8),
        ("r62_trunc3", resnet.cifar_resnet(10, T.truncated_lut(T.Signedness.SIGNED, 3), seed=1), "cifar", 32),
        ("r50_exact", resnet.resnet50(T.exact_lut(T.Signedness.SIGNED), seed=0), "imagenet", 4),
    ]
    out["random_lut_seed123"] = rl.entries
    for tag, nodes, kind, n in runs:
        if kind == "cifar":
            from axemu import synthetic_cifar10

            x, labels = synthetic_cifar10(n, seed=5)
        else:
            from paper_2002_09481_b200.datasets import synthetic_imagenet

            x, _ = synthetic_imagenet(n, seed=2)
        out[f"{tag}_x"] = x
        run_reference(tag, nodes, x, out)
    return out


class _DepthwiseDispatch:
    """The reference has no grouped conv (tensor.py:66-87).  For graphs with depthwise AxConv2D nodes
    (config 5) ``graph.run``'s conv (graph.py:226, :259-267) is wrapped: a node whose filters array is
    registered here runs as per-channel reference ``axconv2d`` calls with the node's shared ranges
    (SURVEY.md 8(d) config 5); every other conv runs the reference's ``axconv2d`` unchanged."""

    def __init__(self, nodes):
        import axemu.graph as G

        self.G, self.orig = G, G.axconv2d
        self.dw = {id(n["attrs"]["filters"]) for n in nodes if n["attrs"].get("depthwise")}

    def __call__(self, inputs, filters, in_range, f_range, lut, cfg, meter=None):
        if id(filters.data) not in self.dw:
            return self.orig(inputs, filters, in_range, f_range, lut, cfg, meter)
        x, f = inputs.data, filters.data
        parts = [self.orig(Tensor4(x[..., c:c + 1], Layout.NHWC), Tensor4(f[:, :, c:c + 1, :], Layout.HWCN),
                           in_range, f_range, lut, cfg, meter).data for c in range(x.shape[3])]
        return Tensor4(np.concatenate(parts, axis=3), Layout.NHWC)

    def __enter__(self):
        self.G.axconv2d = self
        return self

    def __exit__(self, *exc):
        self.G.axconv2d = self.orig


def run_reference(tag, nodes, x, out):
    """Logits, argmax and per-conv output sha256 of ``nodes`` on ``x`` through the reference graph.run."""
    for n in nodes:  # the filters object graph.run hands to the conv must stay the node's own array
        if "filters" in n["attrs"]:
            n["attrs"]["filters"] = np.ascontiguousarray(n["attrs"]["filters"], np.float32)
    g = to_reference_graph(nodes)
    trace = {}
    with _DepthwiseDispatch(nodes):
        y = axemu.run(g, Tensor4(x, Layout.NHWC), "gemm", trace=trace).data
    n = x.shape[0]
    out[f"{tag}_logits"] = y
    out[f"{tag}_argmax"] = y.reshape(n, -1).argmax(1)
    out[f"{tag}_logits_sha"] = np.frombuffer(bytes.fromhex(sha(y)), np.uint8)
    conv_ids = [nd["id"] for nd in nodes if nd["kind"] == "AxConv2D"]
    out[f"{tag}_conv_ids"] = np.array(conv_ids)
    out[f"{tag}_conv_sha"] = np.stack(
        [np.frombuffer(bytes.fromhex(sha(np.asarray(trace[c], np.float32))), np.uint8) for c in conv_ids])
    am = out[f"{tag}_argmax"]
    print(tag, "argmax", am[:16], "distinct", len(set(am.tolist())), flush=True)


BENCH_SEED = 1000  # bench.py: rank r's batch is seeded 1000 + r


def make_bench() -> dict:
    """The benchmarked configurations at their full batch (BASELINE configs 2 and 3), rank 0's batch of
    bench.py: ResNet-8 b1024 (synthetic_cifar10(1024, 1000)) and ResNet-50 224 b256
    (synthetic_imagenet(256, 1000)), both with truncated_lut(signed, 2).  Inputs are NOT stored (the
    GPU test and bench.py regenerate them from the seed); logits, argmax and per-conv sha256 are."""
    from paper_2002_09481_b200 import datasets, resnet
    from paper_2002_09481_b200 import types as T

    lut = T.truncated_lut(T.Signedness.SIGNED, 2)
    out = {}
    which = ([a for a in sys.argv[1:] if a in ("r8", "r50", "mbv1", "r62sweep", "r50exact")]
             or ["r8", "r50", "mbv1", "r62sweep", "r50exact"])
    path = HERE / "bench.npz"
    if path.exists():
        out.update(dict(np.load(path)))
    if "r8" in which:
        x, _ = datasets.synthetic_cifar10(1024, seed=BENCH_SEED)
        run_reference("r8", resnet.cifar_resnet(1, lut, seed=0), x, out)
    if "r50" in which:
        x, _ = datasets.synthetic_imagenet(256, seed=BENCH_SEED)
        run_reference("r50", resnet.resnet50(lut, seed=0), x, out)
    if "r50exact" in which:
        # config 5 control: the same ResNet-50 b256 with exact_lut(signed) (bench.py --lut exact); logits
        # sha256 + argmax only
        x, _ = datasets.synthetic_imagenet(256, seed=BENCH_SEED)
        nodes = resnet.resnet50(T.exact_lut(T.Signedness.SIGNED), seed=0)
        for n in nodes:
            if "filters" in n["attrs"]:
                n["attrs"]["filters"] = np.ascontiguousarray(n["attrs"]["filters"], np.float32)
        y = axemu.run(to_reference_graph(nodes), Tensor4(x, Layout.NHWC), "gemm").data
        out["r50exact_logits_sha"] = np.frombuffer(bytes.fromhex(sha(y)), np.uint8)
        out["r50exact_argmax"] = y.reshape(256, -1).argmax(1)
        print("r50exact argmax distinct", len(set(out["r50exact_argmax"].tolist())), flush=True)
    if "mbv1" in which:
        x, _ = datasets.synthetic_imagenet(256, seed=BENCH_SEED)
        run_reference("mbv1", resnet.mobilenet_v1(lut, seed=0), x, out)
    if "r62sweep" in which:
        # config 4: the sweep's first candidate network (bench.py sweep_luts()[0], truncated_lut(signed, 0))
        # on the sweep batch synthetic_cifar10(1000, 1000); logits only (63 traced convs at 1000 images
        # would be 4 GB)
        sys.path.insert(0, str(HERE.parent.parent))
        import bench

        x, _ = datasets.synthetic_cifar10(1000, seed=BENCH_SEED)
        nodes = resnet.cifar_resnet(10, bench.sweep_luts()[0], seed=0)
        for n in nodes:
            if "filters" in n["attrs"]:
                n["attrs"]["filters"] = np.ascontiguousarray(n["attrs"]["filters"], np.float32)
        y = axemu.run(to_reference_graph(nodes), Tensor4(x, Layout.NHWC), "gemm").data
        out["r62sweep_logits_sha"] = np.frombuffer(bytes.fromhex(sha(y)), np.uint8)
        out["r62sweep_argmax"] = y.reshape(1000, -1).argmax(1)
        print("r62sweep argmax distinct", len(set(out["r62sweep_argmax"].tolist())), flush=True)
    return out


def make_formats() -> dict:
    """Bytes written / decoded by the reference's axemu.formats (formats.py:58-255)."""
    import tempfile

    from axemu import (load_cifar10, make_report, report_csv, save_cifar10, save_lut, save_tensor,
                       synthetic_cifar10)

    out = {}
    with tempfile.TemporaryDirectory() as td:
        td = Path(td)
        for tag, lut in (("exact_unsigned", exact_lut(Signedness.UNSIGNED)),
                         ("trunc3_signed", truncated_lut(Signedness.SIGNED, 3))):
            save_lut(lut, td / f"{tag}.axm")
            out[f"lut_{tag}_sha"] = np.frombuffer(bytes.fromhex(hashlib.sha256(
                (td / f"{tag}.axm").read_bytes()).hexdigest()), np.uint8)
        t = Tensor4(np.array([0.0, 0.5, -1.25, 3.0], np.float32).reshape(1, 2, 2, 1))
        save_tensor(t, td / "unit.axt")
        out["tensor_unit_bytes"] = np.frombuffer((td / "unit.axt").read_bytes(), np.uint8)
        images, labels = synthetic_cifar10(6, seed=3)
        save_cifar10(td / "b.bin", images, labels)
        out["cifar_records"] = np.frombuffer((td / "b.bin").read_bytes(), np.uint8)
        batch = load_cifar10(td / "b.bin")
        out["cifar_images"] = batch.images.data
        out["cifar_labels"] = batch.labels
        rep = make_report(0.25, 1.5, 0.75, 0.5, 123456, {"conv1": 0.4, "conv2": 0.35})
        out["report_csv"] = np.frombuffer(report_csv(rep).encode(), np.uint8)
        # a small float model -> transform -> save_model (graph.py:107-141, formats.py:298-339), and its
        # logits through the reference executor
        from axemu import LayerGraph, Node, NodeKind, run, save_model, transform

        g = LayerGraph(model_graph_reference(Node, NodeKind))
        tg, rep = transform(g, truncated_lut(Signedness.SIGNED, 2))
        out["model_transform_report"] = np.array([rep.replaced_count, rep.inserted_min_max])
        save_model(tg, td / "ax.json")
        out["model_json"] = np.frombuffer((td / "ax.json").read_bytes(), np.uint8)
        out["model_weights"] = np.frombuffer((td / "ax.weights.bin").read_bytes(), np.uint8)
        out["model_axm_sha"] = np.frombuffer(bytes.fromhex(hashlib.sha256((td / "ax.axm").read_bytes()).hexdigest()),
                                             np.uint8)
        x = np.random.default_rng(17).uniform(0, 1, (4, 12, 12, 3)).astype(np.float32)
        out["model_input"] = x
        out["model_logits"] = run(tg, Tensor4(x), engine="gemm").data
    return out


def model_graph_reference(Node, NodeKind):
    kinds = {k.value: k for k in NodeKind}
    return [Node(i, kinds[k], list(ins), dict(a)) for i, k, ins, a in my_cases.model_graph_spec()]


def main():
    if "--bench" in sys.argv:
        np.savez_compressed(HERE / "bench.npz", **make_bench())
        print("bench ok", flush=True)
        return
    if "--nets" in sys.argv:
        np.savez_compressed(HERE / "nets.npz", **make_nets())
        print("nets ok", flush=True)
        return
    if "--formats" in sys.argv:
        np.savez_compressed(HERE / "formats.npz", **make_formats())
        print("formats ok", flush=True)
        return
    c1 = make_c1()
    np.savez_compressed(HERE / "c1.npz", **c1)
    print("c1 ok", flush=True)
    kat = make_kat()
    np.savez_compressed(HERE / "kat.npz", **kat)
    print("kat ok", flush=True)
    nets = make_nets()
    np.savez_compressed(HERE / "nets.npz", **nets)
    print("nets ok", flush=True)
    np.savez_compressed(HERE / "formats.npz", **make_formats())
    print("formats ok", flush=True)


if __name__ == "__main__":
    main()
