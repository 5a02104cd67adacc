"""ResNet graph builders for the benchmark / parity workloads.

Graphs use the reference's node vocabulary (``axemu.graph.NodeKind`` names:
Input, Min, Max, AxConv2D, ReLU, Add, MaxPool, AvgPool; graph.py:25-37) in
the *transformed* form that ``axemu.graph.transform`` (graph.py:107-141)
produces: every convolution is an ``AxConv2D`` fed by ``<id>.in_min`` /
``<id>.in_max`` range nodes over its data input, with the filter range folded
to constants ``f_min`` / ``f_max``.  BatchNorm is folded (the reference has no
BN node), so every conv carries a bias.  The classifier is a 1x1 AxConv2D on
the globally pooled (n,1,1,C) tensor, so *all* conv/dense layers are
approximate and logits are integer-exact (Dense would go through float BLAS,
graph.py:295, which is not reproducible).

Nodes are plain dicts ``{"id", "kind", "inputs", "attrs"}``; ``to_reference``
in the tests converts them to ``axemu.graph.Node`` for the real reference.

Weights are synthetic: He-normal filters and N(0, 0.05) biases from a seed,
then **calibrated** (``apply_calibration``).  A BatchNorm is folded into every
conv: one power-of-two filter scale per layer and one bias per output channel.
They were measured on the approximate network itself by the real reference
(``scripts/make_calibration.py``, a fixed calibration batch) and committed in
``calib.npz``, keyed by architecture, seed and multiplier: a network uses the
calibration for its own table when one exists, else the one for
truncated_lut(signed, 2), the benchmark multiplier.  Each conv's output then has roughly
unit variance and per-channel zero mean, and so do the classifier's logits.
Without this, the un-normalised He-normal nets predict one class for every
image (every golden net did in round 1).
"""

from __future__ import annotations

import numpy as np


class _Builder:
    def __init__(self, seed: int, lut):
        self.rng = np.random.default_rng(seed)
        self.lut = lut
        self.nodes: list[dict] = []

    def add(self, nid, kind, inputs=(), **attrs):
        self.nodes.append({"id": nid, "kind": kind, "inputs": list(inputs), "attrs": attrs})
        return nid

    def conv(self, nid, x, cin, cout, k, stride=1, relu=False, bias=True):
        std = float(np.sqrt(2.0 / (k * k * cin)))
        f = (self.rng.standard_normal((k, k, cin, cout)) * std).astype(np.float32)
        b = (self.rng.standard_normal(cout) * 0.05).astype(np.float32) if bias else None
        self.add(f"{nid}.in_min", "Min", [x])
        self.add(f"{nid}.in_max", "Max", [x])
        attrs = dict(filters=f, strides=(stride, stride), dilations=(1, 1), padding="same",
                     lut=self.lut, f_min=float(f.min()), f_max=float(f.max()))
        if b is not None:
            attrs["bias"] = b
        self.add(nid, "AxConv2D", [x, f"{nid}.in_min", f"{nid}.in_max"], **attrs)
        if relu:
            return self.add(f"{nid}.relu", "ReLU", [nid])
        return nid

    def dwconv(self, nid, x, c, k, stride=1, relu=True):
        """Depthwise k x k conv (channel multiplier 1): filters (k, k, c, 1), ``depthwise=True``."""
        std = float(np.sqrt(2.0 / (k * k)))
        f = (self.rng.standard_normal((k, k, c, 1)) * std).astype(np.float32)
        b = (self.rng.standard_normal(c) * 0.05).astype(np.float32)
        self.add(f"{nid}.in_min", "Min", [x])
        self.add(f"{nid}.in_max", "Max", [x])
        self.add(nid, "AxConv2D", [x, f"{nid}.in_min", f"{nid}.in_max"], filters=f, strides=(stride, stride),
                 dilations=(1, 1), padding="same", lut=self.lut, f_min=float(f.min()), f_max=float(f.max()),
                 bias=b, depthwise=True)
        return self.add(f"{nid}.relu", "ReLU", [nid]) if relu else nid


# ---------------------------------------------------------------------------- calibration

_CALIB_SEED = 424242
_CALIB_FILE = __import__("pathlib").Path(__file__).with_name("calib.npz")
_CALIB = None


def lut_tag(lut) -> str:
    """Short content tag of a truth table (signedness + sha256 prefix of the entries)."""
    import hashlib

    m = getattr(lut.mode, "value", lut.mode)
    return f"{m[0]}{hashlib.sha256(np.ascontiguousarray(lut.entries).tobytes()).hexdigest()[:10]}"


def _calib():
    global _CALIB
    if _CALIB is None:
        _CALIB = dict(np.load(_CALIB_FILE)) if _CALIB_FILE.exists() else {}
    return _CALIB


def calibration_key(arch_seed: str, lut) -> str:
    """The committed calibration for this network and multiplier, else the one for the benchmark
    multiplier truncated_lut(signed, 2): a network calibrated once and evaluated with other candidate
    multipliers (the sweep of config 4)."""
    from .types import Signedness, truncated_lut

    cal = _calib()
    own = f"{arch_seed}_{lut_tag(lut)}"
    if any(k.startswith(own + "/") for k in cal):
        return own
    return f"{arch_seed}_{lut_tag(truncated_lut(Signedness.SIGNED, 2))}"


def apply_calibration(nodes, key: str) -> list[dict]:
    """Fold the committed calibration ``key`` (``scripts/make_calibration.py``) into the convs, in place.

    Per conv: filters *= 2^exp (exact in fp32; exp per layer, or per output channel), bias = the
    calibrated per-channel bias; f_min / f_max follow the filters (transform folds the filter range to constants, graph.py:129-130).
    """
    cal = _calib()
    for nd in nodes:
        if nd["kind"] != "AxConv2D":
            continue
        ek, bk = f"{key}/{nd['id']}/exp", f"{key}/{nd['id']}/bias"
        if ek not in cal:
            raise KeyError(f"no calibration {key!r} for conv {nd['id']!r} (scripts/make_calibration.py); "
                           "build the network with calibrated=False")
        a = nd["attrs"]
        e = np.asarray(cal[ek])
        if e.ndim == 0:  # one power of two per layer: codes unchanged, output scaled exactly
            f = (a["filters"] * np.float32(2.0 ** int(e))).astype(np.float32)
        else:  # one per output channel (axis 3; axis 2 of (kh, kw, C, 1) depthwise filters)
            sc = (2.0 ** e.astype(np.float64)).astype(np.float32)
            f = (a["filters"] * (sc[None, None, :, None] if a.get("depthwise") else sc[None, None, None, :]))
            f = f.astype(np.float32)
        a["filters"], a["bias"] = f, cal[bk].astype(np.float32)
        a["f_min"], a["f_max"] = float(f.min()), float(f.max())
    return nodes


def cifar_resnet(n: int, lut, seed: int = 0, width: int = 16, classes: int = 10,
                 calibrated: bool = True) -> list[dict]:
    """He et al. 6n+2 CIFAR ResNet (n=1: ResNet-8, n=10: ResNet-62), 32x32x3 input.

    Projection (1x1, stride 2) shortcuts where the shape changes.
    """
    g = _Builder(seed, lut)
    g.add("in", "Input", shape=(32, 32, 3))
    x = g.conv("stem", "in", 3, width, 3, relu=True)
    cin = width
    for stage, cout in enumerate((width, 2 * width, 4 * width)):
        for blk in range(n):
            stride = 2 if (stage > 0 and blk == 0) else 1
            p = f"s{stage}b{blk}"
            a = g.conv(f"{p}.a", x, cin, cout, 3, stride, relu=True)
            b = g.conv(f"{p}.b", a, cout, cout, 3, 1)
            short = x if (stride == 1 and cin == cout) else g.conv(f"{p}.proj", x, cin, cout, 1, stride)
            g.add(f"{p}.add", "Add", [b, short])
            x = g.add(f"{p}.relu", "ReLU", [f"{p}.add"])
            cin = cout
    g.add("pool", "AvgPool", [x], pool=(8, 8), strides=(8, 8))
    g.conv("fc", "pool", cin, classes, 1)
    if calibrated:
        apply_calibration(g.nodes, calibration_key(f"cifar{n}_s{seed}", lut))
    return g.nodes


def resnet50(lut, seed: int = 0, classes: int = 1000, calibrated: bool = True) -> list[dict]:
    """ImageNet ResNet-50 (v1.5: stride on the 3x3), 224x224x3 input, 53 convs + 1x1 classifier."""
    g = _Builder(seed, lut)
    g.add("in", "Input", shape=(224, 224, 3))
    x = g.conv("stem", "in", 3, 64, 7, 2, relu=True)
    x = g.add("maxpool", "MaxPool", [x], pool=(3, 3), strides=(2, 2), padding="same")
    cin = 64
    for stage, (mid, blocks) in enumerate(((64, 3), (128, 4), (256, 6), (512, 3))):
        cout = mid * 4
        for blk in range(blocks):
            stride = 2 if (stage > 0 and blk == 0) else 1
            p = f"s{stage}b{blk}"
            a = g.conv(f"{p}.a", x, cin, mid, 1, 1, relu=True)
            b = g.conv(f"{p}.b", a, mid, mid, 3, stride, relu=True)
            c = g.conv(f"{p}.c", b, mid, cout, 1, 1)
            short = x if blk > 0 else g.conv(f"{p}.proj", x, cin, cout, 1, stride)
            g.add(f"{p}.add", "Add", [c, short])
            x = g.add(f"{p}.relu", "ReLU", [f"{p}.add"])
            cin = cout
    g.add("pool", "AvgPool", [x], pool=(7, 7), strides=(7, 7))
    g.conv("fc", "pool", cin, classes, 1)
    if calibrated:
        apply_calibration(g.nodes, calibration_key(f"r50_s{seed}", lut))
    return g.nodes


# MobileNet v1 (Howard et al. 2017, width 1.0): (stride, output channels) of the 13 depthwise-separable blocks
MOBILENET_V1 = ((1, 64), (2, 128), (1, 128), (2, 256), (1, 256), (2, 512), (1, 512), (1, 512), (1, 512),
                (1, 512), (1, 512), (2, 1024), (1, 1024))


def mobilenet_v1(lut, seed: int = 0, classes: int = 1000, calibrated: bool = True) -> list[dict]:
    """MobileNet-v1-shaped network (BASELINE config 5's depthwise approximate conv, in context): 224x224x3,
    3x3/2 stem to 32 channels, 13 blocks of depthwise 3x3 (``depthwise=True``) + pointwise 1x1, global
    average pool, 1x1 AxConv2D classifier; BN folded into every conv.  The depthwise layers include the
    (n,112,112,32) and (n,56,56,128) shapes at stride 1 and 2 (blocks 0-3).  The reference has no
    grouped conv: a depthwise node means per-channel ``axconv2d`` with shared ranges (oracle
    ``depthwise_conv``)."""
    g = _Builder(seed, lut)
    g.add("in", "Input", shape=(224, 224, 3))
    x = g.conv("stem", "in", 3, 32, 3, 2, relu=True)
    c = 32
    for i, (stride, cout) in enumerate(MOBILENET_V1):
        x = g.dwconv(f"b{i}.dw", x, c, 3, stride)
        x = g.conv(f"b{i}.pw", x, c, cout, 1, 1, relu=True)
        c = cout
    g.add("pool", "AvgPool", [x], pool=(7, 7), strides=(7, 7))
    g.conv("fc", "pool", c, classes, 1)
    if calibrated:
        apply_calibration(g.nodes, calibration_key(f"mbv1_s{seed}", lut))
    return g.nodes


def single_conv(lut, seed: int = 0, in_shape=(32, 32, 3), cout: int = 16, k: int = 3) -> list[dict]:
    """Config 1: one approximate conv layer (3x3x3 -> 16, "same")."""
    g = _Builder(seed, lut)
    g.add("in", "Input", shape=tuple(in_shape))
    rng = g.rng
    f = rng.normal(0.0, 0.4, (k, k, in_shape[2], cout)).astype(np.float32)
    g.add("conv.in_min", "Min", ["in"])
    g.add("conv.in_max", "Max", ["in"])
    g.add("conv", "AxConv2D", ["in", "conv.in_min", "conv.in_max"], filters=f, strides=(1, 1),
          dilations=(1, 1), padding="same", lut=lut, f_min=float(f.min()), f_max=float(f.max()))
    return g.nodes


def input_shape(nodes) -> tuple[int, int, int]:
    return tuple(nodes[0]["attrs"]["shape"])


def macs_per_image(nodes) -> int:
    """Algorithmic MACs per image (graph_mac_count semantics, graph.py:316-349)."""
    from .types import ConvGeometry, output_shape

    shapes = {}
    total = 0
    for nd in nodes:
        k, a = nd["kind"], nd["attrs"]
        if k == "Input":
            shapes[nd["id"]] = (1,) + tuple(a["shape"])
        elif k == "AxConv2D":
            x = shapes[nd["inputs"][0]]
            geo = ConvGeometry(tuple(a["strides"]), tuple(a["dilations"]), a["padding"])
            fs = a["filters"].shape
            if a.get("depthwise"):  # (kh, kw, C, 1): C independent single-channel convs
                fs = (fs[0], fs[1], 1, fs[2])
                x = x[:3] + (1,)
            o = output_shape(x, fs, geo)
            kh, kw, cin, cout = fs
            total += o[1] * o[2] * kh * kw * cin * cout
            shapes[nd["id"]] = o
        elif k in ("Min", "Max"):
            shapes[nd["id"]] = ()
        elif k in ("ReLU", "Add"):
            shapes[nd["id"]] = shapes[nd["inputs"][0]]
        elif k in ("MaxPool", "AvgPool"):
            x = shapes[nd["inputs"][0]]
            ph, pw = a.get("pool", (2, 2))
            geo = ConvGeometry(tuple(a.get("strides", (ph, pw))), (1, 1), a.get("padding", "valid"))
            o = output_shape(x, (ph, pw, x[3], 1), geo)
            shapes[nd["id"]] = (1, o[1], o[2], x[3])
    return total
