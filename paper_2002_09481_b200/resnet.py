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

Weights are synthetic: He-normal filters, N(0, 0.05) biases, from a seed.
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


def cifar_resnet(n: int, lut, seed: int = 0, width: int = 16, classes: int = 10) -> list[dict]:
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
    return g.nodes


def resnet50(lut, seed: int = 0, classes: int = 1000) -> list[dict]:
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
            o = output_shape(x, a["filters"].shape, geo)
            kh, kw, cin, cout = a["filters"].shape
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
