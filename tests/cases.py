"""Restatement of the reference test-case generators (tests/cases.py in axemu).

random_conv_case replays the exact rng draw sequence of the reference's
``random_conv_case`` (pkg/tests/cases.py:33-99) so seeded case streams are
identical; tests/golden/make_golden.py asserts that against the real
reference when it regenerates the fixtures.  Modes are plain strings
(oracle vocabulary).
"""

from __future__ import annotations

import numpy as np

from oracle import axemu_oracle as O

MODES = [O.UNSIGNED, O.SIGNED]
ROUNDS = [O.HALF_AWAY, O.HALF_EVEN, O.TOWARD_ZERO]
ACCS = [O.EXACT64, O.WRAP32, O.SATURATE32]


def random_conv_case(rng: np.random.Generator, exact_only: bool = False) -> dict:
    mode = MODES[int(rng.choice(2))]
    n = int(rng.integers(1, 5))
    h = int(rng.integers(1, 9))
    w = int(rng.integers(1, 9))
    cin = int(rng.integers(1, 5))
    cout = int(rng.integers(1, 5))
    pad_kind = ["valid", "same", "explicit"][int(rng.choice(3))]
    dh = int(rng.integers(1, 3))
    dw = int(rng.integers(1, 3))
    if pad_kind == "valid":
        kh = int(rng.integers(1, (h - 1) // dh + 2))
        kw = int(rng.integers(1, (w - 1) // dw + 2))
        padding = "valid"
    elif pad_kind == "same":
        kh = int(rng.integers(1, 5))
        kw = int(rng.integers(1, 5))
        padding = "same"
    else:
        kh = int(rng.integers(1, (h - 1) // dh + 2))
        kw = int(rng.integers(1, (w - 1) // dw + 2))
        padding = tuple(int(v) for v in rng.integers(0, 3, 4))
    strides = (int(rng.integers(1, 4)), int(rng.integers(1, 4)))
    lo = float(rng.uniform(-4.0, 0.5))
    hi = lo + float(rng.uniform(0.1, 6.0))
    x = rng.uniform(lo, hi, (n, h, w, cin)).astype(np.float32)
    f = rng.normal(0.0, 1.5, (kh, kw, cin, cout)).astype(np.float32)
    if exact_only:
        lut = O.exact_lut(mode)
    else:
        pick = rng.integers(0, 3)
        if pick == 0:
            lut = O.exact_lut(mode)
        elif pick == 1:
            lut = O.truncated_lut(mode, int(rng.integers(0, 8)))
        else:
            lut = O.random_lut(rng, mode)
    if exact_only or rng.random() < 0.7:
        acc = O.EXACT64
    else:
        acc = [O.WRAP32, O.SATURATE32][int(rng.choice(2))]
    chunk = [None, 1, 2, 3][int(rng.choice(4))]
    round_mode = ROUNDS[int(rng.choice(3))]
    workers = [None, 1, 2, 8][int(rng.choice(4))]
    return dict(x=x, f=f, in_range=(float(x.min()), float(x.max())),
                f_range=(float(f.min()), float(f.max())), lut=lut, mode=mode, padding=padding,
                strides=strides, dilations=(dh, dw), accumulator=acc, round_mode=round_mode,
                chunk=chunk, workers=workers)


def oracle_conv(case, engine="gemm", return_acc=False):
    fn = O.axconv2d if engine == "gemm" else O.direct_conv
    kw = dict(padding=case["padding"], strides=case["strides"], dilations=case["dilations"],
              accumulator=case["accumulator"], round_mode=case["round_mode"])
    if return_acc:
        return O.axconv2d(case["x"], case["f"], case["in_range"], case["f_range"], case["lut"],
                          case["mode"], return_acc=True, **kw)
    return fn(case["x"], case["f"], case["in_range"], case["f_range"], case["lut"], case["mode"], **kw)


def model_graph_spec():
    """Deterministic small float graph: conv-relu-conv(stride 2)+proj add-relu-avgpool-1x1 conv."""
    rng = np.random.default_rng(99)
    f = lambda *s: (rng.standard_normal(s) * 0.3).astype(np.float32)  # noqa: E731
    return [
        ("in", "Input", [], {"shape": [12, 12, 3]}),
        ("c1", "Conv2D", ["in"], {"filters": f(3, 3, 3, 8), "bias": f(8), "strides": [1, 1], "dilations": [1, 1],
                                  "padding": "same"}),
        ("r1", "ReLU", ["c1"], {}),
        ("c2", "Conv2D", ["r1"], {"filters": f(3, 3, 8, 16), "bias": f(16), "strides": [2, 2], "dilations": [1, 1],
                                  "padding": "same"}),
        ("p2", "Conv2D", ["r1"], {"filters": f(1, 1, 8, 16), "strides": [2, 2], "dilations": [1, 1],
                                  "padding": "valid"}),
        ("a2", "Add", ["c2", "p2"], {}),
        ("r2", "ReLU", ["a2"], {}),
        ("gp", "AvgPool", ["r2"], {"pool": [6, 6], "strides": [6, 6], "padding": "valid"}),
        ("fc", "Conv2D", ["gp"], {"filters": f(1, 1, 16, 5), "bias": f(5), "strides": [1, 1], "dilations": [1, 1],
                                  "padding": "valid"}),
    ]
