"""Calibrate the synthetic ResNets on the REAL reference (run in the build container).

    python scripts/make_calibration.py

The benchmark networks have random He-normal weights.  Un-normalised, they
predict one class for every image, which makes argmax parity vacuous.  This
script folds a BatchNorm into every conv, measured on the *approximate*
network itself, on a calibration batch of the benchmark's size (ranges are per
batch, graph.py:270-275, so the statistics depend on the batch size): 1024
CIFAR images for ResNet-8, 1000 for ResNet-62, 256 ImageNet-shaped images for
ResNet-50 and the MobileNet-v1-shaped net (config 5), from their own seed.  The calibration multiplier is truncated_lut(signed, 2), the
benchmark's table, or the golden network's own table.  The reference's own ``axconv2d``
(/root/reference/pkg/src/axemu/axconv.py:266-297), run layer by layer in
graph.run order (graph.py:248-286), computes the statistics.

Per conv, with y its pre-bias approximate output on the calibration batch:
  exp  = round(log2(1 / std(y)))   one power of two per layer.  Scaling all
         filters and the filter range by 2^exp leaves the filter codes and the
         zero point unchanged, so the approximate output scales exactly by 2^exp.
  bias = round_{2^-12}(beta_c - mean_c(y * 2^exp))   per output channel.
         beta_c is the builder's N(0, 0.05) draw, or 0 for the classifier.
The MobileNet-v1-shaped net (27 convs, 13 of them depthwise with only 9 taps) needs a full BatchNorm
fold: one power of two per OUTPUT CHANNEL (the conv is re-run with the scaled filters, whose codes
change), else per-channel offsets swamp the image signal and every image gets the same class.
The exponents and biases go to paper_2002_09481_b200/calib.npz, keyed
"<arch>_s<seed>_<table tag>" (resnet.lut_tag).  That file
is a model artefact, like a checkpoint.  ``resnet.py`` applies it to the
seeded He-normal draws.
"""

from __future__ import annotations

import os
import sys
import time
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/axemu_numba_cache")
sys.dont_write_bytecode = True
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from axemu import (ConvConfig, ConvGeometry, Layout, MultLut, Range, Signedness, Tensor4,  # noqa: E402
                   axconv2d)
from axemu.graph import _pool2d  # noqa: E402

from paper_2002_09481_b200 import datasets, resnet  # noqa: E402

CALIB_SEED = resnet._CALIB_SEED


def _chscale(f, e, depthwise):
    """Filters scaled by 2^e per output channel (axis 3; axis 2 for (kh, kw, C, 1) depthwise filters)."""
    sc = (2.0 ** np.asarray(e, np.float64)).astype(np.float32)
    return (f * (sc[None, None, :, None] if depthwise else sc[None, None, None, :])).astype(np.float32)


def calibrate(nodes, images, lut: MultLut, per_channel: bool = False) -> dict:
    """per_channel: one power of two per OUTPUT CHANNEL (a full BatchNorm fold); the conv is re-run with
    the scaled filters (their codes change), so the stored statistics are the exact reference outputs."""
    vals, out = {}, {}
    for nd in nodes:
        k, a, ins = nd["kind"], nd["attrs"], nd["inputs"]
        if k == "Input":
            vals[nd["id"]] = np.asarray(images, np.float32)
        elif k in ("Min", "Max"):
            continue
        elif k == "AxConv2D":
            x = vals[ins[0]]
            f = a["filters"]
            geo = ConvGeometry(tuple(a["strides"]), tuple(a["dilations"]), a["padding"])
            rin, rf = Range(float(x.min()), float(x.max())), Range(a["f_min"], a["f_max"])
            if a.get("depthwise"):  # per-channel reference axconv2d, shared ranges (oracle depthwise_conv)
                y = np.concatenate([axconv2d(Tensor4(x[..., c:c + 1], Layout.NHWC),
                                             Tensor4(f[:, :, c:c + 1, :], Layout.HWCN), rin, rf, lut,
                                             ConvConfig(geometry=geo)).data for c in range(x.shape[3])], axis=3)
            else:
                y = axconv2d(Tensor4(x, Layout.NHWC), Tensor4(f, Layout.HWCN), rin, rf, lut,
                             ConvConfig(geometry=geo)).data
            if per_channel:
                sd = y.astype(np.float64).std(axis=(0, 1, 2))
                e = np.where(sd > 0, np.round(np.log2(1.0 / np.maximum(sd, 1e-30))), 0).astype(np.int32)
                f2 = _chscale(f, e, a.get("depthwise"))
                rf2 = Range(float(f2.min()), float(f2.max()))
                if a.get("depthwise"):
                    ys = np.concatenate([axconv2d(Tensor4(x[..., c:c + 1], Layout.NHWC),
                                                  Tensor4(f2[:, :, c:c + 1, :], Layout.HWCN), rin, rf2, lut,
                                                  ConvConfig(geometry=geo)).data for c in range(x.shape[3])],
                                        axis=3)
                else:
                    ys = axconv2d(Tensor4(x, Layout.NHWC), Tensor4(f2, Layout.HWCN), rin, rf2, lut,
                                  ConvConfig(geometry=geo)).data
            else:
                std = float(y.astype(np.float64).std())
                e = int(np.round(np.log2(1.0 / std))) if std > 0 else 0
                ys = (y * np.float32(2.0 ** e)).astype(np.float32)
            beta = np.zeros(y.shape[3]) if nd["id"] == "fc" else np.asarray(a["bias"], np.float64)
            mean = ys.astype(np.float64).mean(axis=(0, 1, 2))
            bias = (np.round((beta - mean) * 4096.0) / 4096.0).astype(np.float32)
            out[nd["id"]] = (e, bias)
            vals[nd["id"]] = (ys + bias).astype(np.float32)
        elif k == "ReLU":
            vals[nd["id"]] = np.maximum(vals[ins[0]], np.float32(0.0))
        elif k == "Add":
            vals[nd["id"]] = (vals[ins[0]] + vals[ins[1]]).astype(np.float32)
        elif k in ("MaxPool", "AvgPool"):
            vals[nd["id"]] = _pool2d(vals[ins[0]], a, take_max=(k == "MaxPool"))
        else:
            raise ValueError(k)
    return out


def golden_random_lut():
    """The random table of the r8_random golden (tests/golden/make_golden.py: default_rng(123))."""
    from paper_2002_09481_b200 import types as T

    return T.random_lut(np.random.default_rng(123), T.Signedness.SIGNED)


def main():
    from paper_2002_09481_b200 import types as T

    S, U = T.Signedness.SIGNED, T.Signedness.UNSIGNED
    trunc2 = T.truncated_lut(S, 2)
    # (arch, seed, table): the benchmark networks with the benchmark table, and the golden networks with
    # their own tables (tests/golden/make_golden.py)
    jobs = [("cifar1", 0, trunc2), ("cifar1", 3, trunc2), ("cifar10", 0, trunc2), ("cifar10", 1, trunc2),
            ("r50", 0, trunc2), ("mbv1", 0, trunc2),
            ("cifar1", 0, golden_random_lut()), ("cifar1", 3, T.truncated_lut(U, 1)),
            ("cifar10", 1, T.truncated_lut(S, 3)), ("r50", 0, T.exact_lut(S))]
    want = sys.argv[1:]
    path = ROOT / "paper_2002_09481_b200" / "calib.npz"
    store = dict(np.load(path)) if path.exists() else {}
    for arch, seed, lut_mine in jobs:
        key = f"{arch}_s{seed}_{resnet.lut_tag(lut_mine)}"
        if want and not any(w in (arch, key) for w in want):
            continue
        if any(k.startswith(key + "/") for k in store) and "--force" not in want:
            print(key, "present", flush=True)
            continue
        t0 = time.time()
        lut = MultLut(Signedness(lut_mine.mode.value), lut_mine.entries)
        if arch in ("r50", "mbv1"):
            build = resnet.resnet50 if arch == "r50" else resnet.mobilenet_v1
            nodes = build(lut_mine, seed=seed, calibrated=False)
            images = datasets.synthetic_imagenet(256, seed=CALIB_SEED)[0]
        else:
            nodes = resnet.cifar_resnet(int(arch[5:]), lut_mine, seed=seed, calibrated=False)
            images = datasets.synthetic_cifar10(1024 if arch == "cifar1" else 1000, seed=CALIB_SEED)[0]
        cal = calibrate(nodes, images, lut, per_channel=arch == "mbv1")
        for cid, (e, b) in cal.items():
            store[f"{key}/{cid}/exp"] = np.asarray(e, np.int32)
            store[f"{key}/{cid}/bias"] = b
        np.savez_compressed(path, **store)
        print(key, f"{time.time() - t0:.1f} s", "exps", [np.asarray(e).tolist() for e, _ in cal.values()][:3],
              flush=True)


if __name__ == "__main__":
    main()
