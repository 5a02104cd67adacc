"""``run_benchmark`` on the GPU engine: t_init + t_comp and the Fig. 2 phase split.

Restates the reference harness (``axemu.bench.run_benchmark``, bench.py:37-87;
phases and scoped timers, metering.py:12-46) for ``engine="b200"``:

* t_init (wall clock): model load, ``GpuGraph`` construction (filter codes,
  product tables and device LUT uploaded once) and one warm-up batch;
* t_comp (wall clock): every batch, host -> device copy, the graph run and the
  device -> host copy of the outputs (the first batch runs again, as in the
  reference, so t_comp covers the whole dataset);
* phases from CUDA events on the launching stream, summed over the timed batches:
  ``lut_lookup`` = the LUT-conv kernels (their fused dequant / bias / residual /
  ReLU epilogue included -- it cannot be split from the gather),
  ``quant_dequant_minmax`` = the rest of each conv node (quantize / im2col
  kernels) plus the graph input's range kernel, ``init`` = t_init, and
  ``im2cols_gemm_other`` = t_comp minus the two device phases (pools, adds,
  classifier, copies, host work, and the on-device decode of CIFAR-10 records,
  which the reference does at load time);
* ``per_layer`` = device seconds per executed node (fused Min/Max/ReLU/Add
  nodes have no launch of their own and do not appear);
* ``mac_count`` = algorithmic MACs of the conv launches (``meter.add_macs``,
  axconv.py:244).

Outputs are identical to the reference's for the same model and data; the
report's times are this engine's.
"""

from __future__ import annotations

import time
from pathlib import Path

import numpy as np
import torch

from .formats import CIFAR_RECORD_BYTES, RunReport, load_tensor, make_report, read_cifar10_records
from .graph import GpuGraph
from .model import load_model

ENGINES = ("b200",)


def _load_images(data, seed: int, needed: int) -> np.ndarray:
    """bench.py:23-34; a CIFAR-10 file stays as raw records (decoded on the device)."""
    if data is None:
        from .datasets import synthetic_cifar10

        images, _ = synthetic_cifar10(needed, seed)
        return images
    if isinstance(data, np.ndarray):
        return data
    path = Path(data)
    if path.suffix == ".axt":
        return load_tensor(path).data
    return read_cifar10_records(path)


def run_benchmark(model, data=None, engine: str = "b200", batches: int | None = None, batch_size: int = 1000,
                  workers: int | None = None, chunk_size: int | None = None, seed: int = 0,
                  device=None) -> tuple[RunReport, np.ndarray]:
    """Benchmark a model over the dataset on the GPU; returns (report, concatenated outputs).

    ``model``: node list, model-file path (``model.load_model``) or a ``GpuGraph``.
    ``data``: None (``synthetic_cifar10``), NHWC float32 images, (n, 3073) uint8
    CIFAR-10 records, a ``.axt`` tensor file or a CIFAR-10 binary file.
    ``workers`` / ``chunk_size`` are accepted for signature parity and never
    change bits (README.md:77-81 of the reference); ``chunk_size < 1`` is rejected
    as in ``ConvConfig`` (axconv.py:68-70).
    """
    if engine not in ENGINES:
        raise ValueError(f"engine must be 'b200' on this build (the reference's 'gemm' / 'direct' run on the "
                         f"host), got {engine!r}")
    if chunk_size is not None and chunk_size < 1:
        raise ValueError(f"chunk_size must be >= 1, got {chunk_size}")
    if batch_size < 1:
        raise ValueError(f"batch_size must be >= 1, got {batch_size}")
    t0 = time.perf_counter()
    if isinstance(model, GpuGraph):
        g = model
    else:
        nodes = load_model(model) if isinstance(model, (str, Path)) else model
        g = GpuGraph(nodes, device=device)
    images = _load_images(data, seed, batch_size * (batches or 1))
    records = images.dtype == np.uint8
    if records and (images.ndim != 2 or images.shape[1] != CIFAR_RECORD_BYTES):
        raise ValueError(f"uint8 data must be (n, {CIFAR_RECORD_BYTES}) CIFAR-10 records")
    if not records:
        images = np.ascontiguousarray(images, dtype=np.float32)
    n = images.shape[0]
    if n == 0:
        raise ValueError("no input images to benchmark")
    available = -(-n // batch_size)
    n_batches = available if batches is None else min(batches, available)
    slices = [torch.from_numpy(np.ascontiguousarray(images[i * batch_size:min((i + 1) * batch_size, n)]))
              for i in range(n_batches)]

    g.run(slices[0]).cpu()
    torch.cuda.synchronize(g.device)
    t_init = time.perf_counter() - t0

    timeline: list = []
    profile: list = []
    outputs = []
    t1 = time.perf_counter()
    for batch in slices:
        out = g.run(batch, timeline=timeline, profile=profile)
        outputs.append(out.cpu().numpy())  # D2H of the batch result (synchronises the stream)
    t_comp = time.perf_counter() - t1

    lut_node: dict[str, float] = {}
    mac_count = 0
    for nid, e0, e1, macs, *_ in profile:
        lut_node[nid] = lut_node.get(nid, 0.0) + e0.elapsed_time(e1) / 1e3
        mac_count += int(macs)
    per_layer: dict[str, float] = {}
    quant_s = 0.0
    for nid, kind, e0, e1 in timeline:
        s = e0.elapsed_time(e1) / 1e3
        per_layer[nid] = per_layer.get(nid, 0.0) + s
        if kind == "Input" and nid in g.need_range and not records:  # range kernel of the graph input
            quant_s += s
    lut_s = sum(lut_node.values())
    for nid, s in lut_node.items():  # conv node time minus its conv kernel = quantize / im2col kernels
        quant_s += max(0.0, per_layer[nid] - s)
    report = make_report(t_init=t_init, t_comp=t_comp, lut_s=lut_s, quant_s=quant_s, mac_count=mac_count,
                         per_layer=per_layer)
    return report, np.concatenate(outputs, axis=0)


def speedup(baseline: RunReport, current: RunReport) -> float:
    """How many times faster the current run is than the baseline (total time; bench.py:90-94)."""
    if current.total <= 0:
        raise ValueError("current run has no measured time")
    return baseline.total / current.total
