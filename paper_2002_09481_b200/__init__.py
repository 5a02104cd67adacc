"""paper_2002_09481_b200 -- B200-native approximate-convolution path (TFApprox / axemu).

The hot path of the reference ``axemu`` package (quantized 8-bit conv2d whose
multiply is a 65,536-entry truth-table lookup) rebuilt as sm_100a CUDA
kernels behind a C ABI (``include/axb.h``, ``libaxb.so``), driven from
Python through ctypes and a torch custom op.

Public API (mirrors the reference names):
  axconv2d, torch_axconv2d, DeviceLut          -- the operator (axconv.py)
  Tensor4, Range, ConvGeometry, ConvConfig, MultLut, Signedness, RoundMode,
  Accumulator, QuantParams, compute_coeffs, exact_lut, truncated_lut, ...
  graph.GpuGraph / graph.run                    -- GPU executor for AxConv2D graphs
  model.transform / save_model / load_model     -- Conv2D -> AxConv2D, model files
  formats.*                                     -- .axm / .axt / CIFAR-10 / report files
  benchmark.run_benchmark / speedup             -- t_init + t_comp RunReport on the GPU engine
  resnet.*                                      -- ResNet graph builders (benchmarks)
"""

from .types import (  # noqa: F401
    Accumulator,
    ConvConfig,
    ConvGeometry,
    Layout,
    MultLut,
    QuantParams,
    Range,
    RoundMode,
    Signedness,
    Tensor4,
    compute_coeffs,
    conv_mac_count,
    exact_lut,
    output_shape,
    perturbed_lut,
    random_lut,
    resolve_padding,
    stitch_index,
    truncated_lut,
)
from .axconv import DeviceLut, axconv2d, device_lut, torch_axconv2d  # noqa: F401

__version__ = "0.1.0"
