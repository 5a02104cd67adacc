"""Drop-in ``axconv2d``: the reference operator API over the B200 kernels.

``axconv2d(inputs, filters, in_range, f_range, lut, cfg, meter=None)`` has the
signature, argument meaning, output bits and error behaviour of the
reference ``axemu.axconv.axconv2d`` (``/root/reference/pkg/src/axemu/axconv.py:266-297``):
NHWC float32 inputs, HWCN float32 filters, per-batch ranges, a 65,536-entry
truth table and a ``ConvConfig``; it returns an NHWC float32 ``Tensor4``.
The work runs in ``libaxb.so`` (``axb_axconv2d``): quantize + zp-pad (K2),
filter preparation, the LUT implicit GEMM with the fused correction /
dequantize epilogue (K3).  ``chunk_size`` and ``workers`` are accepted and
ignored -- as in the reference, they can never change the bits.

``torch_axconv2d`` is the same operator on CUDA torch tensors (no host
copies), also registered as the torch custom op ``axb::axconv2d``.
"""

from __future__ import annotations

import hashlib
import threading

import numpy as np
import torch

from . import _lib
from .types import (
    Accumulator,
    ConvConfig,
    Layout,
    RoundMode,
    Tensor4,
    _mode_value,
    compute_coeffs,
    conv_mac_count,
    is_signed,
    layout_name,
    output_shape,
    resolve_padding,
)

PHASE_LUT = "lut_lookup"  # metering.py:13 phase names, for a reference Meter


class DeviceLut:
    """A truth table resident on one CUDA device (an ``axb_lut`` handle).

    Uploads the 128 KiB table once and keeps a b-major transposed copy for
    the conv kernels (``axb_lut_create``).
    """

    def __init__(self, lut, device: int | None = None):
        entries = np.ascontiguousarray(lut.entries)
        if entries.shape != (65536,):
            raise ValueError(f"truth table needs 65536 entries, got shape {entries.shape}")
        self.signed = is_signed(lut.mode)
        self.mode = _mode_value(lut.mode)
        self.device = torch.cuda.current_device() if device is None else int(device)
        raw = np.ascontiguousarray(entries.view(np.uint16))
        self.entries = raw.copy()
        lib = _lib.load()
        h = _lib.c_vp()
        with torch.cuda.device(self.device):
            _lib.check(lib.axb_lut_create(raw.ctypes.data, int(self.signed), h))
        self.handle = h

    def __del__(self):  # pragma: no cover - interpreter teardown order
        try:
            if getattr(self, "handle", None) and self.handle.value:
                with torch.cuda.device(self.device):
                    _lib.load().axb_lut_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


_lut_cache: dict[tuple, DeviceLut] = {}
_lut_lock = threading.Lock()


def device_lut(lut, device: int | None = None) -> DeviceLut:
    """Cached DeviceLut for a (table bytes, mode, device)."""
    if isinstance(lut, DeviceLut):
        return lut
    dev = torch.cuda.current_device() if device is None else int(device)
    entries = np.ascontiguousarray(lut.entries)
    key = (hashlib.blake2b(entries.view(np.uint8), digest_size=16).digest(), _mode_value(lut.mode), dev)
    with _lut_lock:
        d = _lut_cache.get(key)
        if d is None:
            if len(_lut_cache) > 64:
                _lut_cache.clear()
            d = DeviceLut(lut, dev)
            _lut_cache[key] = d
        return d


def _require_cuda() -> None:
    if not torch.cuda.is_available():
        raise _lib.AxbError("axconv2d needs a CUDA device (the B200 path has no CPU fallback)")


def _check_operands(inputs, filters) -> None:
    """Same checks and messages as axconv.py:117-125."""
    if layout_name(inputs.layout) != "NHWC":
        raise ValueError("input tensor must be NHWC")
    if layout_name(filters.layout) != "HWCN":
        raise ValueError("filter tensor must be HWCN")
    if inputs.shape[3] != filters.shape[2]:
        raise ValueError(
            f"filter channels {filters.shape[2]} do not match input channels {inputs.shape[3]}"
        )


def torch_axconv2d(
    x: torch.Tensor,
    f: torch.Tensor,
    in_range: tuple[float, float],
    f_range: tuple[float, float],
    lut,
    geometry,
    accumulator="exact64",
    round_mode="half-away-from-zero",
    acc_out: torch.Tensor | None = None,
) -> torch.Tensor:
    """axconv2d on CUDA tensors: x (n,h,w,c) fp32, f (kh,kw,c,cout) fp32 -> (n,oh,ow,cout)."""
    _require_cuda()
    if x.dim() != 4 or f.dim() != 4:
        raise ValueError("axconv2d expects 4-D NHWC input and HWCN filters")
    if x.shape[3] != f.shape[2]:
        raise ValueError(f"filter channels {f.shape[2]} do not match input channels {x.shape[3]}")
    x = x.contiguous().to(torch.float32)
    f = f.contiguous().to(device=x.device, dtype=torch.float32)
    n, h, w, c = (int(v) for v in x.shape)
    kh, kw, _, cout = (int(v) for v in f.shape)
    _, oh, ow, _ = output_shape((n, h, w, c), (kh, kw, c, cout), geometry)
    pt, pb, pl, pr = resolve_padding(geometry, h, w, kh, kw)
    out = torch.empty((n, oh, ow, cout), dtype=torch.float32, device=x.device)
    if n == 0:
        return out
    dl = device_lut(lut, x.device.index)
    if acc_out is not None:
        assert acc_out.dtype == torch.int64 and acc_out.shape == out.shape and acc_out.is_contiguous()
    stream = torch.cuda.current_stream(x.device).cuda_stream
    with torch.cuda.device(x.device):  # the library launches and allocates on the current device
        rc = _lib.load().axb_axconv2d(
            x.data_ptr(), n, h, w, c, f.data_ptr(), kh, kw, cout,
            int(geometry.strides[0]), int(geometry.strides[1]),
            int(geometry.dilations[0]), int(geometry.dilations[1]), pt, pb, pl, pr,
            float(in_range[0]), float(in_range[1]), float(f_range[0]), float(f_range[1]),
            _lib.ROUND[_mode_value(round_mode)], _lib.ACC[_mode_value(accumulator)], dl.handle,
            out.data_ptr(), acc_out.data_ptr() if acc_out is not None else None, stream,
        )
    _lib.check(rc)
    return out


def axconv2d(inputs, filters, in_range, f_range, lut, cfg=None, meter=None) -> Tensor4:
    """Reference-compatible approximate conv2d (axconv.py:266-297) on the GPU."""
    cfg = cfg or ConvConfig()
    _check_operands(inputs, filters)
    # coefficient validation and errors exactly as the reference (Range / QuantParams)
    compute_coeffs(in_range, lut.mode, cfg.round_mode)
    compute_coeffs(f_range, lut.mode, cfg.round_mode)
    geom = cfg.geometry
    n, oh, ow, cout = output_shape(inputs.shape, filters.shape, geom)
    if n == 0:
        return Tensor4(np.zeros((0, oh, ow, cout), np.float32), Layout.NHWC)
    _require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    x = torch.from_numpy(np.ascontiguousarray(inputs.data, dtype=np.float32)).to(dev)
    f = torch.from_numpy(np.ascontiguousarray(filters.data, dtype=np.float32)).to(dev)
    y = torch_axconv2d(x, f, (in_range.min, in_range.max), (f_range.min, f_range.max), lut, geom,
                       _mode_value(cfg.accumulator), _mode_value(cfg.round_mode))
    if meter is not None and hasattr(meter, "add_macs"):
        meter.add_macs(conv_mac_count(inputs.shape, filters.shape, geom))
    return Tensor4(y.cpu().numpy(), Layout.NHWC)


# ---------------------------------------------------------------------------
# torch custom op (the op a torch-side graph or user code calls)

_LUT_REGISTRY: dict[int, object] = {}


def register_lut(lut) -> int:
    """Register a table for use by the torch custom op; returns its id."""
    key = id(lut)
    _LUT_REGISTRY[key] = lut
    return key


@torch.library.custom_op("axb::axconv2d", mutates_args=())
def _axconv2d_op(x: torch.Tensor, f: torch.Tensor, in_min: float, in_max: float, f_min: float,
                 f_max: float, lut_id: int, strides: list[int], dilations: list[int],
                 padding: list[int], accumulator: str, round_mode: str) -> torch.Tensor:
    from .types import ConvGeometry

    geom = ConvGeometry(tuple(strides), tuple(dilations), tuple(padding))
    return torch_axconv2d(x, f, (in_min, in_max), (f_min, f_max), _LUT_REGISTRY[lut_id], geom,
                          accumulator, round_mode)


@_axconv2d_op.register_fake
def _(x, f, in_min, in_max, f_min, f_max, lut_id, strides, dilations, padding, accumulator, round_mode):
    from .types import ConvGeometry

    geom = ConvGeometry(tuple(strides), tuple(dilations), tuple(padding))
    n, oh, ow, cout = output_shape(tuple(x.shape), tuple(f.shape), geom)
    return x.new_empty((n, oh, ow, cout))


__all__ = ["axconv2d", "torch_axconv2d", "DeviceLut", "device_lut", "register_lut", "Accumulator",
           "RoundMode"]
