"""Host-side types of the approximate-convolution operator API.

Mirrors the reference interface objects the hot path takes
(``axemu.tensor`` / ``quantizer`` / ``axmult`` / ``axconv``): same names,
same field meaning, same validation errors.  Objects created by the
reference package itself are accepted everywhere too -- the adapters read
them by attribute and compare enums by their string ``value``.

Reference anchors (``/root/reference/pkg/src/axemu``):
  Layout / Tensor4 / Range / ConvGeometry   tensor.py:20-87
  resolve_padding / output_shape            tensor.py:94-140
  Signedness / RoundMode / QuantParams      quantizer.py:28-74
  compute_coeffs                            quantizer.py:98-117 (via axb_coeffs_host)
  MultLut / stitch_index / table builders   axmult.py:22-96
  Accumulator / ConvConfig / conv_mac_count axconv.py:47-71, :106-114
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field

import numpy as np

LUT_ENTRIES = 1 << 16
LUT_TABLE_BYTES = LUT_ENTRIES * 2


class Layout(enum.Enum):
    NHWC = "NHWC"
    HWCN = "HWCN"


class Signedness(enum.Enum):
    UNSIGNED = "unsigned"
    SIGNED = "signed"

    @property
    def bounds(self) -> tuple[int, int]:
        return {"unsigned": (0, 255), "signed": (-128, 127)}[self.value]

    @property
    def code_dtype(self) -> np.dtype:
        return np.dtype(np.int8 if self.value == "signed" else np.uint8)

    @property
    def entry_dtype(self) -> np.dtype:
        return np.dtype(np.int16 if self.value == "signed" else np.uint16)


class RoundMode(enum.Enum):
    HALF_AWAY_FROM_ZERO = "half-away-from-zero"
    HALF_TO_EVEN = "half-to-even"
    TOWARD_ZERO = "toward-zero"


class Accumulator(enum.Enum):
    EXACT64 = "exact64"
    WRAP32 = "wrap32"
    SATURATE32 = "saturate32"


@dataclass(frozen=True)
class Tensor4:
    """Dense 4-D float32 tensor with a layout tag (NHWC activations, HWCN filters)."""

    data: np.ndarray
    layout: Layout = Layout.NHWC

    def __post_init__(self) -> None:
        arr = np.ascontiguousarray(self.data, dtype=np.float32)
        if arr.ndim != 4:
            raise ValueError(f"Tensor4 needs 4 dimensions, got {arr.ndim}")
        if not isinstance(self.layout, Layout):
            raise TypeError(f"layout must be a Layout, got {type(self.layout).__name__}")
        object.__setattr__(self, "data", arr)

    @property
    def shape(self) -> tuple[int, int, int, int]:
        return tuple(int(v) for v in self.data.shape)  # type: ignore[return-value]

    @property
    def size(self) -> int:
        return int(self.data.size)


@dataclass(frozen=True)
class Range:
    """Closed, finite value interval [min, max]."""

    min: float
    max: float

    def __post_init__(self) -> None:
        if not (math.isfinite(self.min) and math.isfinite(self.max)):
            raise ValueError(f"range must be finite, got ({self.min}, {self.max})")
        if self.min > self.max:
            raise ValueError(f"range min {self.min} exceeds max {self.max}")


@dataclass(frozen=True)
class ConvGeometry:
    strides: tuple[int, int] = (1, 1)
    dilations: tuple[int, int] = (1, 1)
    padding: str | tuple[int, int, int, int] = "valid"

    def __post_init__(self) -> None:
        for label, pair in (("strides", self.strides), ("dilations", self.dilations)):
            if len(pair) != 2 or any(int(v) != v or v < 1 for v in pair):
                raise ValueError(f"{label} must be two positive integers, got {pair}")
        pad = self.padding
        if isinstance(pad, str):
            if pad not in ("valid", "same"):
                raise ValueError(f"padding must be 'valid', 'same', or 4 integers, got {pad!r}")
        elif len(pad) != 4 or any(int(v) != v or v < 0 for v in pad):
            raise ValueError(f"explicit padding needs 4 non-negative integers, got {pad}")


@dataclass(frozen=True)
class QuantParams:
    scale: float
    zero_point: int
    mode: Signedness
    round_mode: RoundMode = RoundMode.HALF_AWAY_FROM_ZERO

    def __post_init__(self) -> None:
        if not (math.isfinite(self.scale) and self.scale > 0):
            raise ValueError(f"scale must be positive and finite, got {self.scale}")
        lo, hi = _bounds(self.mode)
        if not lo <= self.zero_point <= hi:
            raise ValueError(f"zero point {self.zero_point} outside [{lo}, {hi}]")


@dataclass(frozen=True)
class MultLut:
    """65,536-entry 16-bit truth table, index (a_byte << 8) | b_byte."""

    mode: Signedness
    entries: np.ndarray

    def __post_init__(self) -> None:
        arr = np.ascontiguousarray(self.entries)
        if arr.shape != (LUT_ENTRIES,):
            raise ValueError(f"truth table needs {LUT_ENTRIES} entries, got shape {arr.shape}")
        want = np.dtype(np.int16 if _mode_value(self.mode) == "signed" else np.uint16)
        if arr.dtype != want:
            raise ValueError(
                f"entries dtype {arr.dtype} does not match mode {_mode_value(self.mode)} (expected {want})"
            )
        object.__setattr__(self, "entries", arr)

    @property
    def raw(self) -> np.ndarray:
        return self.entries.view(np.uint16)


@dataclass(frozen=True)
class ConvConfig:
    geometry: ConvGeometry = field(default_factory=ConvGeometry)
    chunk_size: int | None = None  # accepted for API parity; never changes bits
    accumulator: Accumulator = Accumulator.EXACT64
    round_mode: RoundMode = RoundMode.HALF_AWAY_FROM_ZERO
    workers: int | None = None  # accepted for API parity; the GPU ignores it

    def __post_init__(self) -> None:
        if self.chunk_size is not None and self.chunk_size < 1:
            raise ValueError(f"chunk_size must be >= 1, got {self.chunk_size}")


# ---------------------------------------------------------------------------
# duck-typed accessors (reference objects work too)


def _mode_value(mode) -> str:
    return getattr(mode, "value", mode)


def _bounds(mode) -> tuple[int, int]:
    return (-128, 127) if _mode_value(mode) == "signed" else (0, 255)


def is_signed(mode) -> bool:
    return _mode_value(mode) == "signed"


def layout_name(layout) -> str:
    return getattr(layout, "value", layout)


# ---------------------------------------------------------------------------
# geometry


def resolve_padding(geometry, in_h: int, in_w: int, kh: int, kw: int) -> tuple[int, int, int, int]:
    """Concrete (top, bottom, left, right); "same" puts the odd cell bottom/right."""
    pad = geometry.padding
    if not isinstance(pad, str):
        return tuple(int(v) for v in pad)  # type: ignore[return-value]
    if pad == "valid":
        return (0, 0, 0, 0)
    out = []
    for size, k, s, d in ((in_h, kh, geometry.strides[0], geometry.dilations[0]),
                          (in_w, kw, geometry.strides[1], geometry.dilations[1])):
        n_out = (size + s - 1) // s
        total = max(0, (n_out - 1) * s + (k - 1) * d + 1 - size)
        out.extend((total // 2, total - total // 2))
    return (out[0], out[1], out[2], out[3])


def output_shape(input_shape, filter_shape, geometry) -> tuple[int, int, int, int]:
    n, h, w, c = (int(v) for v in input_shape)
    kh, kw, fc, cout = (int(v) for v in filter_shape)
    if fc != c:
        raise ValueError(f"filter channels {fc} do not match input channels {c}")
    pt, pb, pl, pr = resolve_padding(geometry, h, w, kh, kw)
    dims = []
    for size, pad, k, s, d in ((h, pt + pb, kh, geometry.strides[0], geometry.dilations[0]),
                               (w, pl + pr, kw, geometry.strides[1], geometry.dilations[1])):
        extent = (k - 1) * d + 1
        if size + pad < extent:
            raise ValueError(f"kernel extent {extent} exceeds padded input {size + pad}")
        dims.append((size + pad - extent) // s + 1)
    return (n, dims[0], dims[1], cout)


def conv_mac_count(input_shape, filter_shape, geometry) -> int:
    n, oh, ow, cout = output_shape(input_shape, filter_shape, geometry)
    kh, kw, cin, _ = filter_shape
    return int(n) * oh * ow * int(kh) * int(kw) * int(cin) * int(cout)


# ---------------------------------------------------------------------------
# coefficients (single implementation: the C ABI's host function)


def compute_coeffs(rng, mode, round_mode=RoundMode.HALF_AWAY_FROM_ZERO) -> QuantParams:
    from . import _lib

    out = _lib.QParams()
    rm = _lib.ROUND[_mode_value(round_mode)]
    _lib.check(_lib.load().axb_coeffs_host(float(rng.min), float(rng.max), int(is_signed(mode)), rm, out))
    m = mode if isinstance(mode, Signedness) else Signedness(_mode_value(mode))
    r = round_mode if isinstance(round_mode, RoundMode) else RoundMode(_mode_value(round_mode))
    return QuantParams(scale=out.scale, zero_point=int(out.zero_point), mode=m, round_mode=r)


# ---------------------------------------------------------------------------
# table builders (axmult.py:66-96) -- host data generation


def stitch_index(a: int, b: int) -> int:
    return ((a & 0xFF) << 8) | (b & 0xFF)


def _operand_values(mode) -> np.ndarray:
    v = np.arange(256, dtype=np.int32)
    return v.astype(np.int8).astype(np.int32) if is_signed(mode) else v


def exact_lut(mode) -> MultLut:
    v = _operand_values(mode)
    m = mode if isinstance(mode, Signedness) else Signedness(_mode_value(mode))
    return MultLut(m, np.multiply.outer(v, v).ravel().astype(m.entry_dtype))


def truncated_lut(mode, drop_bits: int) -> MultLut:
    if not 0 <= drop_bits <= 7:
        raise ValueError(f"drop_bits must be in 0..7, got {drop_bits}")
    keep = (0xFF << drop_bits) & 0xFF
    v = _operand_values(mode)
    t = np.sign(v) * (np.abs(v) & keep)
    m = mode if isinstance(mode, Signedness) else Signedness(_mode_value(mode))
    return MultLut(m, np.multiply.outer(t, t).ravel().astype(m.entry_dtype))


def perturbed_lut(rng: np.random.Generator, mode, err_bits: int) -> MultLut:
    """Exact products plus a uniform integer error in [-2^err_bits, 2^err_bits] per entry, clipped to
    the 16-bit entry range: a stand-in for a characterised approximate multiplier (error-injected
    candidate for multiplier sweeps; a uniform random table makes deep networks diverge)."""
    m = mode if isinstance(mode, Signedness) else Signedness(_mode_value(mode))
    v = _operand_values(m)
    exact = np.multiply.outer(v, v).ravel().astype(np.int64)
    e = rng.integers(-(1 << err_bits), (1 << err_bits) + 1, exact.size)
    lo, hi = (-(1 << 15), (1 << 15) - 1) if m is Signedness.SIGNED else (0, (1 << 16) - 1)
    return MultLut(m, np.clip(exact + e, lo, hi).astype(m.entry_dtype))


def random_lut(rng: np.random.Generator, mode) -> MultLut:
    """Uniform random 16-bit table (the reference tests' generator, cases.py:25-30)."""
    m = mode if isinstance(mode, Signedness) else Signedness(_mode_value(mode))
    if m is Signedness.UNSIGNED:
        return MultLut(m, rng.integers(0, 1 << 16, 65536).astype(np.uint16))
    return MultLut(m, rng.integers(-(1 << 15), 1 << 15, 65536).astype(np.int16))
