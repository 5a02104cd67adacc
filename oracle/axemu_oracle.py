"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the approximate-convolution path.

A from-scratch restatement of the reference package ``axemu``
(``/root/reference/pkg/src/axemu``) in numpy plus one small C library
(``oracle/c/axemu_oracle.c``: the int64 LUT-GEMM and the nested-loop direct
convolution, OpenMP-parallel).  Every function cites the reference
``file:line`` it restates.

Pinning: ``tests/test_oracle_golden.py`` checks this oracle bit-for-bit
against golden vectors produced by the *real* reference imported in the
build container (``tests/golden/make_golden.py`` writes
``tests/golden/*.npz``), plus the reference's own known-answer tests.

Allowed importers: ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs -- as the checker or as the
timed CPU baseline, never as the product path.  The product package
(``paper_2002_09481_b200``) does not import this module.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "libaxemu_oracle.so"

SIGNED = "signed"
UNSIGNED = "unsigned"
HALF_AWAY = "half-away-from-zero"
HALF_EVEN = "half-to-even"
TOWARD_ZERO = "toward-zero"
EXACT64 = "exact64"
WRAP32 = "wrap32"
SATURATE32 = "saturate32"

LEVELS = 256  # quantizer.py:21
GRID_SNAP = 2.0**-16  # quantizer.py:25
INT32_MIN = -(1 << 31)  # axconv.py:43
INT32_MAX = (1 << 31) - 1  # axconv.py:44


# ---------------------------------------------------------------------------
# native helpers


def build_lib(force: bool = False) -> Path:
    """Compile oracle/c/axemu_oracle.c with gcc -O3 -fopenmp (oracle/Makefile recipe)."""
    src = HERE / "c" / "axemu_oracle.c"
    if LIB_PATH.exists() and not force and LIB_PATH.stat().st_mtime >= src.stat().st_mtime:
        return LIB_PATH
    LIB_PATH.parent.mkdir(parents=True, exist_ok=True)
    subprocess.check_call(
        ["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-fPIC", "-shared",
         "-o", str(LIB_PATH), str(src)]
    )
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        path = LIB_PATH if LIB_PATH.exists() else build_lib()
        _lib = ctypes.CDLL(str(path))
        i64 = ctypes.c_int64
        p = ctypes.c_void_p
        _lib.lut_matmul.argtypes = [p, p, p, i64, i64, i64, p]
        _lib.lut_matmul.restype = None
        _lib.direct_lut_sums.argtypes = [p, p, p, p] + [i64] * 13 + [p, p]
        _lib.direct_lut_sums.restype = None
        _lib.oracle_max_threads.restype = ctypes.c_int
    return _lib


def threads() -> int:
    return int(lib().oracle_max_threads())


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


# ---------------------------------------------------------------------------
# quantizer.py restatement


def bounds(mode: str) -> tuple[int, int]:
    """quantizer.py:33-34"""
    return (0, 255) if mode == UNSIGNED else (-128, 127)


def code_dtype(mode: str):
    """quantizer.py:37-38"""
    return np.uint8 if mode == UNSIGNED else np.int8


def entry_dtype(mode: str):
    """quantizer.py:40-43"""
    return np.uint16 if mode == UNSIGNED else np.int16


def apply_round(x, round_mode: str):
    """quantizer.py:52-57"""
    if round_mode == HALF_AWAY:
        return np.copysign(np.floor(np.abs(x) + 0.5), x)
    if round_mode == HALF_EVEN:
        return np.rint(x)
    return np.trunc(x)


def compute_coeffs(mn: float, mx: float, mode: str, round_mode: str = HALF_AWAY):
    """(scale, zero_point) -- quantizer.py:98-117."""
    mn = min(mn, 0.0)
    mx = max(mx, 0.0)
    scale = (mx - mn) / (LEVELS - 1)
    if scale == 0.0:
        scale = 1.0
    lo, hi = bounds(mode)
    zp_real = lo - mn / scale
    zp = int(np.clip(apply_round(np.float64(zp_real), round_mode), lo, hi))
    return scale, zp


def quantize_values(values, scale: float, zp: int, mode: str, round_mode: str = HALF_AWAY):
    """quantizer.py:120-131 (raises ValueError on non-finite input)."""
    values = np.asarray(values)
    if not np.isfinite(values).all():
        raise ValueError("cannot quantize non-finite values")
    x = values.astype(np.float64) / scale
    nearest = np.rint(x)
    snapped = np.abs(x - nearest) <= GRID_SNAP * np.maximum(1.0, np.abs(x))
    rounded = np.where(snapped, nearest, apply_round(x, round_mode))
    lo, hi = bounds(mode)
    codes = np.clip(rounded + zp, lo, hi)
    return codes.astype(code_dtype(mode))


def dequantize_values(codes, scale: float, zp: int):
    """quantizer.py:134-137"""
    return ((codes.astype(np.float64) - zp) * scale).astype(np.float32)


# ---------------------------------------------------------------------------
# tensor.py restatement


def resolve_padding(padding, strides, dilations, in_h, in_w, kh, kw):
    """tensor.py:94-115 ("same" puts the odd cell bottom/right)."""
    if isinstance(padding, (tuple, list)):
        return tuple(int(v) for v in padding)
    if padding == "valid":
        return (0, 0, 0, 0)
    pads = []
    for size, k, s, d in ((in_h, kh, strides[0], dilations[0]), (in_w, kw, strides[1], dilations[1])):
        out = -(-size // s)
        total = max(0, (out - 1) * s + (k - 1) * d + 1 - size)
        pads.append((total // 2, total - total // 2))
    (pt, pb), (pl, pr) = pads
    return (pt, pb, pl, pr)


def output_shape(in_shape, f_shape, padding, strides, dilations):
    """tensor.py:118-140"""
    n, h, w, c = in_shape
    kh, kw, fc, cout = f_shape
    if fc != c:
        raise ValueError(f"filter channels {fc} do not match input channels {c}")
    pt, pb, pl, pr = resolve_padding(padding, strides, dilations, h, w, kh, kw)
    out = []
    for size, pad, k, s, d in ((h, pt + pb, kh, strides[0], dilations[0]),
                               (w, pl + pr, kw, strides[1], dilations[1])):
        span = size + pad - ((k - 1) * d + 1)
        if span < 0:
            raise ValueError(f"kernel extent {(k - 1) * d + 1} exceeds padded input {size + pad}")
        out.append(span // s + 1)
    return (n, out[0], out[1], cout)


# ---------------------------------------------------------------------------
# axmult.py restatement (table builders)


def operand_values(mode: str) -> np.ndarray:
    """axmult.py:66-71"""
    vals = np.arange(256, dtype=np.int32)
    if mode == SIGNED:
        vals = vals.astype(np.int8).astype(np.int32)
    return vals


def exact_lut(mode: str) -> np.ndarray:
    """axmult.py:74-82 -> entries (int16 or uint16, 65,536)"""
    v = operand_values(mode)
    return np.multiply.outer(v, v).ravel().astype(entry_dtype(mode))


def truncated_lut(mode: str, drop_bits: int) -> np.ndarray:
    """axmult.py:85-96"""
    if not 0 <= drop_bits <= 7:
        raise ValueError(f"drop_bits must be in 0..7, got {drop_bits}")
    mask = (0xFF << drop_bits) & 0xFF
    v = operand_values(mode)
    masked = np.sign(v) * (np.abs(v) & mask)
    return np.multiply.outer(masked, masked).ravel().astype(entry_dtype(mode))


def random_lut(rng: np.random.Generator, mode: str) -> np.ndarray:
    """tests/cases.py:25-30"""
    if mode == UNSIGNED:
        return rng.integers(0, 1 << 16, 65536).astype(np.uint16)
    return rng.integers(-(1 << 15), 1 << 15, 65536).astype(np.int16)


# ---------------------------------------------------------------------------
# axconv.py restatement


def emulate_accumulator(acc: np.ndarray, accumulator: str) -> np.ndarray:
    """axconv.py:128-133"""
    if accumulator == EXACT64:
        return acc
    if accumulator == WRAP32:
        return ((acc + (1 << 31)) % (1 << 32)) - (1 << 31)
    return np.clip(acc, INT32_MIN, INT32_MAX)


def im2cols(x, scale, zp, mode, round_mode, kh, kw, padding, strides, dilations):
    """axconv.py:160-196 -> (codes rows x K, patch_sums int32)."""
    if x.size == 0:
        raise ValueError("chunk has no elements")
    n, h, w, cin = x.shape
    _, oh, ow, _ = output_shape(x.shape, (kh, kw, cin, 1), padding, strides, dilations)
    codes = quantize_values(x, scale, zp, mode, round_mode)
    pt, pb, pl, pr = resolve_padding(padding, strides, dilations, h, w, kh, kw)
    padded = np.pad(codes, ((0, 0), (pt, pb), (pl, pr), (0, 0)), constant_values=zp)
    hh = np.arange(oh)[:, None] * strides[0] + np.arange(kh)[None, :] * dilations[0]
    ww = np.arange(ow)[:, None] * strides[1] + np.arange(kw)[None, :] * dilations[1]
    win = padded[:, hh[:, None, :, None], ww[None, :, None, :], :]
    mat = np.ascontiguousarray(win.reshape(n * oh * ow, kh * kw * cin))
    sums = mat.astype(np.int64).sum(axis=1)
    if sums.size and (sums.max() > INT32_MAX or sums.min() < INT32_MIN):
        raise OverflowError("patch length too large for 32-bit code sums")
    return mat, sums.astype(np.int32)


def quantize_filters(f, scale, zp, mode, round_mode):
    """axconv.py:199-210 -> (codes K x Cout, filter_sums int32)."""
    kh, kw, cin, cout = f.shape
    codes = quantize_values(f, scale, zp, mode, round_mode).reshape(kh * kw * cin, cout)
    sums = codes.astype(np.int64).sum(axis=0)
    if sums.size and (sums.max() > INT32_MAX or sums.min() < INT32_MIN):
        raise OverflowError("filter size too large for 32-bit code sums")
    return codes, sums.astype(np.int32)


def widened_entries(entries: np.ndarray) -> np.ndarray:
    """int16 -> sign-extended / uint16 -> zero-extended int32 (numba's load)."""
    return np.ascontiguousarray(entries.astype(np.int32))


def lut_matmul(patch_codes, filt_codes, entries) -> np.ndarray:
    """Raw LUT accumulators A (int64) -- axconv.py:136-146, :236-242."""
    raw_p = np.ascontiguousarray(patch_codes).view(np.uint8)
    raw_ft = np.ascontiguousarray(filt_codes.T).view(np.uint8)
    rows, depth = raw_p.shape
    cout = raw_ft.shape[0]
    out = np.empty((rows, cout), dtype=np.int64)
    ent = widened_entries(entries)
    if rows and cout:
        lib().lut_matmul(_ptr(raw_p), _ptr(raw_ft), _ptr(ent), rows, depth, cout, _ptr(out))
    return out


def approx_gemm(patch_codes, patch_sums, filt_codes, filt_sums, s1, zp1, s2, zp2,
                entries, accumulator=EXACT64, return_acc=False):
    """axconv.py:213-257"""
    if patch_codes.shape[1] != filt_codes.shape[0]:
        raise ValueError(
            f"patch length {patch_codes.shape[1]} does not match filter rows {filt_codes.shape[0]}"
        )
    depth = patch_codes.shape[1]
    acc = emulate_accumulator(lut_matmul(patch_codes, filt_codes, entries), accumulator)
    z1 = np.int64(zp1)
    z2 = np.int64(zp2)
    corr = (
        acc
        - z2 * patch_sums.astype(np.int64)[:, None]
        - z1 * filt_sums.astype(np.int64)[None, :]
        + np.int64(depth) * z1 * z2
    )
    out = ((s1 * s2) * corr).astype(np.float32)
    return (out, acc) if return_acc else out


def axconv2d(x, f, in_range, f_range, entries, mode, padding="valid", strides=(1, 1),
             dilations=(1, 1), accumulator=EXACT64, round_mode=HALF_AWAY,
             chunk_images=64, return_acc=False):
    """axconv.py:266-297.  x NHWC float32, f HWCN float32 -> NHWC float32.

    Chunking never changes bits (integer reductions); it only bounds memory.
    """
    x = np.ascontiguousarray(x, dtype=np.float32)
    f = np.ascontiguousarray(f, dtype=np.float32)
    if x.shape[3] != f.shape[2]:
        raise ValueError(f"filter channels {f.shape[2]} do not match input channels {x.shape[3]}")
    s1, zp1 = compute_coeffs(in_range[0], in_range[1], mode, round_mode)
    s2, zp2 = compute_coeffs(f_range[0], f_range[1], mode, round_mode)
    kh, kw, cin, cout = f.shape
    n, oh, ow, _ = output_shape(x.shape, f.shape, padding, strides, dilations)
    if n == 0:
        out = np.zeros((0, oh, ow, cout), np.float32)
        return (out, np.zeros((0, oh, ow, cout), np.int64)) if return_acc else out
    fc, fs = quantize_filters(f, s2, zp2, mode, round_mode)
    outs, accs = [], []
    for start in range(0, n, chunk_images):
        stop = min(start + chunk_images, n)
        pc, ps = im2cols(x[start:stop], s1, zp1, mode, round_mode, kh, kw, padding,
                         strides, dilations)
        o, a = approx_gemm(pc, ps, fc, fs, s1, zp1, s2, zp2, entries, accumulator,
                           return_acc=True)
        outs.append(o.reshape(stop - start, oh, ow, cout))
        accs.append(a.reshape(stop - start, oh, ow, cout))
    out = np.concatenate(outs, axis=0)
    return (out, np.concatenate(accs, axis=0)) if return_acc else out


def direct_conv(x, f, in_range, f_range, entries, mode, padding="valid", strides=(1, 1),
                dilations=(1, 1), accumulator=EXACT64, round_mode=HALF_AWAY):
    """axconv.py:300-379 -- per-tap nested loops (C), same int64 corrections."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    f = np.ascontiguousarray(f, dtype=np.float32)
    if x.shape[3] != f.shape[2]:
        raise ValueError(f"filter channels {f.shape[2]} do not match input channels {x.shape[3]}")
    s1, zp1 = compute_coeffs(in_range[0], in_range[1], mode, round_mode)
    s2, zp2 = compute_coeffs(f_range[0], f_range[1], mode, round_mode)
    kh, kw, cin, cout = f.shape
    n, oh, ow, _ = output_shape(x.shape, f.shape, padding, strides, dilations)
    icodes = quantize_values(x, s1, zp1, mode, round_mode)
    fcodes = quantize_values(f, s2, zp2, mode, round_mode)
    pt, pb, pl, pr = resolve_padding(padding, strides, dilations, x.shape[1], x.shape[2], kh, kw)
    padded = np.ascontiguousarray(
        np.pad(icodes, ((0, 0), (pt, pb), (pl, pr), (0, 0)), constant_values=zp1))
    depth = kh * kw * cin
    fmat = np.ascontiguousarray(fcodes.reshape(depth, cout))
    f_sums = fmat.astype(np.int64).sum(axis=0)
    lut_sums = np.zeros((n, oh, ow, cout), np.int64)
    patch_sums = np.zeros((n, oh, ow), np.int64)
    if lut_sums.size:
        pvals = np.ascontiguousarray(padded.astype(np.int32))
        ent = widened_entries(entries)
        lib().direct_lut_sums(
            _ptr(padded.view(np.uint8)), _ptr(pvals), _ptr(fmat.view(np.uint8)), _ptr(ent),
            n, padded.shape[1], padded.shape[2], cin, kh, kw, cout, oh, ow,
            strides[0], strides[1], dilations[0], dilations[1],
            _ptr(lut_sums), _ptr(patch_sums))
    acc = emulate_accumulator(lut_sums, accumulator)
    corr = (acc - np.int64(zp2) * patch_sums[..., None] - np.int64(zp1) * f_sums
            + np.int64(depth) * np.int64(zp1) * np.int64(zp2))
    return ((s1 * s2) * corr).astype(np.float32)


def depthwise_conv(x, f, in_range, f_range, entries, mode, padding="valid", strides=(1, 1),
                   dilations=(1, 1), accumulator=EXACT64, round_mode=HALF_AWAY, return_acc=False):
    """Depthwise approximate conv (BASELINE config 5; the reference has no grouped conv, tensor.py:66-87).

    Defined as the per-channel decomposition SURVEY.md 8(d) config 5 prescribes: output channel c =
    axconv2d(x[..., c:c+1], f[:, :, c:c+1, :]) (axconv.py:266-297) with the SAME input and filter
    ranges for every channel.  f is (kh, kw, C, 1) (channel multiplier 1).
    """
    x = np.ascontiguousarray(x, dtype=np.float32)
    f = np.ascontiguousarray(f, dtype=np.float32)
    if f.ndim != 4 or f.shape[3] != 1:
        raise ValueError("depthwise filters must be (kh, kw, channels, 1)")
    if x.shape[3] != f.shape[2]:
        raise ValueError(f"filter channels {f.shape[2]} do not match input channels {x.shape[3]}")
    parts = [axconv2d(x[..., c:c + 1], f[:, :, c:c + 1, :], in_range, f_range, entries, mode, padding=padding,
                      strides=strides, dilations=dilations, accumulator=accumulator, round_mode=round_mode,
                      return_acc=return_acc) for c in range(x.shape[3])]
    if return_acc:
        return (np.concatenate([o for o, _ in parts], axis=3), np.concatenate([a for _, a in parts], axis=3))
    return np.concatenate(parts, axis=3)


def conv_filter_shape(attrs) -> tuple:
    """The dense-equivalent (kh, kw, cin, cout) of an AxConv2D node's filters: a depthwise node's
    (kh, kw, C, 1) filters act as (kh, kw, 1, C) per channel -- MACs n*oh*ow*kh*kw*C."""
    f = attrs["filters"]
    return (f.shape[0], f.shape[1], 1, f.shape[2]) if attrs.get("depthwise") else tuple(f.shape)


def conv_mac_count(in_shape, f_shape, padding, strides, dilations) -> int:
    """axconv.py:106-114"""
    n, oh, ow, cout = output_shape(in_shape, f_shape, padding, strides, dilations)
    kh, kw, cin, _ = f_shape
    return n * oh * ow * kh * kw * cin * cout


# ---------------------------------------------------------------------------
# graph.py restatement (run over a node list; the kinds the hot path touches)


def _gather_windows(x, padding, strides, kh, kw, fill):
    """graph.py:157-167 (pool geometry: dilation 1)."""
    n, h, w, c = x.shape
    pt, pb, pl, pr = resolve_padding(padding, strides, (1, 1), h, w, kh, kw)
    padded = np.pad(x, ((0, 0), (pt, pb), (pl, pr), (0, 0)), constant_values=fill)
    _, oh, ow, _ = output_shape((n, h, w, c), (kh, kw, c, 1), padding, strides, (1, 1))
    hh = np.arange(oh)[:, None] * strides[0] + np.arange(kh)[None, :]
    ww = np.arange(ow)[:, None] * strides[1] + np.arange(kw)[None, :]
    return padded[:, hh[:, None, :, None], ww[None, :, None, :], :]


def pool2d(x, attrs, take_max):
    """graph.py:182-199"""
    ph, pw = tuple(attrs.get("pool", (2, 2)))
    strides = tuple(attrs.get("strides", (ph, pw)))
    padding = attrs.get("padding", "valid")
    if isinstance(padding, list):
        padding = tuple(padding)
    if take_max:
        win = _gather_windows(x, padding, strides, ph, pw, -np.inf)
        return win.max(axis=(3, 4)).astype(np.float32)
    win = _gather_windows(x, padding, strides, ph, pw, np.nan)
    n, h, w, _ = x.shape
    ones = np.ones((1, h, w, 1), dtype=np.float32)
    counts = _gather_windows(ones, padding, strides, ph, pw, np.nan)
    valid = np.isfinite(counts).sum(axis=(3, 4))
    total = np.nansum(win, axis=(3, 4))
    return (total / valid).astype(np.float32)


def run_graph(nodes, batch, accumulator=EXACT64, round_mode=HALF_AWAY, engine="gemm",
              trace=None):
    """graph.py:202-313 for node dicts {id, kind, inputs, attrs}.

    Kinds: Input, AxConv2D, Min, Max, ReLU, MaxPool, AvgPool, Add, Flatten,
    Dense, Softmax (the reference's names).  AxConv2D attrs: filters (HWCN),
    bias (optional), lut (entries), mode, f_min, f_max, strides, dilations,
    padding, depthwise (optional: (kh, kw, C, 1) filters -> depthwise_conv, config 5).
    engine "gemm" -> axconv2d, "direct" -> direct_conv.
    """
    dense_conv = axconv2d if engine == "gemm" else direct_conv
    values = {}
    out = None
    for node in nodes:
        kind = node["kind"]
        attrs = node.get("attrs", {})
        ins = [values[i] for i in node.get("inputs", [])]
        if kind == "Input":
            out = np.asarray(batch, np.float32)
        elif kind == "AxConv2D":
            padding = attrs.get("padding", "valid")
            if isinstance(padding, list):
                padding = tuple(padding)
            conv = depthwise_conv if attrs.get("depthwise") else dense_conv
            y = conv(ins[0], attrs["filters"], (float(ins[1]), float(ins[2])),
                     (attrs["f_min"], attrs["f_max"]), attrs["lut"], attrs["mode"],
                     padding=padding, strides=tuple(attrs.get("strides", (1, 1))),
                     dilations=tuple(attrs.get("dilations", (1, 1))),
                     accumulator=accumulator, round_mode=round_mode)
            bias = attrs.get("bias")
            out = y if bias is None else (y + bias.astype(np.float32)).astype(np.float32)
        elif kind in ("Min", "Max"):
            arr = np.asarray(ins[0])
            if not np.isfinite(arr).all():
                raise ValueError(f"non-finite values reaching {node['id']!r}")
            out = float(arr.min() if kind == "Min" else arr.max())
        elif kind == "ReLU":
            out = np.maximum(ins[0], np.float32(0.0))
        elif kind == "MaxPool":
            out = pool2d(ins[0], attrs, True)
        elif kind == "AvgPool":
            out = pool2d(ins[0], attrs, False)
        elif kind == "Add":
            a, b = ins
            if a.shape != b.shape:
                raise ValueError(f"Add node {node['id']!r} input shapes differ")
            out = (a + b).astype(np.float32)
        elif kind == "Flatten":
            out = np.ascontiguousarray(ins[0]).reshape(ins[0].shape[0], -1)
        elif kind == "Dense":
            out = ins[0] @ attrs["weights"]
            if attrs.get("bias") is not None:
                out = out + attrs["bias"]
            out = out.astype(np.float32)
        elif kind == "Softmax":
            z = ins[0] - ins[0].max(axis=-1, keepdims=True)
            e = np.exp(z)
            out = (e / e.sum(axis=-1, keepdims=True)).astype(np.float32)
        else:
            raise ValueError(f"unsupported node kind {kind!r}")
        values[node["id"]] = out
    if trace is not None:
        trace.update(values)
    res = np.asarray(out, np.float32)
    if res.ndim == 2:
        res = res.reshape(res.shape[0], 1, 1, res.shape[1])
    return res


def graph_mac_count(nodes, batch_shape) -> int:
    """graph.py:316-349 (conv MACs; padding taps counted)."""
    shapes = {}
    total = 0
    for node in nodes:
        kind = node["kind"]
        attrs = node.get("attrs", {})
        if kind == "Input":
            shapes[node["id"]] = tuple(batch_shape)
        elif kind == "AxConv2D":
            x = shapes[node["inputs"][0]]
            padding = attrs.get("padding", "valid")
            if isinstance(padding, list):
                padding = tuple(padding)
            st = tuple(attrs.get("strides", (1, 1)))
            dl = tuple(attrs.get("dilations", (1, 1)))
            fs = conv_filter_shape(attrs)
            xs = (x[0], x[1], x[2], 1) if attrs.get("depthwise") else x
            total += conv_mac_count(xs, fs, padding, st, dl)
            shapes[node["id"]] = output_shape(xs, fs, padding, st, dl)
        elif kind in ("Min", "Max"):
            shapes[node["id"]] = ()
        elif kind in ("ReLU", "Softmax", "Add"):
            shapes[node["id"]] = shapes[node["inputs"][0]]
        elif kind in ("MaxPool", "AvgPool"):
            x = shapes[node["inputs"][0]]
            ph, pw = tuple(attrs.get("pool", (2, 2)))
            padding = attrs.get("padding", "valid")
            if isinstance(padding, list):
                padding = tuple(padding)
            n, oh, ow, _ = output_shape(x, (ph, pw, x[3], 1), padding,
                                        tuple(attrs.get("strides", (ph, pw))), (1, 1))
            shapes[node["id"]] = (n, oh, ow, x[3])
        elif kind == "Flatten":
            x = shapes[node["inputs"][0]]
            shapes[node["id"]] = (x[0], int(np.prod(x[1:])))
        elif kind == "Dense":
            x = shapes[node["inputs"][0]]
            shapes[node["id"]] = (x[0], attrs["weights"].shape[1])
    return total


# ---------------------------------------------------------------------------
# datasets.py restatement (synthetic CIFAR-shaped inputs)

_PATTERN_SEED = 20908  # datasets.py:17


def class_patterns() -> np.ndarray:
    """datasets.py:20-24"""
    prng = np.random.default_rng(_PATTERN_SEED)
    base = prng.uniform(0.0, 1.0, (10, 4, 4, 3))
    return np.repeat(np.repeat(base, 8, axis=1), 8, axis=2).astype(np.float32)


def synthetic_cifar10(n: int, seed: int = 0):
    """datasets.py:27-36"""
    rng = np.random.default_rng(seed)
    patterns = class_patterns()
    labels = rng.integers(0, 10, n)
    noise = rng.uniform(0.0, 1.0, (n, 32, 32, 3)).astype(np.float32)
    images = np.clip(0.7 * patterns[labels] + 0.3 * noise, 0.0, 1.0)
    images = (np.rint(images * 255.0) / 255.0).astype(np.float32)
    return images, labels.astype(np.uint8)


def cpu_count_used() -> int:
    return threads()


if __name__ == "__main__":  # pragma: no cover
    build_lib(force=True)
    print("built", LIB_PATH, "threads", threads(), "cpus", os.cpu_count(), math.pi)
