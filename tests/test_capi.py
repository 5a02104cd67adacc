"""CPU-only checks of the C ABI boundary: the library loads, exports every
symbol include/axb.h declares, and its host-side functions (no GPU needed)
agree with the oracle / reference fixtures."""

import re
from pathlib import Path

import numpy as np
import pytest

from golden_io import load_golden
from oracle import axemu_oracle as O

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "axb.h"


def header_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    names = set(re.findall(r"\b(axb_[a-z0-9_]+)\s*\(", text))
    return sorted(names)


def test_library_exports_every_header_symbol():
    from paper_2002_09481_b200 import _lib

    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    # and the ctypes binding declares exactly these
    assert set(_lib.SIGNATURES) == set(names)


def test_lib_exports_are_c_abi(tmp_path):
    """nm: the exported axb_* symbols are unmangled C symbols."""
    import subprocess

    from paper_2002_09481_b200 import _lib

    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (axb_[a-z0-9_]+)\b", out))
    assert set(header_functions()) <= exported


def test_conv_desc_layout_matches_header():
    """ctypes ConvDesc mirrors axb_conv_desc field-for-field (names and order)."""
    from paper_2002_09481_b200 import _lib

    text = HEADER.read_text()
    body = text[text.index("typedef struct axb_conv_desc"):text.index("} axb_conv_desc;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = []
    for decl in body.split(";")[:-1]:
        decl = decl.replace("typedef struct axb_conv_desc {", "")
        for part in decl.split(","):
            nm = re.findall(r"\**\s*([a-z_0-9]+)\s*$", part.strip())
            if nm:
                fields.append(nm[0])
    assert [f for f, _ in _lib.ConvDesc._fields_] == fields


def test_host_coefficients_match_reference_fixtures():
    from paper_2002_09481_b200 import _lib

    lib = _lib.load()
    g = load_golden("kat")
    for i in range(int(g["q_count"])):
        mn, mx = g[f"q{i}_range"]
        sgn, rm = (int(v) for v in g[f"q{i}_mode"])
        p = _lib.QParams()
        _lib.check(lib.axb_coeffs_host(float(mn), float(mx), sgn, rm, p))
        assert (p.scale, p.zero_point) == (g[f"q{i}_coeffs"][0], int(g[f"q{i}_coeffs"][1])), i


@pytest.mark.parametrize("seed", range(3))
def test_host_coefficients_random_ranges(seed):
    from paper_2002_09481_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(seed)
    rounds = [O.HALF_AWAY, O.HALF_EVEN, O.TOWARD_ZERO]
    for _ in range(400):
        lo = float(rng.uniform(-1e4, 1e4)) * 10.0 ** int(rng.integers(-30, 5))
        hi = lo + abs(float(rng.standard_normal())) * 10.0 ** int(rng.integers(-30, 5))
        for sgn in (0, 1):
            for rm in range(3):
                p = _lib.QParams()
                _lib.check(lib.axb_coeffs_host(lo, hi, sgn, rm, p))
                want = O.compute_coeffs(lo, hi, O.SIGNED if sgn else O.UNSIGNED, rounds[rm])
                assert (p.scale, p.zero_point) == want


def test_host_coefficients_reject_bad_ranges():
    from paper_2002_09481_b200 import _lib

    lib = _lib.load()
    p = _lib.QParams()
    with pytest.raises(ValueError, match="finite"):
        _lib.check(lib.axb_coeffs_host(float("nan"), 1.0, 0, 0, p))
    with pytest.raises(ValueError, match="exceeds"):
        _lib.check(lib.axb_coeffs_host(2.0, 1.0, 0, 0, p))


def test_layout_helpers():
    from paper_2002_09481_b200 import _lib

    lib = _lib.load()
    assert [lib.axb_channel_stride(c) for c in (1, 3, 16, 17, 64)] == [16, 16, 16, 32, 64]
    assert lib.axb_filter_kpad(3, 3, 16) == 144 and lib.axb_filter_kpad(1, 1, 3) == 16
    assert lib.axb_filter_coutp(10) == 16 and lib.axb_filter_coutp(1000) == 1008
    assert lib.axb_conv_im2col_kp(3, 7, 7) == 160 and lib.axb_conv_im2col_kp(3, 3, 3) == 32
    assert lib.axb_conv_im2col_kp(64, 3, 3) == 0 and lib.axb_conv_im2col_kp(3, 1, 1) == 0
    assert lib.axb_conv_variant_count() >= 2
    assert lib.axb_conv_variant_name(0) == b"auto"


def test_product_fails_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2002_09481_b200 import _lib, axconv2d
    from paper_2002_09481_b200 import types as T

    with pytest.raises(_lib.AxbError):
        axconv2d(T.Tensor4(np.zeros((1, 4, 4, 1), np.float32)), T.Tensor4(np.ones((2, 2, 1, 1), np.float32),
                 T.Layout.HWCN), T.Range(0, 1), T.Range(0, 1), T.exact_lut(T.Signedness.UNSIGNED))
    from paper_2002_09481_b200.graph import GpuGraph

    with pytest.raises(_lib.AxbError):
        GpuGraph([{"id": "in", "kind": "Input", "inputs": [], "attrs": {}}])


def test_missing_library_raises(tmp_path):
    from paper_2002_09481_b200 import _lib

    with pytest.raises(_lib.AxbError, match="no CPU fallback"):
        _lib.load(tmp_path / "nope.so")


def _codes_from_bounds(p, vals, signed):
    b = np.array(p.bound, np.float32)
    lo = -128 if signed else 0
    # lo + max{u : bound[u] <= x}
    return (lo + np.searchsorted(b, vals.astype(np.float32), side="right") - 1).astype(np.int64)


@pytest.mark.parametrize("seed", range(4))
def test_exact_code_boundary_tables(seed):
    """The boundary table reproduces the reference quantizer bit-for-bit (host build of the device code)."""
    from paper_2002_09481_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(seed)
    rounds = [O.HALF_AWAY, O.HALF_EVEN, O.TOWARD_ZERO]
    ranges = [(-2.3, 5.9), (0.0, 1.0), (0.0, 0.0), (-1e6, 1e6), (0.0, 1e-9), (-9.0, -1.0), (-1e-3, 1e5),
              (0.0, 5e-324), (-3e38, 3e38), (1e-40, 1e-39)]
    for _ in range(6):
        lo = float(rng.uniform(-50, 5)) * 10.0 ** int(rng.integers(-8, 4))
        ranges.append((lo, lo + abs(float(rng.standard_normal())) * 10.0 ** int(rng.integers(-8, 4))))
    for mn, mx in ranges:
        for sgn in (0, 1):
            for rm in range(3):
                p = _lib.QParams()
                _lib.check(lib.axb_coeffs_host(mn, mx, sgn, rm, p))
                mode = O.SIGNED if sgn else O.UNSIGNED
                span = max(abs(mn), abs(mx), 1e-30)
                vals = np.concatenate([
                    rng.uniform(-1.2 * span, 1.2 * span, 3000),
                    (np.arange(-300, 300) + 0.5) * p.scale, (np.arange(-300, 300)) * p.scale,
                    np.nextafter(np.float32((np.arange(-300, 300) + 0.5) * p.scale), np.float32(np.inf)),
                    np.nextafter(np.float32((np.arange(-300, 300) + 0.5) * p.scale), np.float32(-np.inf)),
                    np.array([0.0, -0.0, 1e-45, -1e-45, 3.4e38, -3.4e38]),
                ]).astype(np.float32)
                vals = vals[np.isfinite(vals)]
                b = np.array(p.bound, np.float32)
                assert b[0] == -np.inf and np.all(np.diff(b) >= 0)
                want = O.quantize_values(vals, p.scale, p.zero_point, mode, rounds[rm]).astype(np.int64)
                got = _codes_from_bounds(p, vals, sgn)
                assert np.array_equal(got, want), (mn, mx, sgn, rm)
