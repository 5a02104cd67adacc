"""Host-side API mirror: same validation, geometry and table builders as the reference."""

import numpy as np
import pytest

from oracle import axemu_oracle as O
from paper_2002_09481_b200 import types as T


def test_geometry_same_valid_explicit_match_oracle():
    rng = np.random.default_rng(3)
    for _ in range(300):
        h, w = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        kh, kw = int(rng.integers(1, 8)), int(rng.integers(1, 8))
        s = (int(rng.integers(1, 4)), int(rng.integers(1, 4)))
        d = (int(rng.integers(1, 3)), int(rng.integers(1, 3)))
        pad = ["valid", "same", tuple(int(v) for v in rng.integers(0, 3, 4))][int(rng.integers(0, 3))]
        g = T.ConvGeometry(s, d, pad)
        assert T.resolve_padding(g, h, w, kh, kw) == O.resolve_padding(pad, s, d, h, w, kh, kw)
        try:
            want = O.output_shape((2, h, w, 3), (kh, kw, 3, 5), pad, s, d)
        except ValueError:
            with pytest.raises(ValueError, match="kernel extent"):
                T.output_shape((2, h, w, 3), (kh, kw, 3, 5), g)
            continue
        assert T.output_shape((2, h, w, 3), (kh, kw, 3, 5), g) == want


def test_same_padding_puts_odd_cell_bottom_right():
    assert T.resolve_padding(T.ConvGeometry(padding="same"), 3, 3, 2, 2) == (0, 1, 0, 1)


def test_validation_errors():
    with pytest.raises(ValueError):
        T.Range(float("nan"), 1.0)
    with pytest.raises(ValueError):
        T.Range(2.0, 1.0)
    with pytest.raises(ValueError):
        T.ConvGeometry(strides=(0, 1))
    with pytest.raises(ValueError):
        T.ConvGeometry(padding="full")
    with pytest.raises(ValueError):
        T.ConvConfig(chunk_size=0)
    with pytest.raises(ValueError):
        T.MultLut(T.Signedness.SIGNED, np.zeros(65536, np.uint16))
    with pytest.raises(ValueError):
        T.MultLut(T.Signedness.SIGNED, np.zeros(100, np.int16))
    with pytest.raises(ValueError):
        T.QuantParams(0.0, 0, T.Signedness.UNSIGNED)
    with pytest.raises(ValueError):
        T.QuantParams(1.0, 200, T.Signedness.SIGNED)
    with pytest.raises(ValueError):
        T.Tensor4(np.zeros((2, 2)))


@pytest.mark.parametrize("mode", ["signed", "unsigned"])
def test_table_builders_match_oracle(mode):
    m = T.Signedness(mode)
    assert np.array_equal(T.exact_lut(m).entries, O.exact_lut(mode))
    for d in range(8):
        assert np.array_equal(T.truncated_lut(m, d).entries, O.truncated_lut(mode, d))
    with pytest.raises(ValueError):
        T.truncated_lut(m, 8)
    assert T.stitch_index(-1, 2) == 0xFF02


def test_compute_coeffs_kats():
    p = T.compute_coeffs(T.Range(0.0, 2.55), T.Signedness.UNSIGNED)
    assert p.scale == 2.55 / 255 and p.zero_point == 0
    p = T.compute_coeffs(T.Range(0.0, 0.0), T.Signedness.SIGNED)
    assert p.scale == 1.0 and p.zero_point == -128
    p = T.compute_coeffs(T.Range(2.0, 4.0), T.Signedness.UNSIGNED)
    assert p.scale == 4.0 / 255 and p.zero_point == 0
    p = T.compute_coeffs(T.Range(-9.0, -1.0), T.Signedness.UNSIGNED)
    assert p.zero_point == 255


def test_mac_count():
    g = T.ConvGeometry(padding="same")
    assert T.conv_mac_count((2, 32, 32, 3), (3, 3, 3, 16), g) == 2 * 32 * 32 * 27 * 16


def test_synthetic_inputs_match_reference_generator():
    from paper_2002_09481_b200 import datasets

    a, la = datasets.synthetic_cifar10(64, seed=4)
    b, lb = O.synthetic_cifar10(64, seed=4)
    assert np.array_equal(a, b) and np.array_equal(la, lb)
