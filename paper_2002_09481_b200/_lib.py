"""ctypes binding of the C ABI in include/axb.h (libaxb.so, built in-tree).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is present, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libaxb.so"

AXB_OK = 0
AXB_E_VALUE = 1
AXB_E_OVERFLOW = 2
AXB_E_CUDA = 3

FLAG_NONFINITE = 1
FLAG_PSUM_OVF = 2
FLAG_OUT_NONFINITE = 4
FLAG_FSUM_OVF = 8
FLAG_LABEL = 16

UNSIGNED = 0
SIGNED = 1
ROUND = {"half-away-from-zero": 0, "half-to-even": 1, "toward-zero": 2}
ACC = {"exact64": 0, "wrap32": 1, "saturate32": 2}

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p


class QParams(ctypes.Structure):
    _fields_ = [("scale", c_dbl), ("zero_point", c_i32), ("valid", c_i32), ("bound", ctypes.c_float * 256)]

QPARAMS_BYTES = 16 + 4 * 256


class ConvDesc(ctypes.Structure):
    """Mirror of axb_conv_desc (include/axb.h)."""

    _fields_ = [
        ("codes", c_vp), ("pixsum", c_vp),
        ("n", c_i64), ("hp", c_i64), ("wp", c_i64), ("cs", c_i64), ("c", c_i64),
        ("kh", c_i32), ("kw", c_i32), ("sh", c_i32), ("sw", c_i32), ("dh", c_i32), ("dw", c_i32),
        ("oh", c_i64), ("ow", c_i64),
        ("fcodes", c_vp), ("fsum", c_vp),
        ("cout", c_i64), ("coutp", c_i64), ("kpad", c_i64),
        ("in_params", c_vp), ("f_params", c_vp),
        ("accumulator", c_i32), ("relu", c_i32),
        ("bias", c_vp), ("residual", c_vp), ("out", c_vp), ("acc_out", c_vp),
        ("out_range", c_vp), ("flags", c_vp),
        ("force_generic", c_i32), ("sm_limit", c_i32), ("variant", c_i32), ("pixel_order", c_i32),
        ("ftable", c_vp), ("ft_variant", c_i32), ("reserved0", c_i32),
    ]


# name -> (restype, argtypes); every symbol include/axb.h declares
SIGNATURES = {
    "axb_last_error": (ctypes.c_char_p, []),
    "axb_last_kernel": (ctypes.c_char_p, []),
    "axb_version": (c_int, []),
    "axb_device_info": (c_int, [c_int, c_vp, c_vp, c_vp, c_vp]),
    "axb_lut_create": (c_int, [c_vp, c_int, ctypes.POINTER(c_vp)]),
    "axb_lut_destroy": (c_int, [c_vp]),
    "axb_lut_is_signed": (c_int, [c_vp]),
    "axb_lut_device_bmajor": (c_vp, [c_vp]),
    "axb_range_reset": (c_int, [c_vp, c_vp]),
    "axb_range_minmax": (c_int, [c_vp, c_i64, c_vp, c_vp, c_vp]),
    "axb_range_read": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "axb_coeffs_host": (c_int, [c_dbl, c_dbl, c_int, c_int, ctypes.POINTER(QParams)]),
    "axb_coeffs_from_range": (c_int, [c_vp, c_int, c_int, c_vp, c_vp]),
    "axb_params_upload": (c_int, [ctypes.POINTER(QParams), c_vp, c_vp]),
    "axb_channel_stride": (c_i64, [c_i64]),
    "axb_quantize_pad": (c_int, [c_vp, c_i64, c_i64, c_i64, c_i64, c_i32, c_i32, c_i32, c_i32, c_i64,
                                 c_vp, c_int, c_int, c_vp, c_vp, c_vp, c_vp]),
    "axb_quantize_pad_range": (c_int, [c_vp, c_i64, c_i64, c_i64, c_i64, c_i32, c_i32, c_i32, c_i32, c_i64,
                                       c_vp, c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "axb_filter_kpad": (c_i64, [c_i64, c_i64, c_i64]),
    "axb_filter_coutp": (c_i64, [c_i64]),
    "axb_filters_prepare": (c_int, [c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_int, c_int, c_vp,
                                    c_vp, c_vp, c_vp]),
    "axb_conv2d_lut": (c_int, [ctypes.POINTER(ConvDesc), c_vp, c_vp]),
    "axb_conv_variant_count": (c_int, []),
    "axb_ftable_bytes": (c_i64, [c_i64, c_i64]),
    "axb_ftable_prepare": (c_int, [c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "axb_ft_variant_count": (c_int, []),
    "axb_ft_variant_clusters": (c_int, [c_int, c_int]),
    "axb_ft_variant_name": (ctypes.c_char_p, [c_int]),
    "axb_ftable_cm_bytes": (c_i64, [c_i64, c_i64]),
    "axb_ftable_cm_prepare": (c_int, [c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "axb_ftable_c64_bytes": (c_i64, [c_i64, c_i64]),
    "axb_ftable_c64_prepare": (c_int, [c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "axb_ftable_cx_bytes": (c_i64, [c_i64, c_i64, c_int]),
    "axb_ft_variant_max_k": (c_i64, [c_int]),
    "axb_ftable_cx_prepare": (c_int, [c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_int]),
    "axb_ft_variant_layout": (c_int, [c_int]),
    "axb_depthwise_lut": (c_int, [ctypes.POINTER(ConvDesc), c_vp, c_vp]),
    "axb_depthwise_table_bytes": (c_i64, [c_i64, c_i64, c_i64]),
    "axb_depthwise_table_prepare": (c_int, [c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "axb_conv_variant_name": (ctypes.c_char_p, [c_int]),
    "axb_conv_im2col_kp": (c_i64, [c_i64, c_i64, c_i64]),
    "axb_im2col_pack": (c_int, [c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32,
                                c_i64, c_i64, c_i64, c_int, c_vp, c_vp, c_vp]),
    "axb_quantize_im2col": (c_int, [c_vp, c_i64, c_i64, c_i64, c_i64, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32,
                                    c_i32, c_i32, c_i64, c_i64, c_i64, c_vp, c_vp, c_int, c_int, c_vp, c_vp, c_vp,
                                    c_vp]),
    "axb_axconv2d": (c_int, [c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_i64, c_i64, c_i64, c_i32, c_i32,
                             c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_dbl, c_dbl, c_dbl, c_dbl, c_i32,
                             c_i32, c_vp, c_vp, c_vp, c_vp]),
    "axb_maxpool": (c_int, [c_vp, c_i64, c_i64, c_i64, c_i64, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32,
                            c_i64, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "axb_avgpool": (c_int, [c_vp, c_i64, c_i64, c_i64, c_i64, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32,
                            c_i64, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "axb_add_relu": (c_int, [c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "axb_cifar_decode": (c_int, [c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
}

_lib = None


class AxbError(RuntimeError):
    pass


def load(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """Load libaxb.so (no compute, works without a GPU).  Raises if absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    # AXB_LIB_PATH: load an alternative in-tree build (A/B kernel experiments)
    p = Path(path) if path else Path(os.environ.get("AXB_LIB_PATH", LIB_PATH))
    if not p.exists():
        raise AxbError(
            f"{p} is missing: the CUDA extension is not built "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`); there is no CPU fallback"
        )
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def check(rc: int) -> None:
    """Map an AXB_E_* status to the reference's exception types."""
    if rc == AXB_OK:
        return
    msg = (load().axb_last_error() or b"").decode(errors="replace")
    if rc == AXB_E_VALUE:
        raise ValueError(msg)
    if rc == AXB_E_OVERFLOW:
        raise OverflowError(msg)
    raise AxbError(msg)


def last_kernel() -> str:
    return (load().axb_last_kernel() or b"").decode()


def kernel_family(variant_name: str) -> str:
    """Kernel behind a variant name reported by axb_last_kernel()."""
    if variant_name.startswith("ft"):
        return "lutconv_ft"
    if variant_name.startswith("cm"):
        return "lutconv_ftcm"
    if variant_name.startswith(("c64", "c32", "c16")):
        return "lutconv_cx"
    if variant_name.startswith("lutconv_"):
        return variant_name
    if variant_name.startswith("depthwise"):
        return variant_name
    return "lutconv_fast"
