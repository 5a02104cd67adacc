"""One prepared approximate-conv layer on one device (the per-node unit of the executor).

Filters are quantized once at construction (the reference re-quantizes them
on every call, axconv.py:287; hoisting is bit-neutral because the filter
range is a constant, graph.py:129-130).  ``run`` executes, stream-ordered:

  K2 coefficients of the device input range (kernel         quantizer.py:98-117
     prologue, no sync) + quantize + zero-point pad        quantizer.py:120-131, axconv.py:181-189
  [im2col of the codes, small-channel layers only]         axconv.py:160-196
  K3 LUT implicit GEMM + fused epilogue                    axconv.py:136-146, :246-256, graph.py:268-286

Path choice (``libaxb``): channels are padded to a multiple of 16 (raw-0
codes whose exact contribution the epilogue removes); when that padding would
waste lookups (c % 16 != 0 with a multi-tap kernel, e.g. the RGB stem) the
codes are gathered into dense kp = roundup16(kh*kw*c) rows and the conv runs
as a 1x1 over them.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _lib
from .axconv import device_lut
from .types import resolve_padding


FTABLE_MAX_BYTES = 4 << 30  # per layer (ResNet-50's largest: 4608 x 512 x 512 B = 1.2 GB)
CX_LAYOUTS = {2: 64, 3: 32, 4: 16}  # axb_ft_variant_layout -> channel block of the CX table


class ConvLayer:
    def __init__(self, filters, f_range, lut, geometry, bias=None, round_mode="half-away-from-zero",
                 accumulator="exact64", device=None, depthwise=False, ftable=None):
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else int(device))
        with torch.cuda.device(self.device):  # uploads and launches on the layer's device
            self._init(filters, f_range, lut, geometry, bias, round_mode, accumulator, depthwise, ftable)

    def _init(self, filters, f_range, lut, geometry, bias, round_mode, accumulator, depthwise, ftable):
        self.lib = lib = _lib.load()
        f = np.ascontiguousarray(filters, dtype=np.float32)
        self.depthwise = bool(depthwise)
        if self.depthwise:  # (kh, kw, C, 1) -> the (kh, kw, 1, C) view: one input channel per output channel
            if f.shape[3] != 1:
                raise ValueError("depthwise filters must be (kh, kw, channels, 1)")
            f = np.ascontiguousarray(f.reshape(f.shape[0], f.shape[1], 1, f.shape[2]))
        self.kh, self.kw, self.cin, self.cout = (int(v) for v in f.shape)
        self.geometry = geometry
        self.round = _lib.ROUND[getattr(round_mode, "value", round_mode)]
        self.acc = _lib.ACC[getattr(accumulator, "value", accumulator)]
        self.lut = device_lut(lut, self.device.index)
        self.sgn = int(self.lut.signed)
        self.cs = int(lib.axb_channel_stride(self.cin))
        self.kp = 0 if self.depthwise else int(lib.axb_conv_im2col_kp(self.cin, self.kh, self.kw))
        if self.kp:  # filters as (1, 1, K, cout): same (ky, kx, ci) flattening
            fk = (1, 1, self.kh * self.kw * self.cin, self.kp)
        else:
            fk = (self.kh, self.kw, self.cin, self.cs)
        self.f_geom = fk
        self.kpad = int(lib.axb_filter_kpad(fk[0], fk[1], fk[3]))
        self.coutp = int(lib.axb_filter_coutp(self.cout))
        stream = torch.cuda.current_stream(self.device).cuda_stream
        self.params = torch.zeros(2, _lib.QPARAMS_BYTES, dtype=torch.uint8, device=self.device)  # [input, filter] axb_qparams
        hp = _lib.QParams()
        _lib.check(lib.axb_coeffs_host(float(f_range[0]), float(f_range[1]), self.sgn, self.round, hp))
        _lib.check(lib.axb_params_upload(hp, self.params[1].data_ptr(), stream))
        fd = torch.from_numpy(f).to(self.device)
        self.fcodes = torch.empty(self.kpad * self.coutp, dtype=torch.uint8, device=self.device)
        self.fsum = torch.empty(max(self.cout, 1), dtype=torch.int64, device=self.device)
        fl = torch.zeros(1, dtype=torch.int32, device=self.device)
        _lib.check(lib.axb_filters_prepare(fd.data_ptr(), fk[0], fk[1], fk[2], self.cout, fk[3],
                                           self.params[1].data_ptr(), self.sgn, self.round, self.fcodes.data_ptr(),
                                           self.fsum.data_ptr(), fl.data_ptr(), stream))
        flags = int(fl.item())
        if flags & _lib.FLAG_NONFINITE:
            raise ValueError("cannot quantize non-finite values")
        if flags & _lib.FLAG_FSUM_OVF:
            raise OverflowError("filter size too large for 32-bit code sums")
        self.bias = None if bias is None else torch.from_numpy(np.ascontiguousarray(bias, np.float32)).to(self.device)
        # filter-specialised product table (axb_ftable_prepare): 512 B per filter weight, built once
        # per layer; the conv then gathers two channels' products per 32-bit shared-memory word
        if ftable is None:
            ftable = os.environ.get("AXB_FTABLE", "1") != "0"
        nbytes = int(lib.axb_ftable_bytes(self.kpad, self.coutp))
        self.has_ft = bool(ftable and not self.depthwise and nbytes and self.kpad <= 32768 and fk[0] * fk[1] <= 256
                           and nbytes <= FTABLE_MAX_BYTES)
        # the same words code-major (cm32_* variants: 8 products per LDS.128) when channels come in 32s;
        # each layout is built on first use and ``keep_tables`` frees the one the layer's kernel does not read
        cm_bytes = int(lib.axb_ftable_cm_bytes(self.kpad, self.coutp)) if self.has_ft else 0
        self.cm_ok = bool(cm_bytes and cm_bytes <= FTABLE_MAX_BYTES and os.environ.get("AXB_FTABLE_CM", "1") != "0")
        # and the CX layouts (c64_* / c32_* / c16_* variants: bank-conflict-free LDS.128, 128-byte rows of
        # 64 / 32 / 16-channel blocks, the narrower ones replicated across the row) when channels divide
        self.cx_ok = {}
        for lay, cb in CX_LAYOUTS.items():
            nb = int(lib.axb_ftable_cx_bytes(self.kpad, self.coutp, cb)) if self.has_ft else 0
            self.cx_ok[lay] = bool(nb and nb <= FTABLE_MAX_BYTES and os.environ.get("AXB_FTABLE_CX", "1") != "0")
        self.c64_ok = self.cx_ok[2]
        self.ftable = self.ftable_cm = self.dwtable = None
        self.ftable_cx = {}
        if self.has_ft:
            self.pair_table()
        # depthwise: the channel-bank product table (axb_depthwise_table_prepare; conflict-free gathers)
        dw_bytes = int(lib.axb_depthwise_table_bytes(self.kh, self.kw, self.cout)) if self.depthwise else 0
        if dw_bytes and ftable:
            self.dwtable = torch.empty(dw_bytes // 4, dtype=torch.int32, device=self.device)
            _lib.check(lib.axb_depthwise_table_prepare(self.fcodes.data_ptr(), self.kh, self.kw, self.cout,
                                                       self.coutp, self.lut.handle, self.dwtable.data_ptr(),
                                                       torch.cuda.current_stream(self.device).cuda_stream))
        self.launches = 0

    def pair_table(self) -> torch.Tensor:
        """The pair-major product table W[sb][k][pair][a] (axb_ftable_prepare), built on first use."""
        if self.ftable is None:
            if not self.has_ft:
                raise ValueError("this layer has no filter-specialised table")
            fk = self.f_geom
            self.ftable = torch.empty(int(self.lib.axb_ftable_bytes(self.kpad, self.coutp)) // 4, dtype=torch.int32,
                                      device=self.device)
            with torch.cuda.device(self.device):
                _lib.check(self.lib.axb_ftable_prepare(self.fcodes.data_ptr(), fk[0], fk[1], fk[2], fk[3], self.cout,
                                                       self.lut.handle, self.ftable.data_ptr(),
                                                       torch.cuda.current_stream(self.device).cuda_stream))
        return self.ftable

    def cm_table(self) -> torch.Tensor:
        """The code-major product table CM[cb][k][a][pair] (axb_ftable_cm_prepare), built on first use."""
        if self.ftable_cm is None:
            if not self.cm_ok:
                raise ValueError("code-major ftable variant needs a code-major table (coutp % 32 == 0)")
            fk = self.f_geom
            self.ftable_cm = torch.empty(int(self.lib.axb_ftable_cm_bytes(self.kpad, self.coutp)) // 4,
                                         dtype=torch.int32, device=self.device)
            with torch.cuda.device(self.device):
                _lib.check(self.lib.axb_ftable_cm_prepare(self.fcodes.data_ptr(), fk[0], fk[1], fk[2], fk[3],
                                                          self.cout, self.lut.handle, self.ftable_cm.data_ptr(),
                                                          torch.cuda.current_stream(self.device).cuda_stream))
        return self.ftable_cm

    def cx_table(self, lay: int = 2) -> torch.Tensor:
        """The CX table of layout ``lay`` (2 / 3 / 4: 64 / 32 / 16-channel blocks; axb_ftable_cx_prepare),
        built on first use."""
        if lay not in self.ftable_cx:
            cb = CX_LAYOUTS[lay]
            if not self.cx_ok.get(lay):
                raise ValueError(f"c{cb} ftable variant needs a {cb}-channel code-major table (coutp % {cb} == 0)")
            fk = self.f_geom
            t = torch.empty(int(self.lib.axb_ftable_cx_bytes(self.kpad, self.coutp, cb)) // 4, dtype=torch.int32,
                            device=self.device)
            with torch.cuda.device(self.device):
                _lib.check(self.lib.axb_ftable_cx_prepare(self.fcodes.data_ptr(), fk[0], fk[1], fk[2], fk[3],
                                                          self.cout, self.lut.handle, t.data_ptr(),
                                                          torch.cuda.current_stream(self.device).cuda_stream, cb))
            self.ftable_cx[lay] = t
        return self.ftable_cx[lay]

    def c64_table(self) -> torch.Tensor:
        """The 64-channel code-major table C64[cb][k][a][pair] (layout 2), built on first use."""
        return self.cx_table(2)

    def layout_ok(self, ft_variant: int) -> bool:
        """Whether this layer can run ftable variant ``ft_variant`` (its table layout fits the channels)."""
        lay = self.lib.axb_ft_variant_layout(int(ft_variant)) if ft_variant > 0 else 0
        if ft_variant > 0 and self.kpad > self.lib.axb_ft_variant_max_k(int(ft_variant)):
            return False
        return self.has_ft and (lay == 0 or (lay == 1 and self.cm_ok) or bool(self.cx_ok.get(lay)))

    def keep_tables(self, ft_variant: int) -> None:
        """Free the product-table layouts the chosen kernel does not read (0 / pair-major variants keep
        the pair-major table, code-major variants their own layout, -1 -- the b-major LUT kernel --
        none).  A later different choice rebuilds what it needs."""
        v = int(ft_variant)
        lay = self.lib.axb_ft_variant_layout(v) if v > 0 else (0 if v == 0 else -1)
        if lay != 0:
            self.ftable = None
        if lay != 1:
            self.ftable_cm = None
        self.ftable_cx = {k: t for k, t in self.ftable_cx.items() if k == lay}

    def table_bytes(self) -> int:
        """Device bytes held by this layer's product tables."""
        return sum(t.numel() * 4 for t in (self.ftable, self.ftable_cm, self.dwtable, *self.ftable_cx.values())
                   if t is not None)

    def shares_codes_with(self, other: "ConvLayer") -> bool:
        """True when this layer can read ``other``'s code tensor of the same input instead of quantizing
        it again: a 1x1 layer without padding on the ftable kernel, same channels, signedness and rounding
        (same range -> identical codes and coefficients; quantizer.py:98-131)."""
        return (self.kh == self.kw == 1 and not self.kp and not self.depthwise and not other.kp
                and not other.depthwise and self.has_ft and self.cin == other.cin
                and self.sgn == other.sgn and self.round == other.round
                and tuple(self.geometry.dilations) == (1, 1))

    def set_input_params(self, mn: float, mx: float) -> None:
        """Host range (the operator-API path): coefficients computed on the host, uploaded."""
        hp = _lib.QParams()
        _lib.check(self.lib.axb_coeffs_host(float(mn), float(mx), self.sgn, self.round, hp))
        _lib.check(self.lib.axb_params_upload(hp, self.params[0].data_ptr(),
                                              torch.cuda.current_stream(self.device).cuda_stream))

    def run(self, x: torch.Tensor, in_range_dev=None, *, relu=False, residual=None, out_range=None,
            out_flag=None, quant_flag=None, acc_out=None, force_generic=False, sm_limit=0, variant=0,
            pixel_order=0, profile=None, ft_variant=0, use_ftable=True, codes_in=None,
            codes_out=None, qprofile=None) -> torch.Tensor:
        with torch.cuda.device(self.device):
            return self._run(x, in_range_dev, relu, residual, out_range, out_flag, quant_flag, acc_out,
                             force_generic, sm_limit, variant, pixel_order, profile, ft_variant, use_ftable,
                             codes_in, codes_out, qprofile)

    def _run(self, x, in_range_dev, relu, residual, out_range, out_flag, quant_flag, acc_out, force_generic,
             sm_limit, variant, pixel_order, profile, ft_variant, use_ftable, codes_in, codes_out,
             qprofile) -> torch.Tensor:
        """x: (n,h,w,cin) fp32 CUDA.  in_range_dev: device int32[2] ordered-float range, or None if
        set_input_params() was called.  Returns (n,oh,ow,cout) fp32.

        ``codes_out`` (a dict) receives this call's zp-padded code tensor and its quantization
        parameters; ``codes_in`` (such a dict, from another layer quantizing the SAME tensor with the
        same range, signedness and rounding) lets a 1x1 unpadded layer on the ftable kernel skip its
        own quantize pass and read the interior of that tensor (``shares_codes_with``).
        ``qprofile`` (a list) receives (kernel kind, start_event, end_event, algorithmic HBM bytes)
        around the quantize launch."""
        lib = self.lib
        n, h, w, c = (int(v) for v in x.shape)
        if c != (self.cout if self.depthwise else self.cin):
            raise ValueError(f"filter channels {self.cin} do not match input channels {c}")
        in_cs = int(lib.axb_channel_stride(c))
        g = self.geometry
        pt, pb, pl, pr = resolve_padding(g, h, w, self.kh, self.kw)
        hp_, wp_ = h + pt + pb, w + pl + pr
        ekh, ekw = (self.kh - 1) * g.dilations[0] + 1, (self.kw - 1) * g.dilations[1] + 1
        if hp_ < ekh or wp_ < ekw:
            raise ValueError(f"kernel extent {max(ekh, ekw)} exceeds padded input")
        oh, ow = (hp_ - ekh) // g.strides[0] + 1, (wp_ - ekw) // g.strides[1] + 1
        out = torch.empty((n, oh, ow, self.cout), dtype=torch.float32, device=self.device)
        if n == 0 or self.cout == 0:
            return out
        stream = torch.cuda.current_stream(self.device).cuda_stream
        self.launches = 0
        qflag = quant_flag if quant_flag is not None else out_flag
        d = _lib.ConvDesc()

        def qtimed(kind, nbytes, fn):
            if qprofile is None:
                return fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            qprofile.append((kind, e0, e1, int(nbytes)))

        if self.kp:  # small-c layer: quantize + zp-pad + im2col in one pass into kp-byte code rows
            codes = torch.empty(n * oh * ow * self.kp, dtype=torch.uint8, device=self.device)
            pixsum = torch.empty(n * oh * ow, dtype=torch.int32, device=self.device)
            qtimed("quantize_im2col", x.numel() * 4 + codes.numel() + pixsum.numel() * 4,
                   lambda: _lib.check(lib.axb_quantize_im2col(
                       x.data_ptr(), n, h, w, c, pt, pl, self.kh, self.kw, g.strides[0], g.strides[1],
                       g.dilations[0], g.dilations[1], oh, ow, self.kp, in_range_dev, self.params[0].data_ptr(),
                       self.sgn, self.round, codes.data_ptr(), pixsum.data_ptr(), qflag, stream)))
            self.launches += 1
            d.n, d.hp, d.wp, d.cs, d.c = n, oh, ow, self.kp, self.kh * self.kw * c
            d.kh = d.kw = d.sh = d.sw = d.dh = d.dw = 1
        elif codes_in is not None:  # read another layer's code tensor: interior pixel (y, x) at (y+pt, x+pl)
            if not (self.has_ft and use_ftable and not variant and not force_generic
                    and (pt, pb, pl, pr) == (0, 0, 0, 0) and self.kh == self.kw == 1 and codes_in["cs"] == in_cs
                    and codes_in["n"] == n and codes_in["h"] == h and codes_in["w"] == w):
                raise ValueError("shared code tensor does not fit this layer")
            codes, pixsum = codes_in["codes"], None
            d.n, d.hp, d.wp, d.cs, d.c = n, codes_in["hp"], codes_in["wp"], in_cs, c
            d.kh = d.kw = 1
            d.sh, d.sw = g.strides
            d.dh, d.dw = g.dilations
        else:
            codes = torch.empty(n * hp_ * wp_ * in_cs, dtype=torch.uint8, device=self.device)
            # the ftable kernel sums patch codes in its loop; only the LUT / generic kernels read pixsum
            # (the depthwise kernel sums its own per-channel patch codes)
            ft = self.has_ft and use_ftable and not variant and not force_generic
            pixsum = None if ft or self.depthwise else torch.empty(n * hp_ * wp_, dtype=torch.int32, device=self.device)
            pix_ptr = pixsum.data_ptr() if pixsum is not None else None
            qbytes = x.numel() * 4 + codes.numel() + (pixsum.numel() * 4 if pixsum is not None else 0)
            if in_range_dev is not None:  # coefficients of the device range computed inside the quantize kernel
                qtimed("quantize", qbytes, lambda: _lib.check(lib.axb_quantize_pad_range(
                    x.data_ptr(), n, h, w, c, pt, pb, pl, pr, in_cs, in_range_dev, self.sgn, self.round,
                    self.params[0].data_ptr(), codes.data_ptr(), pix_ptr, qflag, stream)))
            else:
                qtimed("quantize", qbytes, lambda: _lib.check(lib.axb_quantize_pad(
                    x.data_ptr(), n, h, w, c, pt, pb, pl, pr, in_cs, self.params[0].data_ptr(), self.sgn,
                    self.round, codes.data_ptr(), pix_ptr, qflag, stream)))
            self.launches += 1
            d.n, d.hp, d.wp, d.cs, d.c = n, hp_, wp_, in_cs, c
            d.kh, d.kw = self.kh, self.kw
            d.sh, d.sw = g.strides
            d.dh, d.dw = g.dilations
            if codes_out is not None:
                codes_out.update(codes=codes, n=n, h=h, w=w, hp=hp_, wp=wp_, pt=pt, pl=pl, cs=in_cs,
                                 params=self.params[0])
        d.codes, d.pixsum = codes.data_ptr(), (pixsum.data_ptr() if pixsum is not None else None)
        if codes_in is not None:
            d.codes += (codes_in["pt"] * codes_in["wp"] + codes_in["pl"]) * in_cs
        d.oh, d.ow = oh, ow
        d.fcodes, d.fsum = self.fcodes.data_ptr(), self.fsum.data_ptr()
        d.cout, d.coutp, d.kpad = self.cout, self.coutp, self.kpad
        d.in_params = (codes_in["params"] if codes_in is not None else self.params[0]).data_ptr()
        d.f_params = self.params[1].data_ptr()
        d.accumulator = self.acc
        d.relu = int(relu)
        d.bias = self.bias.data_ptr() if self.bias is not None else None
        if residual is not None:
            if tuple(residual.shape) != tuple(out.shape):
                raise ValueError("Add input shapes differ")
            d.residual = residual.data_ptr()
        d.out = out.data_ptr()
        d.acc_out = acc_out.data_ptr() if acc_out is not None else None
        d.out_range = out_range
        d.flags = out_flag
        d.force_generic = int(force_generic)
        d.sm_limit = int(sm_limit)
        d.variant = int(variant)
        d.pixel_order = int(pixel_order)
        table = None
        if self.depthwise and self.dwtable is not None and use_ftable:
            table = self.dwtable
        elif self.has_ft and use_ftable:
            lay = lib.axb_ft_variant_layout(int(ft_variant)) if ft_variant else 0
            table = self.cm_table() if lay == 1 else (self.cx_table(lay) if lay >= 2 else self.pair_table())
        d.ftable = table.data_ptr() if table is not None else None
        d.ft_variant = int(ft_variant)
        if profile is not None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
        launch = lib.axb_depthwise_lut if self.depthwise else lib.axb_conv2d_lut
        _lib.check(launch(d, self.lut.handle, stream))
        self.launches += 1
        if profile is not None:
            e1.record()
            # algorithmic HBM bytes of the conv launch: codes (+ per-pixel sums), filter codes or the
            # filter-specialised product table (read once), fp32 output, residual read
            ft = d.ftable is not None
            algo = d.n * d.hp * d.wp * (d.cs + (4 if d.pixsum else 0)) \
                + (table.numel() * 4 if ft else self.kpad * self.coutp) \
                + n * oh * ow * self.cout * (8 if residual is not None else 4)
            macs = n * oh * ow * self.kh * self.kw * (1 if self.depthwise else c) * self.cout
            profile.append((e0, e1, macs, algo,
                            _lib.kernel_family(_lib.last_kernel())))
        return out
