"""Time the quantize kernels alone (warm L2 vs flushed) on ResNet-8/50-shaped activations: zero-point padded
with per-pixel sums (pad 1) and padded without them (what 3x3 CX layers run) and unpadded without them (1x1 CX layers)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2002_09481_b200 import _lib  # noqa: E402

lib = _lib.load()
import itertools  # noqa: E402

for (pad, with_pix), (n, h, w, c) in itertools.product(((1, True), (1, False), (0, False)), [(1024, 32, 32, 16), (1024, 16, 16, 32), (1024, 8, 8, 64), (256, 56, 56, 64), (256, 28, 28, 128),
                     (256, 56, 56, 256), (256, 28, 28, 512), (256, 14, 14, 1024), (256, 7, 7, 2048)]):
    x = torch.relu(torch.randn(n, h, w, c, device="cuda"))
    cs = int(lib.axb_channel_stride(c))
    hp, wp = h + 2 * pad, w + 2 * pad
    codes = torch.empty(n * hp * wp * cs, dtype=torch.uint8, device="cuda")
    pix = torch.empty(n * hp * wp, dtype=torch.int32, device="cuda")
    rng = torch.tensor([0, torch.finfo(torch.float32).max], device="cuda")
    rng_i = torch.tensor([0, int(torch.tensor([float(x.max())]).view(torch.int32).item())], dtype=torch.int32,
                         device="cuda")
    params = torch.zeros(_lib.QPARAMS_BYTES, dtype=torch.uint8, device="cuda")
    fl = torch.zeros(1, dtype=torch.int32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def q():
        _lib.check(lib.axb_quantize_pad_range(x.data_ptr(), n, h, w, c, pad, pad, pad, pad, cs, rng_i.data_ptr(), 1, 0,
                                              params.data_ptr(), codes.data_ptr(), pix.data_ptr() if with_pix else None,
                                              fl.data_ptr(), None))
    for _ in range(3):
        q()
    res = {}
    for mode in ("warm", "cold"):
        ts = []
        for _ in range(10):
            if mode == "cold":
                flush.zero_()
            else:
                x.add_(0)  # touch the input like the producing conv would
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); q(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[mode] = sorted(ts)[5]
    byt = x.numel() * 4 + codes.numel() + (pix.numel() * 4 if with_pix else 0)
    print(f"pad {pad} pixsum {int(with_pix)} {(n, h, w, c)}: {byt / 1e6:.1f} MB  warm {res['warm'] * 1e3:.1f} us ({byt / res['warm'] / 1e9:.2f} TB/s)"
          f"  cold {res['cold'] * 1e3:.1f} us ({byt / res['cold'] / 1e9:.2f} TB/s)")
