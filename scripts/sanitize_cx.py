"""Small CX / pair-major / depthwise convs for compute-sanitizer (memcheck, racecheck, synccheck):
every CX variant on a shape that exercises ragged tiles and the tail split, checked against the oracle.

    compute-sanitizer --tool racecheck python scripts/sanitize_cx.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from cases import oracle_conv  # noqa: E402
from golden_io import bits_equal  # noqa: E402
from oracle import axemu_oracle as O  # noqa: E402
from test_gpu_parity import LAYOUT_BLOCK, gpu_conv  # noqa: E402

from paper_2002_09481_b200 import _lib  # noqa: E402


def main():
    lib = _lib.load()
    rng = np.random.default_rng(7)
    x = np.maximum(rng.standard_normal((2, 9, 11, 32)), 0).astype(np.float32)
    f = rng.standard_normal((3, 3, 32, 64)).astype(np.float32)
    case = dict(x=x, f=f, lut=O.random_lut(rng, O.SIGNED), mode=O.SIGNED, padding="same", strides=(1, 1),
                dilations=(1, 1), accumulator=O.EXACT64, round_mode=O.HALF_EVEN,
                in_range=(float(x.min()), float(x.max())), f_range=(float(f.min()), float(f.max())))
    want, want_acc = oracle_conv(case, return_acc=True)
    n = 0
    for v in range(1, lib.axb_ft_variant_count()):
        if 64 % LAYOUT_BLOCK[lib.axb_ft_variant_layout(v)]:
            continue
        y, acc, kern = gpu_conv(case, ft_variant=v)
        assert bits_equal(y, want) and np.array_equal(acc, want_acc), kern
        n += 1
    print("sanitize_cx: variants checked", n, flush=True)


if __name__ == "__main__":
    main()
