import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np
from cases import random_conv_case, oracle_conv
from golden_io import bits_equal, load_golden
from test_gpu_parity import gpu_conv
from paper_2002_09481_b200 import _lib
g = load_golden("c1")
rng = np.random.default_rng(2026)
nft = _lib.load().axb_ft_variant_count()
bad = 0
for i in range(100):
    case = random_conv_case(rng)
    res = []
    for v in range(0, nft):
        y, acc, kern = gpu_conv(case, ft_variant=v)
        ok = bits_equal(y, g[f"out_{i}"]) and np.array_equal(acc, g[f"acc_{i}"])
        res.append((v, kern, ok))
    if not all(r[2] for r in res):
        bad += 1
        if bad < 6:
            print(i, case["x"].shape, case["f"].shape, case["mode"], case["strides"], case["dilations"], case["padding"], case["accumulator"])
            print("   ", [(k, ok) for v, k, ok in res])
            y, acc, kern = gpu_conv(case, ft_variant=5)
            d = acc != g[f"acc_{i}"]
            print("   diff count", d.sum(), "of", d.size, "where", np.argwhere(d)[:5].tolist(), acc[d][:5], g[f"acc_{i}"][d][:5])
print("bad cases", bad)
