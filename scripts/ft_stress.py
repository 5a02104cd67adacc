"""Stress the ftable kernel variants for nondeterminism: same layer, repeated runs, bitwise compare."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2002_09481_b200 import _lib  # noqa: E402
from paper_2002_09481_b200 import types as T  # noqa: E402
from paper_2002_09481_b200.layer import ConvLayer  # noqa: E402

lib = _lib.load()
rng = np.random.default_rng(0)
shapes = [((256, 56, 56, 64), (1, 1, 64, 256), True), ((64, 56, 56, 64), (3, 3, 64, 64), False),
          ((256, 14, 14, 256), (1, 1, 256, 1024), True)]
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
for xs, fs, use_res in shapes:
    x = torch.relu(torch.randn(xs, device="cuda"))
    f = (rng.standard_normal(fs) * 0.05).astype(np.float32)
    lay = ConvLayer(f, (float(f.min()), float(f.max())), T.truncated_lut(T.Signedness.SIGNED, 2),
                    T.ConvGeometry(padding="same"), bias=(rng.standard_normal(fs[3]) * 0.05).astype(np.float32))
    lay.set_input_params(0.0, float(x.max()))
    oshape = xs[:3] + (fs[3],)
    res = torch.randn(oshape, device="cuda") if use_res else None
    flags = torch.zeros(2, dtype=torch.int32, device="cuda")
    ref = lay.run(x, None, residual=res, relu=True, out_flag=flags[0].data_ptr(), quant_flag=flags[1].data_ptr(),
                  variant=1, use_ftable=False).clone()
    for v in range(1, lib.axb_ft_variant_count()):
        bad = 0
        for r in range(reps):
            y = lay.run(x, None, residual=res, relu=True, out_flag=flags[0].data_ptr(),
                        quant_flag=flags[1].data_ptr(), ft_variant=v)
            torch.cuda.synchronize()
            if not torch.equal(y.view(torch.int32), ref.view(torch.int32)):
                bad += 1
                d = (y.view(torch.int32) != ref.view(torch.int32))
                idx = d.nonzero()[:3].tolist()
                if bad == 1:
                    print(f"  v{v} rep{r}: {int(d.sum())} differing outputs, first {idx}", flush=True)
        print(xs, fs, lib.axb_ft_variant_name(v).decode(), f"mismatching runs {bad}/{reps}", flush=True)
