"""Run one conv layer of a workload on its real (traced) input with a chosen ftable variant, a few
times -- a target for ncu (e.g. ncu -k regex:lutconv_ftcm -s 1 -c 1 python scripts/ft_one.py ...).

    python scripts/ft_one.py --workload r8 --node s2b0.b --variant cm32_j4_w16_k4 [--reps 3]
"""

import argparse
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from bench import make_images, workload_spec  # noqa: E402
from paper_2002_09481_b200 import _lib  # noqa: E402
from paper_2002_09481_b200.graph import GpuGraph, _geometry  # noqa: E402
from paper_2002_09481_b200.layer import ConvLayer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="r8")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--node", required=True)
    ap.add_argument("--variant", required=True)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--residual", action="store_true", help="fuse a residual add (an fp32 tensor of the output's shape)")
    args = ap.parse_args()
    spec = workload_spec(args.workload, "trunc2")
    imgs, _ = make_images(spec["kind"], args.batch or spec["batch"], seed=1000)
    g = GpuGraph(spec["nodes"])
    trace = {}
    g.run(torch.from_numpy(imgs).cuda(), trace=trace)
    lib = _lib.load()
    names = {lib.axb_ft_variant_name(v).decode(): v for v in range(1, lib.axb_ft_variant_count())}
    n = next(n for n in spec["nodes"] if n["id"] == args.node)
    a = n["attrs"]
    x = trace[n["inputs"][0]]
    layer = ConvLayer(a["filters"], (a["f_min"], a["f_max"]), a["lut"], _geometry(a), a.get("bias"))
    layer.set_input_params(float(x.min()), float(x.max()))
    flags = torch.zeros(2, dtype=torch.int32, device="cuda")
    res = None
    if args.residual:
        y0 = layer.run(x, None, out_flag=flags[0].data_ptr(), quant_flag=flags[1].data_ptr(),
                       ft_variant=names[args.variant])
        res = torch.randn_like(y0)
    for _ in range(args.reps):
        prof = []
        layer.run(x, None, residual=res, out_flag=flags[0].data_ptr(), quant_flag=flags[1].data_ptr(), profile=prof,
                  ft_variant=names[args.variant])
        torch.cuda.synchronize()
        print(args.variant, round(prof[0][0].elapsed_time(prof[0][1]), 4), "ms")


if __name__ == "__main__":
    main()
