"""Time every ftable-kernel variant (and the b-major LUT kernel) on chosen layers of a workload, on
each layer's real traced input: the autotune's candidate matrix, printed as JSON lines.

    python scripts/variant_matrix.py --workload r50 --nodes s0b1.b,s2b1.b [--batch 256] [--reps 3]
"""

import argparse
import json
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
    ap.add_argument("--workload", default="r50")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--nodes", default="")
    ap.add_argument("--variants", default="")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    spec = workload_spec(args.workload, "trunc2")
    imgs, _ = make_images(spec["kind"], args.batch or spec["batch"], seed=1000)
    g = GpuGraph(spec["nodes"])
    trace = {}
    g.run(torch.from_numpy(imgs).cuda(), trace=trace)
    lib = _lib.load()
    names = {lib.axb_ft_variant_name(v).decode(): v for v in range(1, lib.axb_ft_variant_count())}
    if args.variants:
        names = {k: v for k, v in names.items() if k in args.variants.split(",")}
    want = args.nodes.split(",") if args.nodes else [n["id"] for n in spec["nodes"] if n["kind"] == "AxConv2D"]
    for nid in want:
        n = next(n for n in spec["nodes"] if n["id"] == nid)
        a = n["attrs"]
        x = trace[n["inputs"][0]]
        layer = ConvLayer(a["filters"], (a["f_min"], a["f_max"]), a["lut"], _geometry(a), a.get("bias"),
                          depthwise=bool(a.get("depthwise")))
        layer.set_input_params(float(x.min()), float(x.max()))
        flags = torch.zeros(2, dtype=torch.int32, device="cuda")
        row = {"node": nid, "shape": list(x.shape), "filters": list(a["filters"].shape)}
        ref = None
        cands = [("depthwise_ct", 0)] if layer.depthwise else list(names.items())
        for nm, v in cands + [("lut_bmajor", -1)]:
            if v > 0 and not layer.layout_ok(v):
                continue
            ts = []
            for _ in range(args.reps + 1):
                prof = []
                y = layer.run(x, None, out_flag=flags[0].data_ptr(), quant_flag=flags[1].data_ptr(), profile=prof,
                              ft_variant=max(v, 0), use_ftable=v >= 0)
                torch.cuda.synchronize()
                ts.append(prof[0][0].elapsed_time(prof[0][1]))
            if ref is None:
                ref = y.clone()
            assert torch.equal(ref.view(torch.int32), y.view(torch.int32)), (nid, nm)
            macs = prof[0][2]
            t = sorted(ts[1:])[len(ts[1:]) // 2]
            row[nm] = round(t, 4)
            row[nm + "_gmacs"] = round(macs / (t / 1e3) / 1e9, 1)
        layer.keep_tables(-1)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
