"""Time every fast-kernel tile variant on the real per-layer inputs of a workload.

    python scripts/tune_variants.py --workload r8 [--out gpurun_out/tune_r8.json]

Runs the graph once with a trace to capture each conv's actual input tensor,
then re-runs every AxConv2D layer alone with each variant (CUDA events, median
of 5) and checks the outputs are bit-identical across variants.
"""

import argparse
import json
import statistics
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
    ap.add_argument("--out", default="")
    ap.add_argument("--variants", default="")
    ap.add_argument("--family", default="ft", choices=["ft", "lut", "both"],
                    help="ft: ftable-kernel variants; lut: b-major LUT kernel variants")
    ap.add_argument("--orders", default="", help="compare pixel orders (e.g. 1,4) at the heuristic variant")
    args = ap.parse_args()
    spec = workload_spec(args.workload, "trunc2")
    batch = args.batch or spec["batch"]
    imgs, _ = make_images(spec["kind"], batch, seed=1000)
    g = GpuGraph(spec["nodes"])
    trace = {}
    g.run(torch.from_numpy(imgs).cuda(), trace=trace)
    lib = _lib.load()
    runs = []  # (name, run kwargs)
    if args.family in ("lut", "both"):
        nvar = lib.axb_conv_variant_count()
        vs = [int(v) for v in args.variants.split(",")] if args.variants else list(range(1, nvar))
        runs += [(lib.axb_conv_variant_name(v).decode(), dict(variant=v, use_ftable=False)) for v in vs]
    if args.family in ("ft", "both"):
        nft = lib.axb_ft_variant_count()
        runs += [(lib.axb_ft_variant_name(v).decode(), dict(ft_variant=v)) for v in range(1, nft)]
        if args.family == "ft":
            runs.append(("lut_auto", dict(use_ftable=False)))
    rows = []
    seen = set()
    for n in spec["nodes"]:
        if n["kind"] != "AxConv2D":
            continue
        a = n["attrs"]
        x = trace[n["inputs"][0]]
        key = (tuple(x.shape), a["filters"].shape, tuple(a["strides"]))
        if key in seen:
            continue
        seen.add(key)
        layer = ConvLayer(a["filters"], (a["f_min"], a["f_max"]), a["lut"], _geometry(a), a.get("bias"))
        layer.set_input_params(float(x.min()), float(x.max()))
        flags = torch.zeros(2, dtype=torch.int32, device="cuda")
        res = {}
        ref = None
        for name, kw in runs:
            times = []
            for _ in range(6):
                prof = []
                try:
                    y = layer.run(x, None, out_flag=flags[0].data_ptr(), quant_flag=flags[1].data_ptr(),
                                  profile=prof, **kw)
                except ValueError as e:  # variant not applicable to this layer (resident-table limits)
                    if "resident" not in str(e) and "code-major" not in str(e):
                        raise
                    break
                e0, e1, macs = prof[0][:3]
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
            if not times:
                continue
            t = statistics.median(times[1:])
            if ref is None:
                ref = y
            elif not torch.equal(ref.view(torch.int32), y.view(torch.int32)):
                raise SystemExit(f"variant {name} differs on {n['id']}")
            res[name] = round(t, 4)
        if args.orders:
            for o in [int(v) for v in args.orders.split(",")]:
                if o == 4 and (y.shape[1] % 4 or y.shape[2] % 8):
                    continue
                times = []
                for _ in range(6):
                    prof = []
                    y2 = layer.run(x, None, out_flag=flags[0].data_ptr(), quant_flag=flags[1].data_ptr(), variant=0,
                                   pixel_order=o, profile=prof)
                    torch.cuda.synchronize()
                    times.append(prof[0][0].elapsed_time(prof[0][1]))
                if not torch.equal(ref.view(torch.int32), y2.view(torch.int32)):
                    raise SystemExit(f"pixel order {o} differs on {n['id']}")
                res[f"auto_order{o}"] = round(statistics.median(times[1:]), 4)
        best = min(res, key=res.get)
        sm = torch.cuda.get_device_properties(0).multi_processor_count
        peak = sm * 32 * 1.965e9
        row = {"node": n["id"], "in": list(x.shape), "filters": list(a["filters"].shape), "macs": macs,
               "best": best, "best_frac": round(macs / (res[best] / 1e3) / peak, 4), "ms": res}
        rows.append(row)
        print(json.dumps(row), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
