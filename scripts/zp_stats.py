"""Zero-point code statistics of every conv input of a workload (GPU trace of the real graph).

For each AxConv2D: the fraction of (pixel, row) taps whose activation code is the zero-point code (ReLU
zeros, values within half a step of 0, and the zp padding), and the shared-memory wavefronts a c64
warp instruction (4 consecutive output pixels, one 128-byte table row each) would need if quarters
reading the same row merged / if zero-point quarters were skipped.

    python scripts/zp_stats.py --workload r50 --images 4 [--out gpurun_out/zp_r50.json]
"""

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from bench import make_images, workload_spec  # noqa: E402
from oracle import axemu_oracle as O  # noqa: E402
from paper_2002_09481_b200.graph import GpuGraph, _geometry  # noqa: E402
from paper_2002_09481_b200.types import output_shape, resolve_padding  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="r50")
    ap.add_argument("--images", type=int, default=4)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    spec = workload_spec(args.workload, "trunc2")
    imgs, _ = make_images(spec["kind"], spec["batch"], seed=1000)
    g = GpuGraph(spec["nodes"])
    trace = {}
    g.run(torch.from_numpy(imgs).cuda(), trace=trace)
    rows = []
    for n in spec["nodes"]:
        if n["kind"] != "AxConv2D" or n["attrs"].get("depthwise"):
            continue
        a = n["attrs"]
        xfull = trace[n["inputs"][0]]
        s, zp = O.compute_coeffs(float(xfull.min()), float(xfull.max()), a["lut"].mode.value)
        x = xfull[: args.images].double()
        q = torch.clamp(torch.round(x / s) + zp, -128 if a["lut"].mode.value == "signed" else 0,
                        127 if a["lut"].mode.value == "signed" else 255).to(torch.int16)
        kh, kw = a["filters"].shape[:2]
        geo = _geometry(a)
        sh, sw = geo.strides
        nb, h, w, c = q.shape
        pt, pb, pl, pr = resolve_padding(geo, h, w, kh, kw)
        _, oh, ow, _ = output_shape(q.shape, a["filters"].shape, geo)
        ph, pw = pt + pb, pl + pr
        qp = torch.full((nb, h + ph, w + pw, c), zp, dtype=torch.int16, device=q.device)
        qp[:, pt:pt + h, pl:pl + w] = q
        taps = []
        for ky in range(kh):
            for kx in range(kw):
                taps.append(qp[:, ky:ky + (oh - 1) * sh + 1:sh, kx:kx + (ow - 1) * sw + 1:sw, :])
        m = torch.stack(taps, 3).reshape(nb * oh * ow, kh * kw * c)  # (M, K) codes, row-major pixels
        M = (m.shape[0] // 4) * 4
        if M == 0:
            continue
        grp = m[:M].reshape(M // 4, 4, -1)
        iszp = grp == zp
        srt = torch.sort(grp, dim=1).values
        distinct = 1 + (srt[:, 1:] != srt[:, :-1]).sum(1)
        nz_quarters = (~iszp).sum(1)
        any_zp = iszp.any(1)
        distinct_nz = distinct - any_zp.to(distinct.dtype)
        rows.append({"node": n["id"], "k": int(m.shape[1]), "zp_frac": round(float(iszp.float().mean()), 4),
                     "wf_merge": round(float(distinct.float().mean()), 3),
                     "wf_skip": round(float(nz_quarters.float().mean()), 3),
                     "wf_skip_merge": round(float(distinct_nz.float().mean()), 3)})
        print(json.dumps(rows[-1]), flush=True)
    if args.out:
        json.dump(rows, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
