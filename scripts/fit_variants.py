"""Fit the conv-variant cost model from tune_variants.py outputs and patch the table.

    python scripts/fit_variants.py gpurun_out/tune_r8.json gpurun_out/tune_r50.json [--write]

Model (pick_variant in csrc/axb_conv.cu): time ~ cost_v * waves * BM * BN * NGRP,
waves = ceil(tiles / (SMs * NGRP)).  cost_v = median over layers of the variant's
time / (waves*BM*BN*NGRP), normalised by each layer's best variant.  Prints the
fitted costs and the regret of the model's pick against the measured best.
"""

import collections
import json
import math
import re
import statistics
import sys
from pathlib import Path

CU = Path(__file__).resolve().parent.parent / "paper_2002_09481_b200" / "csrc" / "axb_conv.cu"
SMS = 148


def parse(name):
    m = re.match(r"(g(\d)_)?tm(\d)tn(\d+)_w(\d+)x(\d+)", name)
    return int(m.group(3)), int(m.group(4)), int(m.group(5)), int(m.group(6)), int(m.group(2) or 1)


def geom(r):
    n, h, w, c = r["in"]
    kh, kw, ci, co = r["filters"]
    m = n * (r["macs"] // (n * kh * kw * ci * co))
    return m, (co + 15) // 16 * 16


def base(name, m, coutp):
    tm, tn, wm, wn, ng = parse(name)
    bm, bn = wm * 32 * tm, wn * tn
    tiles = math.ceil(m / bm) * math.ceil(coutp / bn)
    return math.ceil(tiles / (SMS * ng)) * bm * bn * ng


def main():
    files = [a for a in sys.argv[1:] if not a.startswith("--")]
    rows = [r for f in files for r in json.loads(Path(f).read_text())]
    ratio = collections.defaultdict(list)
    for r in rows:
        m, coutp = geom(r)
        c = {k: t / base(k, m, coutp) for k, t in r["ms"].items()}
        lo = min(c.values())
        for k, v in c.items():
            ratio[k].append(v / lo)
    cost = {k: statistics.median(v) for k, v in ratio.items()}
    for k, v in sorted(cost.items(), key=lambda kv: kv[1]):
        print(f"{k:18s} {v:.3f}")
    best = picked = 0.0
    for r in rows:
        m, coutp = geom(r)
        pk = min(r["ms"], key=lambda k: cost[k] * base(k, m, coutp))
        best += min(r["ms"].values())
        picked += r["ms"][pk]
    print(f"sum of per-layer best {best:.3f} ms, model picks {picked:.3f} ms (+{100 * (picked / best - 1):.2f}%)")
    if "--write" in sys.argv:
        src = CU.read_text()

        def sub(mo):
            return mo.group(1) + f"{cost[mo.group(2)]:.3f}f" if mo.group(2) in cost else mo.group(0)

        src = re.sub(r'(\{"((?:g\d_)?tm\d+tn\d+_w\d+x\d+)", \d+, \d+, \d+, \d+, )\d+\.\d+f', sub, src)
        CU.write_text(src)
        print("patched", CU)


if __name__ == "__main__":
    main()
