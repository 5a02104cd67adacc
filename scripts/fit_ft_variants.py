"""Fit the ftable-kernel cost model from tune_variants.py --family ft outputs and patch the table.

    python scripts/fit_ft_variants.py gpurun_out/tune_r8.json gpurun_out/tune_r50.json [--write]

Model (pick_ft_variant in csrc/axb_ftconv.cu): time ~ cost_v * waves * BM * BN,
waves = ceil(super-tiles / resident clusters), super-tile = CL pixel tiles of one
channel block.  cost_v = median over layers of time / (waves*BM*BN), normalised by
each layer's best variant.  Prints the costs and the model's regret vs the measured best.
"""

import collections
import json
import math
import re
import statistics
import sys
from pathlib import Path

CU = Path(__file__).resolve().parent.parent / "paper_2002_09481_b200" / "csrc" / "axb_ftconv.cu"
SMS = 148


def parse(name):
    m = re.match(r"ft(\d+)(r?)_tm(\d+)_w(\d+)(?:_k(\d+))?(?:_c(\d+))?$", name)
    if not m:
        return None
    return int(m.group(1)), int(m.group(3)), int(m.group(4)), int(m.group(6) or 1), m.group(2) == "r"


def geom(r):
    n, h, w, c = r["in"]
    kh, kw, ci, co = r["filters"]
    m = n * (r["macs"] // (n * kh * kw * ci * co))
    return m, (co + 15) // 16 * 16


def base(name, m, coutp):
    bn, tm, warps, cl, res = parse(name)
    bm = warps * 32 * tm
    if res:  # fixed channel block per CTA
        ntb, ntm = coutp // bn, math.ceil(m / bm)
        per = min(SMS // ntb, ntm)
        return math.ceil(ntm / per) * bm * bn
    tiles = math.ceil(math.ceil(m / bm) / cl) * (coutp // bn)
    return math.ceil(tiles / (SMS // cl)) * bm * bn


def main():
    files = [a for a in sys.argv[1:] if not a.startswith("--")]
    rows = [r for f in files for r in json.loads(Path(f).read_text())]
    ratio = collections.defaultdict(list)
    for r in rows:
        m, coutp = geom(r)
        c = {k: t / base(k, m, coutp) for k, t in r["ms"].items() if parse(k)}
        lo = min(c.values())
        for k, v in c.items():
            ratio[k].append(v / lo)
    cost = {k: statistics.median(v) for k, v in ratio.items()}
    for k, v in sorted(cost.items(), key=lambda kv: kv[1]):
        print(f"{k:20s} {v:.3f}")
    best = picked = 0.0
    for r in rows:
        m, coutp = geom(r)
        ks = [k for k in r["ms"] if parse(k)]
        pk = min(ks, key=lambda k: cost[k] * base(k, m, coutp))
        best += min(r["ms"][k] for k in ks)
        picked += r["ms"][pk]
    print(f"sum of per-layer best {best:.3f} ms, model picks {picked:.3f} ms (+{100 * (picked / best - 1):.2f}%)")
    if "--write" in sys.argv:
        src = CU.read_text()

        def sub(mo):
            return mo.group(1) + f"{cost[mo.group(2)]:.3f}f" if mo.group(2) in cost else mo.group(0)

        src = re.sub(r'(\{"(ft\d+r?_tm\d+_w\d+(?:_k\d+)?(?:_c\d+)?)", \d+, \d+, \d+, \d+, )\d+\.\d+f', sub, src)
        CU.write_text(src)
        print("patched", CU)


if __name__ == "__main__":
    main()
