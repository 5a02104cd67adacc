"""Append a one-step kernel breakdown (the last end-to-end replay in an ncu launch list) to a summary.

    python scripts/step_breakdown.py gpurun_out/launches_r8.csv profiles/r1_r8_ftconv_ncu.md
"""
import collections
import csv
import sys
from pathlib import Path


def main():
    src, dst = sys.argv[1], sys.argv[2]
    last = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # take the last N axb launches instead
    lines = Path(src).read_text().splitlines()
    st = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows = list(csv.DictReader(lines[st:]))
    seq = [(r["Kernel Name"], float(r["Metric Value"].replace(",", ""))) for r in rows
           if r["Metric Name"] == "gpu__time_duration.sum"]
    if last:
        step = [(n, v) for n, v in seq if n.startswith(("axb::", "void axb::"))][-last:]
    else:
        i0 = [i for i, (n, _) in enumerate(seq) if "cifar_decode" in n][-1]
        step = []
        for n, v in seq[i0:]:
            if not n.startswith(("axb::", "void axb::")):
                break
            step.append((n, v))
    tot = sum(v for _, v in step)
    agg = collections.OrderedDict()
    for n, v in step:
        a = agg.setdefault(n.split("(")[0][:70], [0, 0.0])
        a[0] += 1
        a[1] += v
    what = f"the last {last} libaxb launches" if last else "the last end-to-end CUDA-graph replay, record decode -> classifier"
    out = ["", f"## One bench step ({what}), ncu gpu__time_duration (serialised, cold cache)", "",
           "| kernel | launches | time (us) | share |", "|---|---|---|---|"]
    for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k}` | {c} | {v / 1e3:.1f} | {100 * v / tot:.1f}% |")
    out.append(f"| total | {len(step)} | {tot / 1e3:.1f} | |")
    with open(dst, "a") as f:
        f.write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main()
