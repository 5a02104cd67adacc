"""Per-instruction stall attribution from an ncu report's SASS source page.

    python scripts/sass_stalls.py gpurun_out/prof.ncu-rep [--top 30]
Prints the instruction mix (by executions), each stall reason's total, and the top instructions per reason.
"""
import argparse
import collections
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=6)
    args = ap.parse_args()
    out = subprocess.run(["ncu", "-i", args.rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, data = rows[1], rows[2:]
    src, ex = hdr.index("Source"), hdr.index("Instructions Executed")
    reasons = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    f = lambda r, i: float(r[i] or 0)
    mix = collections.Counter()
    for r in data:
        t = r[src].split()
        op = (t[1] if t and t[0].startswith("@") else (t[0] if t else "")).split(".")[0]
        mix[op] += f(r, ex)
    T = sum(mix.values())
    print("instructions executed", int(T))
    print("mix:", ", ".join(f"{k} {100 * v / T:.1f}%" for k, v in mix.most_common(14)))
    tot = {h: sum(f(r, i) for r in data) for i, h in reasons}
    S = sum(tot.values())
    for i, h in sorted(reasons, key=lambda x: -tot[x[1]]):
        if tot[h] / S < 0.02:
            continue
        print(f"{h} {100 * tot[h] / S:.1f}%")
        for r in sorted(data, key=lambda r: -f(r, i))[:args.top]:
            print(f"    {100 * f(r, i) / S:5.2f}%  {r[src][:70]}")


if __name__ == "__main__":
    main()
