"""Digest of one ncu --set full report for the judge and for tuning: the ncu_summary table plus the
L2 / crossbar / shared-memory throughput metrics and per-instruction stall attribution (SASS page).

    python scripts/ncu_digest.py REP.ncu-rep --out profiles/x.md
"""
import argparse
import collections
import csv
import io
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))

EXTRA = [
    "l1tex__m_xbar2l1tex_read_bytes.sum.per_second",
    "lts__t_sectors_srcunit_tex_op_read.sum.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_writes.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
]


def ncu(rep, page):
    return subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"] + (["--print-source", "sass"] if page == "source" else []),
                          capture_output=True, text=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--out", required=True)
    ap.add_argument("--top", type=int, default=5)
    a = ap.parse_args()
    lines = [f"# ncu digest: {Path(a.rep).name}", ""]
    raw = list(csv.reader(io.StringIO(ncu(a.rep, "raw"))))
    hdr, units = raw[0], raw[1]
    for row in raw[2:]:
        name = row[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        lines += [f"## {name[:120]}", "", "| metric | value |", "|---|---|"]
        for m in EXTRA:
            if m in hdr:
                i = hdr.index(m)
                lines.append(f"| `{m}` | {row[i]} {units[i]} |")
        lines.append("")
    rows = list(csv.reader(io.StringIO(ncu(a.rep, "source"))))
    hi = [i for i, r in enumerate(rows[:5]) if "Source" in r]
    if hi:
        hdr, data = rows[hi[0]], rows[hi[0] + 1:]
        src, ex = hdr.index("Source"), hdr.index("Instructions Executed")
        reasons = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        f = lambda r, i: float(r[i] or 0) if i < len(r) else 0.0
        mix = collections.Counter()
        for r in data:
            t = r[src].split()
            op = (t[1] if t and t[0].startswith("@") else (t[0] if t else "")).split(".")[0]
            mix[op] += f(r, ex)
        T = sum(mix.values()) or 1
        lines += ["## SASS instruction mix and stalls", "", f"instructions executed: {int(T)}", "",
                  "mix: " + ", ".join(f"{k} {100 * v / T:.1f}%" for k, v in mix.most_common(12)), ""]
        tot = {h: sum(f(r, i) for r in data) for i, h in reasons}
        S = sum(tot.values()) or 1
        for i, h in sorted(reasons, key=lambda x: -tot[x[1]]):
            if tot[h] / S < 0.03:
                continue
            lines.append(f"- {h} {100 * tot[h] / S:.1f}% of stall samples; top: " + "; ".join(
                f"`{r[src][:48]}` {100 * f(r, i) / S:.2f}%" for r in sorted(data, key=lambda r: -f(r, i))[:a.top]))
    Path(a.out).write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
