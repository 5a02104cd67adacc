"""Summarise ncu artefacts into profiles/ (committed; gpurun_out/ is scratch).

    python scripts/ncu_summary.py --rep gpurun_out/prof_r8_i4.ncu-rep --launches gpurun_out/launches_r8_i4.csv \
        --out profiles/r1_r8_lutconv.md [--json profiles/r1_ncu.json]

Per captured kernel: duration, clocks, registers, block size, LDS wavefronts /
bank conflicts, LSU/ALU/FMA pipe use, IPC, warps, DRAM bytes, top stall
reasons; plus the per-kernel share of one bench step from the launch list.
"""

import argparse
import collections
import csv
import json
import subprocess
from pathlib import Path

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "sm clock"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__block_size", "block size"),
    ("launch__grid_size", "grid size"),
    ("smsp__warps_active.avg.per_cycle_active", "warps active / scheduler"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (per SM)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "shared-load wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "shared-load bank conflicts"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__cycles_elapsed.avg", "cycles / SM"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    return [(r[ki].split("(")[0], float(r[vi].replace(",", ""))) for r in data]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches", default="")
    ap.add_argument("--step-launches", type=int, default=0, help="launches per bench step (tail of the list)")
    ap.add_argument("--title", default="")
    ap.add_argument("--out", required=True)
    ap.add_argument("--json", default="")
    args = ap.parse_args()
    hdr, units, data = raw_rows(args.rep)
    lines = [f"# {args.title or Path(args.rep).stem}", "", f"Source: `{args.rep}` (ncu --set full, --clock-control none)", ""]
    summary = []
    for d in data:
        name = d[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        rec = {"kernel": name}
        lines += [f"## {name}", "", "| metric | value |", "|---|---|"]
        for m, label in METRICS:
            if m in hdr:
                i = hdr.index(m)
                rec[m] = d[i]
                lines.append(f"| {label} (`{m}`) | {d[i]} {units[i]} |")
        st = [(h, i) for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
        tot = sum(float(d[i] or 0) for _, i in st) or 1.0
        top = sorted(st, key=lambda x: -float(d[x[1]] or 0))[:8]
        stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): round(100 * float(d[i] or 0) / tot, 1) for h, i in top}
        rec["stalls_pct"] = stalls
        lines += ["", "Stall samples (% of all): " + ", ".join(f"{k} {v}%" for k, v in stalls.items()), ""]
        try:
            wf = float(rec["l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"])
            bc = float(rec["l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"])
            cyc = float(rec["sm__cycles_elapsed.avg"])
            sms = int(float(rec.get("launch__grid_size", "148")))
            lines.append(f"LDS pipe busy: {wf / sms / cyc:.1%} of cycles; conflict wavefronts {bc / wf:.1%} of all.")
            rec["lds_busy"] = round(wf / sms / cyc, 4)
        except Exception:
            pass
        lines.append("")
        summary.append(rec)
    if args.launches:
        seq = launches(args.launches)
        step = seq[-args.step_launches:] if args.step_launches else seq
        tot = collections.defaultdict(float)
        cnt = collections.Counter()
        for nm, v in step:
            tot[nm] += v
            cnt[nm] += 1
        T = sum(tot.values())
        lines += ["## Launch list (one bench step, ncu gpu__time_duration, serialised / cold-cache)", "",
                  "| kernel | launches | time (us) | share |", "|---|---|---|---|"]
        for k, v in sorted(tot.items(), key=lambda x: -x[1]):
            lines.append(f"| `{k[:70]}` | {cnt[k]} | {v / 1000:.1f} | {100 * v / T:.1f}% |")
        lines.append(f"| total | {len(step)} | {T / 1000:.1f} | |")
    Path(args.out).write_text("\n".join(lines) + "\n")
    if args.json:
        Path(args.json).write_text(json.dumps(summary, indent=1))
    print("\n".join(lines))


if __name__ == "__main__":
    main()
