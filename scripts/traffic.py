"""DRAM traffic per LUT-conv launch from an ncu metrics CSV -> profiles/traffic_<workload>.json.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:lutconv \
        -c <convs per step> --csv --log-file gpurun_out/traffic_r8.csv python bench.py --steps 1 ...
    python scripts/traffic.py gpurun_out/traffic_r8.csv r8

ncu replays each kernel with caches flushed, so these are cold-cache bytes per launch: the
number bench.py reports as roofline.traffic beside the algorithmic bytes.
"""

import collections
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def main():
    src, workload = sys.argv[1], sys.argv[2]
    lines = Path(src).read_text().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    per = collections.defaultdict(dict)
    names = {}
    for row in csv.DictReader(lines[start:]):
        v = float(row["Metric Value"].replace(",", ""))
        unit = row["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6}.get(unit, 1)
        per[row["ID"]][row["Metric Name"]] = v * scale
        names[row["ID"]] = row["Kernel Name"]
    launches = []
    for i, m in per.items():
        launches.append({"kernel": names[i].split("(")[0][:60],
                         "dram_bytes": int(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)),
                         "ns": int(m.get("gpu__time_duration.sum", 0))})
    tot = sum(x["dram_bytes"] for x in launches)
    out = {"source": src, "workload": workload, "launches": len(launches),
           "dram_bytes_per_launch": int(tot / max(len(launches), 1)), "per_launch": launches,
           "note": "ncu dram__bytes_read.sum + dram__bytes_write.sum per LUT-conv launch of one step "
                   "(cold cache: ncu flushes caches between replays)"}
    dst = ROOT / "profiles" / f"traffic_{workload}.json"
    dst.write_text(json.dumps(out, indent=1))
    print(dst, out["dram_bytes_per_launch"])


if __name__ == "__main__":
    main()
