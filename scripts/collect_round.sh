#!/bin/bash
# Copy one gpu_round_full.sh run (TAG) from gpurun_out/ into profiles/ as r1_<TAG>_*: bench lines,
# per-layer tables, tuned variants, run reports, launch list, ncu summaries (+ one-step breakdown),
# DRAM traffic per conv launch, shared-memory conflict shares.
#   bash scripts/collect_round.sh p16
set -e
T=${1:?tag}
cd "$(dirname "$0")/.."
G=gpurun_out
P=profiles
cp $G/bench_r8_$T.txt $P/r1_${T}_bench_r8.json
cp $G/bench_r8_k20_$T.txt $P/r1_${T}_bench_r8_k20.json
cp $G/bench_r50_$T.txt $P/r1_${T}_bench_r50.json
cp $G/bench_r62sweep_$T.txt $P/r1_${T}_bench_r62sweep.json
cp $G/bench_ref_$T.txt $P/r1_${T}_bench_reference_r8.json
cp $G/layers_r8_$T.json $P/r1_${T}_layers_r8.json
cp $G/layers_r50_$T.json $P/r1_${T}_layers_r50.json
cp $G/tuned_r8.json $P/r1_${T}_tuned_r8.json
cp $G/tuned_r50.json $P/r1_${T}_tuned_r50.json
cp $G/launches_r8_$T.csv $P/r1_${T}_launches_r8.csv
for w in r8 r50; do
    cp $G/report_${w}_$T.json $P/r1_${T}_report_$w.json
    cp $G/report_${w}_$T.csv $P/r1_${T}_report_$w.csv
done
python scripts/ncu_summary.py --rep $G/prof_r8_$T.ncu-rep --launches $G/launches_r8_$T.csv \
    --out $P/r1_${T}_r8_ftconv_ncu.md --json $G/ncu_r8_$T.json > /dev/null
python scripts/ncu_summary.py --rep $G/prof_r50_l6_$T.ncu-rep --out $P/r1_${T}_r50_s0b1b_ftconv_ncu.md \
    --json $G/ncu_r50a_$T.json > /dev/null
python scripts/ncu_summary.py --rep $G/prof_r50_l29_$T.ncu-rep --out $P/r1_${T}_r50_s2b1b_ftconv_ncu.md \
    --json $G/ncu_r50b_$T.json > /dev/null
python scripts/step_breakdown.py $G/launches_r8_$T.csv $P/r1_${T}_r8_ftconv_ncu.md > /dev/null
python scripts/traffic.py $G/traffic_r8.csv r8
python scripts/traffic.py $G/traffic_r50.csv r50
python - "$T" <<'EOF'
import json, sys
t = sys.argv[1]


def rows(f):
    out = []
    for d in json.load(open(f)):
        w = float(str(d["l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"]).replace(",", ""))
        c = float(str(d["l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"]).replace(",", ""))
        out.append({"kernel": d["kernel"], "shared_ld_wavefronts": w, "bank_conflict_wavefronts": c,
                    "conflict_frac": round(c / w, 4)})
    return out


doc = {"source": f"ncu --set full captures of round {t} (profiles/r1_{t}_*_ftconv_ncu.md): ResNet-8 s0b0.a/b, "
                 "ResNet-50 b64 s0b1.b, s2b1.b",
       "r8": rows(f"gpurun_out/ncu_r8_{t}.json"), "r50": rows(f"gpurun_out/ncu_r50a_{t}.json"),
       "r50_s2b1b": rows(f"gpurun_out/ncu_r50b_{t}.json")}
json.dump(doc, open("profiles/conflicts.json", "w"), indent=1)
EOF
echo "collected $T"
