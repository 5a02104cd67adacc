"""profiles/conflicts.json from ncu summaries (the shared-load wavefront and bank-conflict rows):

    python scripts/conflicts_from_ncu.py r50=profiles/r2_r2a_ncu_s0b1.b.md,profiles/r2_r2a_ncu_s1b1.c.md \
        r8=profiles/r2_r2a_ncu_r8s0b0b.md

bench.py reports the pooled conflict share as roofline.lds_conflict_wavefront_frac for the workload."""
import json
import re
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def rows(md: Path):
    txt = md.read_text()
    kern = re.search(r"^## (.+)$", txt, re.M).group(1)
    w = float(re.search(r"shared-load wavefronts \(`[^`]+`\) \| ([0-9.]+)", txt).group(1))
    c = float(re.search(r"shared-load bank conflicts \(`[^`]+`\) \| ([0-9.]+)", txt).group(1))
    return {"kernel": kern, "source": str(md.relative_to(ROOT)), "shared_ld_wavefronts": w,
            "bank_conflict_wavefronts": c, "conflict_frac": round(c / w, 4)}


def main():
    doc = {"source": "ncu --set full captures (scripts/conflicts_from_ncu.py): " + " ".join(sys.argv[1:])}
    for arg in sys.argv[1:]:
        wl, files = arg.split("=", 1)
        doc[wl] = [rows(ROOT / f) for f in files.split(",")]
    (ROOT / "profiles" / "conflicts.json").write_text(json.dumps(doc, indent=1) + "\n")
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()
