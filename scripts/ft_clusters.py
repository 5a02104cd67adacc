"""Print the resident cluster count of every ftable-kernel variant on cuda:0."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from paper_2002_09481_b200 import _lib  # noqa: E402

torch.cuda.init()
lib = _lib.load()
for v in range(1, lib.axb_ft_variant_count()):
    print(lib.axb_ft_variant_name(v).decode(), lib.axb_ft_variant_clusters(v, 1), lib.axb_ft_variant_clusters(v, 0))
