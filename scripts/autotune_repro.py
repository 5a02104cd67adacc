"""Repeat GpuGraph.autotune on ResNet-50 (batch 256) to catch nondeterministic kernel variants."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from bench import make_images, workload_spec  # noqa: E402
from paper_2002_09481_b200.graph import GpuGraph  # noqa: E402

spec = workload_spec(sys.argv[1] if len(sys.argv) > 1 else "r50", "trunc2")
batch = int(sys.argv[2]) if len(sys.argv) > 2 else spec["batch"]
imgs, _ = make_images(spec["kind"], batch, seed=1000)
g = GpuGraph(spec["nodes"])
x = torch.from_numpy(imgs).cuda()
want = g.run(x).clone()
t0 = time.time()
for it in range(int(sys.argv[3]) if len(sys.argv) > 3 else 4):
    try:
        g.autotune(x, reps=2)
        ok = torch.equal(g.run(x).view(torch.int32), want.view(torch.int32))
        print(f"iter {it}: autotune ok, logits equal {ok}  ({time.time() - t0:.0f}s)", flush=True)
    except Exception as e:
        print(f"iter {it}: {type(e).__name__}: {e}", flush=True)
