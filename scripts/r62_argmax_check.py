import sys, torch, numpy as np
sys.path.insert(0, '.')
from bench import workload_spec, make_images, sweep_luts
from paper_2002_09481_b200 import resnet
from paper_2002_09481_b200.graph import GpuGraph
imgs, _ = make_images("cifar", 1000, seed=1000)
x = torch.from_numpy(imgs).cuda()
from paper_2002_09481_b200 import types as T
for name, lut in [("trunc2", T.truncated_lut(T.Signedness.SIGNED, 2))] + [(f"cand{i}", l) for i, l in enumerate(sweep_luts()[:4])]:
    y = GpuGraph(resnet.cifar_resnet(10, lut, seed=0)).run(x).cpu().numpy().reshape(1000, -1)
    print(name, "distinct", len(set(y.argmax(1).tolist())), "logit std across images", float(y.std(0).mean()), "mean", float(y.mean()))
