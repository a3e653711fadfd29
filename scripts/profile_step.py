"""Profiling driver: builds the ResNet-50 evaluator, warms up, then brackets
exactly one candidate evaluation with cudaProfilerStart/Stop so that
`ncu --profile-from-start off` captures one step's launches."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2103_14949_b200 import fixtures as F  # noqa: E402
from paper_2103_14949_b200 import quantc as Q  # noqa: E402

batch = int(os.environ.get("BATCH", "64"))
b = Q.load_b200()
model = F.resnet(int(os.environ.get("DEPTH", "50")))
data = model.data(batch, seed=9)
g, spec, topo, sim, ds, st, thr = bench.build_pipeline(b, model, data)
ev = b.evaluator(sim, spec, topo, thr, st, ds)
group = int(os.environ.get("GROUP", "1"))  # >1: one losses() call over GROUP candidates
cands = bench.candidates(ev.space(), 3 + group)
for c in cands[:3]:
    ev.loss(c)
ev.losses(cands[:group])
torch.cuda.synchronize()
torch.cuda.profiler.start()
if group > 1:
    ev.losses(cands[3:3 + group])
else:
    ev.loss(cands[3])
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled", group, "candidate(s)")
