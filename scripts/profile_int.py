"""Profiling driver for the realized int8 path: one eval_int call of the
batched realized ResNet-50 bracketed by cudaProfilerStart/Stop."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2103_14949_b200 import fixtures as F  # noqa: E402
from paper_2103_14949_b200 import quantc as Q  # noqa: E402

b = Q.load_b200()
m = F.resnet(50)
data = m.data(64, seed=9)
g, spec, topo, sim, ds, st, thr = bench.build_pipeline(b, m, data)
ev = b.evaluator(sim, spec, topo, thr, st, ds)
mb = F.resnet(50, batch=64)
gb = b.graph(mb.doc, mb.blob)
R = b.realize(b.insert_simulated_quantize(gb, b.generate_topology(gb, spec)),
              ev.strategy_for(ev.space().all_hi()), spec)
x = np.ascontiguousarray(data.reshape(64, 3, 224, 224))
b.eval_int(R, x)
torch.cuda.synchronize()
torch.cuda.profiler.start()
b.eval_int(R, x)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled eval_int")
