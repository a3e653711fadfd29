"""Realized int8 ResNet-50 (batch 64) eval_int: wall time per call and, with
QUANTC_STEP_PROF=<ms>, the engine's per-op host-time summary."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2103_14949_b200 import fixtures as F  # noqa: E402
from paper_2103_14949_b200 import quantc as Q  # noqa: E402

b = Q.load_b200()
B = int(os.environ.get("B", "64"))
m = F.resnet(50)
data = m.data(B, seed=9)
g, spec, topo, sim, ds, st, thr = bench.build_pipeline(b, m, data)
ev = b.evaluator(sim, spec, topo, thr, st, ds)
mb = F.resnet(50, batch=B)
gb = b.graph(mb.doc, mb.blob)
R = b.realize(b.insert_simulated_quantize(gb, b.generate_topology(gb, spec)),
              ev.strategy_for(ev.space().all_hi()), spec)
x = np.ascontiguousarray(data.reshape(B, 3, 224, 224))
for i in range(4):
    t0 = time.perf_counter()
    y, dt = b.eval_int(R, x)
    t1 = time.perf_counter()
    print(f"call {i}: {1e3 * (t1 - t0):.2f} ms wall", flush=True)
