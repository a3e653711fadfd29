"""Realized ResNet-50 (int8_int32 strategy from a calibrated search space)
through eval_int on the B200 engine: batch consistency and timing."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2103_14949_b200 import cuda_ops  # noqa: E402
from paper_2103_14949_b200 import fixtures as F  # noqa: E402
from paper_2103_14949_b200 import quantc as Q  # noqa: E402

b = Q.load_b200()
ops = cuda_ops.load()
m = F.resnet(int(os.environ.get("DEPTH", "50")))
data = m.data(8, seed=9)
g, spec, topo, sim, ds, st, thr = bench.build_pipeline(b, m, data)
ev = b.evaluator(sim, spec, topo, thr, st, ds)
strategy = ev.strategy_for(ev.space().all_hi())
B = int(os.environ.get("BATCH", "64"))
# the same network declared with a batched input, lowered under that strategy
mb = F.resnet(int(os.environ.get("DEPTH", "50")), batch=B)
gb = b.graph(mb.doc, mb.blob)
simb = b.insert_simulated_quantize(gb, b.generate_topology(gb, spec))
R = b.realize(simb, strategy, spec)
R1 = b.realize(sim, strategy, spec)
x = m.data(B, seed=3).reshape(B, 3, 224, 224)
c0 = ops.counters()
t0 = time.perf_counter()
y, dt = b.eval_int(R, x)
t1 = time.perf_counter()
y, dt = b.eval_int(R, x)
t2 = time.perf_counter()
c1 = ops.counters()
print(f"batch {B}: first {1e3*(t1-t0):.1f} ms, second {1e3*(t2-t1):.1f} ms -> {B/(t2-t1):.0f} img/s; "
      f"tc {c1['tcgen05_gemms']-c0['tcgen05_gemms']} simt {c1['simt_int_convs']-c0['simt_int_convs']}")
y1, _ = b.eval_int(R1, x[:1])
per = y.size // B
print("batch row 0 == single:", np.array_equal(y[:per], y1))
