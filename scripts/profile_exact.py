"""Profiling driver for the exact FP64 engine: ResNet-50 under the reference's
default thresholds (quantile 0.99, pow2 off -> non-power-of-two scales), one
candidate evaluation over 16 images between cudaProfilerStart/Stop."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_14949_b200 import fixtures as F  # noqa: E402
from paper_2103_14949_b200 import quantc as Q  # noqa: E402

b = Q.load_b200()
model = F.resnet(50)
data = model.data(int(os.environ.get("BATCH", "16")), seed=9)
g = b.graph(model.doc, model.blob)
spec = b.parse_spec(F.spec_fixture("int8_int32"))
topo = b.generate_topology(g, spec)
sim = b.insert_simulated_quantize(g, topo)
ds = b.dataset(data)
st = b.collect_stats(g, ds, 2048, b.simulated_edge_indices(g, topo))
thr = st.estimate_thresholds("quantile", quantile=0.99, pow2=False)
ev = b.evaluator(sim, spec, topo, thr, st, ds)
sp = ev.space()
ev.loss(sp.all_hi())
torch.cuda.synchronize()
torch.cuda.profiler.start()
ev.loss(sp.all_lo())
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("engine:", b.fused_status(sim, ev.bind(sp.all_lo())) or "fused")
