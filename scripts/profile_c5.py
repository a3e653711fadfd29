"""Profiling driver for C5 (native Inception-v3-style @299, int8_int32, the bench leg's
layout, fused engine): one grouped losses() call of 4 candidates bracketed by
cudaProfilerStart/Stop (`ncu --profile-from-start off`)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2103_14949_b200 import fixtures as F  # noqa: E402
from paper_2103_14949_b200 import quantc as Q  # noqa: E402

b = Q.load_b200()
model = F.inception_v3(image=299, width=16, modules=2, head="gap", native=True)
data = model.data(int(os.environ.get("BATCH", "8")), seed=9)
g = b.graph(model.doc, model.blob)
spec = b.parse_spec(F.spec_fixture("int8_int32"))
topo = b.generate_topology(g, spec)
sim = b.insert_simulated_quantize(g, topo)
ds = b.dataset(data)
st = b.collect_stats(g, ds, 2048, b.simulated_edge_indices(g, topo))
thr = st.estimate_thresholds("quantile", quantile=0.999, pow2=True)
ev = b.evaluator(sim, spec, topo, thr, st, ds, min_bit=4)
cands = [[min(v, 8) for v in c] for c in bench.candidates(ev.space(), 8)]
print("fused:", repr(b.fused_status(sim, ev.bind(cands[0]))))
ev.losses(cands[:4])
torch.cuda.synchronize()
torch.cuda.profiler.start()
ev.losses(cands[4:8])
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled 4 candidates")
