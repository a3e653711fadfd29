"""Profiling driver for C3 (native MobileNetV2 @224, arm_vmlal_like with 8-bit
codes, fused engine): one grouped losses() call of 4 candidates bracketed by
cudaProfilerStart/Stop (`ncu --profile-from-start off`)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2103_14949_b200 import fixtures as F  # noqa: E402
from paper_2103_14949_b200 import quantc as Q  # noqa: E402

b = Q.load_b200()
model = F.mobilenet_v2(image=224, width=1.0, classes=1000, native=True)
data = model.data(int(os.environ.get("BATCH", "64")), seed=9)
g = b.graph(model.doc, model.blob)
spec = b.parse_spec(F.spec_fixture("arm_vmlal_like"))
topo = b.generate_topology(g, spec)
sim = b.insert_simulated_quantize(g, topo)
ds = b.dataset(data)
st = b.collect_stats(g, ds, 2048, b.simulated_edge_indices(g, topo))
thr = st.estimate_thresholds("quantile", quantile=0.999, pow2=True)
ev = b.evaluator(sim, spec, topo, thr, st, ds, min_bit=8)
cands = [[min(v, 8) for v in c] for c in bench.candidates(ev.space(), 8)]
print("fused:", repr(b.fused_status(sim, ev.bind(cands[0]))))
ev.losses(cands[:4])
torch.cuda.synchronize()
torch.cuda.profiler.start()
ev.losses(cands[4:8])
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled 4 candidates")
