"""Print the fused-engine stage programs of ResNet-50 (QUANTC_DUMP_PLAN=1); needs a GPU."""
import os, sys
sys.path.insert(0, "/root/repo")
os.environ["QUANTC_DUMP_PLAN"] = "1"
from paper_2103_14949_b200 import quantc as Q, fixtures as F
import bench
b = Q.load_b200()
m = F.resnet(50)
data = m.data(2, seed=9)
g, spec, topo, sim, ds, st, thr = bench.build_pipeline(b, m, data)
ev = b.evaluator(sim, spec, topo, thr, st, ds)
ev.loss(bench.candidates(ev.space(), 1)[0])
