import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import bench
from paper_2103_14949_b200 import quantc as Q, fixtures as F
b = Q.load_b200()
m = F.resnet(50)
data = m.data(64, seed=9)
g, spec, topo, sim, ds, st, thr = bench.build_pipeline(b, m, data)
ev = b.evaluator(sim, spec, topo, thr, st, ds)
cands = bench.candidates(ev.space(), 8)
for i in range(6):
    t0 = time.perf_counter(); bd = ev.bind(cands[i]); t1 = time.perf_counter()
    b.predict_top1(sim, ds, 0, bd); t2 = time.perf_counter()
    print("bind %.2f ms  predict_top1 %.2f ms" % (1e3*(t1-t0), 1e3*(t2-t1)), file=sys.stderr)
