"""e2e probe: predict_top1 through the C-ABI (host dataset -> predictions),
ms per call at the bench workload; run once per QUANTC_E2E_PARTS value."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2103_14949_b200 import fixtures as F  # noqa: E402
from paper_2103_14949_b200 import quantc as Q  # noqa: E402

b = Q.load_b200()
m = F.resnet(50)
data = m.data(int(os.environ.get("BATCH", "64")), seed=9)
g, spec, topo, sim, ds, st, thr = bench.build_pipeline(b, m, data)
ev = b.evaluator(sim, spec, topo, thr, st, ds)
cands = bench.candidates(ev.space(), 12)
binds = [ev.bind(c) for c in cands]
b.predict_top1(sim, ds, 0, binds[0])
for rep in range(2):
    t0 = time.perf_counter()
    for i in range(10):
        b.predict_top1(sim, ds, 0, binds[1 + i])
    dt = (time.perf_counter() - t0) / 10
    print(f"parts={os.environ.get('QUANTC_E2E_PARTS', '1')} {1e3 * dt:.3f} ms/call "
          f"{len(data) / dt:.0f} img/s")
