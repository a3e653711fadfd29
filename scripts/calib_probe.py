"""C4 probe: ResNet-50 calibration (collect_stats: extrema pass + histogram
pass, B=2048) and KL thresholds on one GPU through the C-ABI."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_14949_b200 import fixtures as F  # noqa: E402
from paper_2103_14949_b200 import quantc as Q  # noqa: E402

n = int(os.environ.get("N", "128"))
b = Q.load_b200()
m = F.resnet(50)
g = b.graph(m.doc, m.blob)
spec = b.parse_spec(F.spec_fixture("int8_int32"))
topo = b.generate_topology(g, spec)
edges = b.simulated_edge_indices(g, topo)
ds = b.dataset(m.data(n, seed=9))
warm = b.dataset(m.data(4, seed=1))
b.collect_stats(g, warm, 2048, edges)
t0 = time.perf_counter()
st = b.collect_stats(g, ds, 2048, edges)
t1 = time.perf_counter()
thr = st.estimate_thresholds("kl", kl_bits=8)
t2 = time.perf_counter()
print(f"collect_stats {n} imgs {len(edges)} edges: {t1 - t0:.3f} s = {n / (t1 - t0):.1f} img/s; "
      f"KL thresholds {1e3 * (t2 - t1):.1f} ms")
