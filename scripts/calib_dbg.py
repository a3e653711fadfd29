import ctypes as C, os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import bench
from paper_2103_14949_b200 import fixtures as F, quantc as Q, parallel as P
MODE = os.environ.get("MODE", "")
if "setdev" in MODE:
    torch.cuda.set_device(0)
b = Q.load_b200()
if "ops" in MODE:
    from paper_2103_14949_b200 import cuda_ops
    ops = cuda_ops.load()
    ops.set_engine_mode("auto")
L = b.lib
m = F.resnet(50)
data = m.data(64, seed=9)
g, spec, topo, sim, ds, st, thr = bench.build_pipeline(b, m, data)
cal_data = np.ascontiguousarray(m.data(128, seed=17))
def cal(tag):
    cds = b.dataset(cal_data)
    loc = P.B200Local(b, g, cds)
    edges = b.simulated_edge_indices(g, topo)
    P.B200Local(b, g, b.dataset(cal_data[:2])).extrema(edges)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    lo, hi = loc.extrema(edges); t1 = time.perf_counter()
    print(tag, f"extrema {1e3*(t1-t0):.0f} ms", flush=True)
cal("start")
cal("again")
