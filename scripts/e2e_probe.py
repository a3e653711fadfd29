"""Break down one qc_predict_top1 call (e2e path) on the GPU box: host->device
rates (pageable / pinned / memcpy into pinned) and the call at several
dataset sizes.  Diagnostic only."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2103_14949_b200 import quantc as Q, fixtures as F

def rate(fn, nbytes, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return nbytes * reps / (time.perf_counter() - t0) / 1e9

n = 38535168
host = torch.empty(n, dtype=torch.uint8)
host.numpy()[:] = 1
pin = torch.empty(n, dtype=torch.uint8, pin_memory=True)
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
out = {}
out["pageable_h2d_GBs"] = rate(lambda: dev.copy_(host, non_blocking=False), n)
out["pinned_h2d_GBs"] = rate(lambda: dev.copy_(pin, non_blocking=True), n)
out["memcpy_to_pinned_GBs"] = rate(lambda: pin.copy_(host), n)
out["cpus"] = os.cpu_count()
b = Q.load_b200()
model = F.resnet(50)
for B in (64, 16):
    data = model.data(B, seed=9)
    g, spec, topo, sim, ds, st, thr = bench.build_pipeline(b, model, data)
    ev = b.evaluator(sim, spec, topo, thr, st, ds)
    sp = ev.space()
    binding = ev.bind(sp.all_hi())
    b.predict_top1(sim, ds, 0, binding)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); b.predict_top1(sim, ds, 0, binding); ts.append(time.perf_counter() - t0)
    out[f"predict_top1_B{B}_ms"] = 1e3 * min(ts)
    t0 = time.perf_counter(); bd = ev.bind(sp.all_lo()); out[f"bind_ms_B{B}"] = 1e3 * (time.perf_counter() - t0)
print(json.dumps(out))
