"""How much of a step is host/sync gap: evaluate the same candidates one per
agreement_counts call vs four per call (one host sync per call)."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2103_14949_b200 import fixtures as F, quantc as Q  # noqa: E402

b = Q.load_b200()
L = b.lib
L.qc_evaluator_agreement.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.c_size_t, C.c_size_t,
                                     C.POINTER(C.c_int64)]
m = F.resnet(50)
data = m.data(64, seed=9)
g, spec, topo, sim, ds, st, thr = bench.build_pipeline(b, m, data)
ev = b.evaluator(sim, spec, topo, thr, st, ds)
cands = bench.candidates(ev.space(), 40)
arr = np.asarray(cands, np.int32)
counts = np.zeros(len(cands), np.int64)


def run(per_call, n=32):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(0, n, per_call):
        sub = np.ascontiguousarray(arr[i:i + per_call])
        L.qc_evaluator_agreement(ev.h, sub.ctypes.data_as(C.POINTER(C.c_int)), per_call,
                                 arr.shape[1], counts.ctypes.data_as(C.POINTER(C.c_int64)))
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


run(1, 8)
for k in (1, 4, 1, 4):
    print(f"{k} candidate(s)/call: {run(k):.3f} ms per candidate")
