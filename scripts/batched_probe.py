"""Per-candidate step time: one C-ABI call per candidate vs one call for a
batch of candidates (CandidateEvaluator::agreement_counts over a span)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2103_14949_b200 import fixtures as F  # noqa: E402
from paper_2103_14949_b200 import quantc as Q  # noqa: E402

b = Q.load_b200()
L = b.lib
L.qc_evaluator_agreement.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.c_size_t, C.c_size_t,
                                     C.POINTER(C.c_int64)]
m = F.resnet(50)
data = m.data(64, seed=9)
g, spec, topo, sim, ds, st, thr = bench.build_pipeline(b, m, data)
ev = b.evaluator(sim, spec, topo, thr, st, ds)
cands = bench.candidates(ev.space(), 40)


def agree(cs):
    a = np.ascontiguousarray(np.asarray(cs, np.int32))
    out = np.zeros(len(cs), np.int64)
    b.check(L.qc_evaluator_agreement(ev.h, a.ctypes.data_as(C.POINTER(C.c_int)), a.shape[0],
                                     a.shape[1], out.ctypes.data_as(C.POINTER(C.c_int64))))
    return out


agree(cands[:4])
for rep in range(2):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    one = [agree([c])[0] for c in cands[4:34]]
    e1.record()
    torch.cuda.synchronize()
    t_one = e0.elapsed_time(e1) / 30
    e0.record()
    many = agree(cands[4:34])
    e1.record()
    torch.cuda.synchronize()
    t_many = e0.elapsed_time(e1) / 30
    assert list(many) == one
    print(f"per candidate: single calls {t_one:.3f} ms, one batched call {t_many:.3f} ms "
          f"({64 / t_one * 1e3:.0f} vs {64 / t_many * 1e3:.0f} img/s)")
