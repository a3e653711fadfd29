"""Diagnose SPEC acceptance 4 on the committed small_cnn fixture: search loss,
sim-quant vs fp32 agreement, realized vs fp32 agreement, per-sample outputs."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests import test_gpu_acceptance as T  # noqa: E402
from paper_2103_14949_b200 import quantc as Q  # noqa: E402

b = Q.load_b200()
for method, kw in (("kl", dict(kl_bits=8)), ("max", {}), ("quantile", dict(quantile=0.999))):
    g, spec, sim, ev = T._pipeline(b, "small_cnn", "int8_int32", method, **kw)
    sp = ev.space()
    ev_x = T._samples("small_cnn_evaluation")
    ds = b.dataset(ev_x)
    ref = b.predict_top1(g, ds)
    for name, cand in (("all_hi", sp.all_hi()),):
        bnd = ev.bind(cand)
        simp = b.predict_top1(sim, ds, binding=bnd)
        R = b.realize(sim, ev.strategy_for(cand), spec)
        outs = [b.eval_int(R, x, trap=False) for x in ev_x[:4]]
        rp = []
        for x in ev_x:
            y, dt = b.eval_int(R, x, trap=False)
            rp.append(int(np.argmax(np.asarray(y, np.float64).reshape(-1))))
        print(method, name, "loss", ev.loss(cand), "sim agree", np.mean(simp == ref),
              "realized agree", np.mean(np.asarray(rp) == ref), "dtype", outs[0][1])
        print("  fp32", b.eval_fp32(g, ev_x[0]).reshape(-1)[:5])
        print("  realized", np.asarray(outs[0][0]).reshape(-1)[:5])
        print("  sim", b.eval_fp32(sim, ev_x[0], bnd).reshape(-1)[:5])
