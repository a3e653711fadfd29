"""Acceptance 4 settings sweep on the committed small_cnn fixture: threshold
estimator x min_bit x greedy tolerance -> chosen bits and realized agreement."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests import test_gpu_acceptance as T  # noqa: E402
from paper_2103_14949_b200 import quantc as Q  # noqa: E402

b = Q.load_b200()
ev_x = T._samples("small_cnn_evaluation")
for method, kw in (("max", {}), ("quantile", dict(quantile=0.999)), ("quantile", dict(quantile=0.9999))):
    g, spec, sim, ev = T._pipeline(b, "small_cnn", "int8_int32", method, **kw)
    for tol in (0.0, 0.01):
        res = b.search("greedy", ev.space(), evaluator=ev, rounds=1, tol=tol)
        R = b.realize(sim, ev.strategy_for(res.best), spec)
        print(method, kw, "tol", tol, "bits", res.best, "cal loss", res.best_loss,
              "eval agree", T._agreement(b, g, R, ev_x), flush=True)
