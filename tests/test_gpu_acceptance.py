"""SPEC.md acceptance criteria 4 and 5 on the committed
fixtures (tests/fixtures/quantc, quantc::fixtures::write_all):

4. int8 -> int32 desk-scale analog of Table 1: on make_small_cnn the searched
   strategy's REALIZED integer model reaches top-1 agreement >= 0.99 with fp32
   on the 256-sample evaluation set.
5. int8 -> int16 analog (arm_vmlal_like) on make_overflow_probe: (a) 8 bits on
   every edge ((i8,i8)->i16 accumulation) overflows in trap mode; (b) greedy
   search finds a strategy with no trap-mode overflow and agreement >= 0.97;
   (c) that strategy uses fewer than the maximum bits on an accumulator-
   feeding edge (the paper's Fig. 5 pattern)."""
import json
import os

import numpy as np
import pytest

from paper_2103_14949_b200 import quantc as Q

pytestmark = pytest.mark.gpu

FX = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fixtures", "quantc")


def _samples(name):
    man = json.load(open(os.path.join(FX, name + ".json")))
    out = []
    for s in man:
        ref = s["inputs"][0]
        n = int(np.prod(ref["shape"]))
        blob = open(os.path.join(FX, ref["file"]), "rb").read()
        out.append(np.frombuffer(blob, np.float32, n, ref["offset"]).reshape(ref["shape"]))
    return np.stack(out)


def _pipeline(b, model, spec_name, method, **kw):
    g = b.load_graph(os.path.join(FX, model + ".json"))
    cal = _samples(model + "_calibration")
    spec = b.parse_spec(open(os.path.join(FX, "specs", spec_name + ".json")).read())
    topo = b.generate_topology(g, spec)
    sim = b.insert_simulated_quantize(g, topo)
    ds = b.dataset(cal)
    st = b.collect_stats(g, ds, 2048, b.simulated_edge_indices(g, topo))
    thr = st.estimate_thresholds(method, **kw)
    ev = b.evaluator(sim, spec, topo, thr, st, ds)
    return g, spec, sim, ev


def _agreement(b, g_fp32, realized, xs):
    ds = b.dataset(xs)
    ref = b.predict_top1(g_fp32, ds)
    got = []
    for x in xs:
        y, _ = b.eval_int(realized, x, trap=True)
        got.append(int(np.argmax(np.asarray(y, np.float64).reshape(-1))))
    return float(np.mean(np.asarray(got) == ref))


def test_acceptance4_small_cnn_int8_int32(b200):
    # max thresholds (the criterion leaves the estimator open; 8-bit KL
    # thresholds clip this fixture's 1,024 pooled feature values so hard
    # that even all_hi loses 89% agreement — scripts/diag_acceptance.py)
    g, spec, sim, ev = _pipeline(b200, "small_cnn", "int8_int32", "max")
    res = b200.search("greedy", ev.space(), evaluator=ev, rounds=1, tol=0.01)
    R = b200.realize(sim, ev.strategy_for(res.best), spec)
    assert _agreement(b200, g, R, _samples("small_cnn_evaluation")) >= 0.99


def test_acceptance5_overflow_probe_int16(b200):
    g, spec, sim, ev = _pipeline(b200, "overflow_probe", "arm_vmlal_like", "max")
    sp = ev.space()
    cal = _samples("overflow_probe_calibration")
    # (a) 8 bits everywhere -> (i8, i8) -> i16 accumulation, which overflows
    R8 = b200.realize(sim, ev.strategy_for([8] * len(sp.hi)), spec)
    with pytest.raises(Q.OverflowError_):
        for x in cal:
            b200.eval_int(R8, x, trap=True)
    # (b) greedy: no trap-mode overflow on the calibration set, agreement >= 0.97
    res = b200.search("greedy", sp, evaluator=ev, rounds=1, tol=0.01)
    R = b200.realize(sim, ev.strategy_for(res.best), spec)
    for x in cal:
        b200.eval_int(R, x, trap=True)
    assert _agreement(b200, g, R, _samples("overflow_probe_evaluation")) >= 0.97
    # (c) fewer than the maximum bits on an edge feeding the dense accumulator
    assert min(res.best) < max(sp.hi)
