"""GPU: the B200 implementation against the committed reference golden
vectors (tests/golden/reference_golden.json, produced by the compiled
reference).  Independent of oracle/_ref being present."""
import json
import os

import numpy as np
import pytest

from paper_2103_14949_b200 import fixtures as F
from paper_2103_14949_b200 import quantc as Q

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


def test_sim_quant_values_golden(b200):
    for x, t, b, want in GOLD["sim_quant_value"]:
        assert b200.simulated_quantize_value(x, Q.QParams.symmetric(t, b)) == want
    xs, wants, params = [], [], []
    for x, t, bit, sign, zp, acc, acc_scale, want in GOLD["sim_quant_tuples"]:
        p = Q.QParams.make(t, bit, sign, Q.I8 if sign else Q.U8, zero_point=zp,
                           acc_dtype=Q.I16 if acc else Q.NONE, acc_scale=acc_scale)
        got = b200.simulated_quantize(np.array([x], np.float32), p)[0]
        assert np.float32(got).tobytes() == np.float32(want).tobytes()


def test_kl_golden(b200):
    for h, absmax, tb, want in GOLD["kl_random"]:
        assert b200.threshold_kl(np.array(h, np.int64), absmax, tb) == want
    h0 = np.zeros(2048, np.int64)
    h0[0] = 1000
    assert b200.threshold_kl(h0, 5.0, 8) == GOLD["kl_all_mass_bin0"]


def test_small_cnn_pipeline_golden(b200):
    pipe = GOLD["small_cnn_pipeline"]
    m = F.small_cnn()
    data = m.data(16)
    g = b200.graph(m.doc, m.blob)
    spec = b200.parse_spec(F.spec_fixture("int8_int32"))
    topo = b200.generate_topology(g, spec)
    sim = b200.insert_simulated_quantize(g, topo)
    ds = b200.dataset(data)
    edges = b200.simulated_edge_indices(g, topo)
    assert edges == pipe["edges"]
    st = b200.collect_stats(g, ds, 2048, edges)
    for k in edges:
        e, want = st.get(k), pipe["stats"][str(k)]
        assert (e["min"], e["max"], e["absmax"]) == (want["min"], want["max"], want["absmax"])
        nz = {str(i): int(c) for i, c in enumerate(e["counts"]) if c}
        assert nz == want["counts_nonzero"]
    for key, want in pipe["thresholds"].items():
        meth, pw = (key[:-5], True) if key.endswith("_pow2") else (key, False)
        got = st.estimate_thresholds(meth, pow2=pw)
        assert {str(k): v for k, v in got.items()} == want
    thr = st.estimate_thresholds("quantile", pow2=False)
    ev = b200.evaluator(sim, spec, topo, thr, st, ds)
    assert ev.reference_predictions().tolist() == pipe["refs"]
    assert ev.losses(pipe["candidates"]).tolist() == pipe["losses"]
    res = b200.search("greedy", ev.space(), evaluator=ev, rounds=1, tol=0.05)
    assert {"best": res.best, "best_loss": res.best_loss,
            "evaluations": res.evaluations} == pipe["greedy"]


def test_overflow_probe_trap_and_saturate(b200):
    doc, blob = F.overflow_dense(256, 127, "int16")
    g = b200.graph(doc, blob)
    x = np.full((1, 256), 127.0, np.float32)
    out, dt = b200.eval_int(g, x, trap=False)
    assert dt == Q.I16 and (out == 32767).all()
    with pytest.raises(Q.OverflowError_) as ei:
        b200.eval_int(g, x, trap=True)
    assert ei.value.flat_index == 0 and ei.value.value == 127 * 127 * 256
