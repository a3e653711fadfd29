"""realize() (SPEC.md realize module, SURVEY §8(f) "next" row): the lowering
of a simulated graph under a strategy into an integer graph, checked on CPU
through the reference's own integer interpreter (reference
interpreter.cpp:113-482 eval_int), which is the oracle for the realized
semantics.  The calibration pipeline runs on the reference build; only
realize() itself is the B200 library's (pure host code)."""
import numpy as np
import pytest

from paper_2103_14949_b200 import fixtures as F
from paper_2103_14949_b200 import quantc as Q

MODELS = {
    "small_cnn": lambda: F.small_cnn(),
    "resnet18": lambda: F.resnet(18, image=32, classes=10, width=8),
}


def realized(ref, b200, model, spec_name="int8_int32", pow2=True, n=4):
    data = model.data(n)
    g = ref.graph(model.doc, model.blob)
    spec = ref.parse_spec(F.spec_fixture(spec_name))
    topo = ref.generate_topology(g, spec)
    sim = ref.insert_simulated_quantize(g, topo)
    ds = ref.dataset(data)
    st = ref.collect_stats(g, ds, 2048, ref.simulated_edge_indices(g, topo))
    thr = st.estimate_thresholds("quantile", quantile=0.999, pow2=pow2)
    ev = ref.evaluator(sim, spec, topo, thr, st, ds)
    cand = ev.space().all_hi()
    R = b200.realize(sim.copy_to(b200), ev.strategy_for(cand), b200.parse_spec(
        F.spec_fixture(spec_name)))
    return dict(R=R, data=data, sim=sim, ev=ev, cand=cand)


@pytest.mark.parametrize("name", list(MODELS))
def test_realized_graph_is_integer_and_runs_on_reference(ref, b200, name):
    p = realized(ref, b200, MODELS[name]())
    doc = p["R"].to_json()
    ops = [nd["op"] for nd in doc["nodes"]]
    assert "simulated_quantize" not in ops
    assert "quantize" in ops and "requantize" in ops
    # pow2 thresholds: every requantize is an exact power-of-two rescale
    for nd in doc["nodes"]:
        if nd["op"] == "requantize":
            assert nd["attrs"]["multiplier"] == 1 << 30, nd
    Rr = p["R"].copy_to(ref)
    agree = 0
    for x in p["data"]:
        y, dt = ref.eval_int(Rr, x)
        yf = ref.eval_fp32(p["sim"], x, p["ev"].bind(p["cand"]))
        agree += int(np.argmax(y) == np.argmax(yf))
    # the integer graph reproduces the simulated graph's decisions
    assert agree >= len(p["data"]) - 1


@pytest.mark.parametrize("spec_name", ["x86_vnni_like", "arm_vmlal_like"])
def test_realize_other_specs_run_on_reference(ref, b200, spec_name):
    p = realized(ref, b200, F.small_cnn(), spec_name=spec_name, n=2)
    Rr = p["R"].copy_to(ref)
    y, dt = ref.eval_int(Rr, p["data"][0])
    assert y.size > 0
