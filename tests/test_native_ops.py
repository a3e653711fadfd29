"""Op-set extension, host side and oracle pinning.

The reference op set is closed (graph.hpp:20-37, graph.cpp:17-35; conv2d has
no groups, interpreter.cpp:196-236).  This repo adds conv2d `groups`,
avg_pool2d and concat with the semantics of their exact rewrites into the
reference op set (fixtures.py).  The checker is tests/oracle_graph.py, a
graph interpreter on the C restatement; here it is pinned to the compiled
reference on the rewritten graphs (fp32 and sim-quant under the reference's
own bindings), and shown equal on the native and rewritten forms."""
import json

import numpy as np
import pytest

from paper_2103_14949_b200 import fixtures as F
from paper_2103_14949_b200 import quantc as Q
from tests import oracle_graph

MNV2 = [(1, 16, 1, 1), (6, 24, 2, 2)]


def _models():
    return [(F.mobilenet_v2(blocks=MNV2), F.mobilenet_v2(blocks=MNV2, native=True)),
            (F.inception_v3(modules=1, image=29, width=4),
             F.inception_v3(modules=1, image=29, width=4, native=True))]


@pytest.mark.parametrize("k", [0, 1])
def test_oracle_graph_pinned_fp32_and_native_equal(ref, port, k):
    rw, nat = _models()[k]
    x = rw.data(2)
    for i in range(2):
        y_ref = ref.eval_fp32(ref.graph(rw.doc, rw.blob), x[i]).reshape(-1)
        y_rw = oracle_graph.GraphOracle(port, rw.doc, rw.blob).run(x[i]).reshape(-1)
        y_nat = oracle_graph.GraphOracle(port, nat.doc, nat.blob).run(x[i]).reshape(-1)
        assert y_ref.tobytes() == y_rw.tobytes()
        assert y_rw.tobytes() == y_nat.tobytes()


def test_oracle_graph_pinned_simquant(ref, port):
    """Sim-quant forward under the reference evaluator's own bindings: the
    oracle's scores and predictions equal the reference's predict_top1."""
    rw = F.mobilenet_v2(blocks=MNV2)
    data = rw.data(4)
    g = ref.graph(rw.doc, rw.blob)
    spec = ref.parse_spec(F.spec_fixture("arm_vmlal_like"))
    topo = ref.generate_topology(g, spec)
    sim = ref.insert_simulated_quantize(g, topo)
    ds = ref.dataset(data)
    st = ref.collect_stats(g, ds, 2048, ref.simulated_edge_indices(g, topo))
    thr = st.estimate_thresholds("quantile", quantile=0.999, pow2=True)
    ev = ref.evaluator(sim, spec, topo, thr, st, ds, min_bit=8)
    sp = ev.space()
    orc = oracle_graph.GraphOracle(port, sim.to_json(), sim.blob())
    for cand in (sp.all_hi(), sp.all_lo()):
        bnd = ev.bind(cand)
        want = ref.predict_top1(sim, ds, binding=bnd)
        got, _ = orc.predict(data.reshape(-1, *data.shape[2:]), bnd)
        np.testing.assert_array_equal(got, want)


def test_native_graph_validation(b200):
    nat = F.mobilenet_v2(blocks=MNV2, native=True)
    assert b200.graph(nat.doc, nat.blob).validate() == []
    gb = F.GraphBuilder()
    x = gb.input("data", [1, 6, 8, 8])
    w = gb.constant(np.zeros((4, 3, 3, 3), np.float32))
    gb.output(gb.op("conv2d", [x, w], strides=[1, 1], padding=[1, 1], groups=2))
    doc, blob = gb.build()
    assert b200.graph(doc, blob).validate() == []
    bad = json.loads(json.dumps(doc))
    bad["nodes"][-1]["attrs"]["groups"] = 4  # does not divide O = 4 x (C/G = 3) channels
    assert any("groups" in v["message"] or "channel" in v["message"]
               for v in b200.graph(bad, blob).validate())
    gb = F.GraphBuilder()
    a = gb.input("a", [1, 2, 4, 4])
    b = gb.input("b", [1, 3, 5, 5])
    gb.output(gb.op("concat", [a, b], axis=1))
    doc, blob = gb.build()
    assert any("concat" in v["message"] for v in b200.graph(doc, blob).validate())
    gb = F.GraphBuilder()
    a = gb.input("a", [1, 2, 4, 4])
    gb.output(gb.op("avg_pool2d", [a], pool_size=[3, 3], strides=[1, 1], padding=[1, 1]))
    doc, blob = gb.build()
    assert b200.graph(doc, blob).validate() == []


def test_native_ops_are_float_only_in_topology(b200):
    """concat / avg_pool2d have no spec signatures: Algorithm 1 keeps them in
    fp32 (nqv) and places boundary sqs around them; grouped convs are MAC ops
    like conv2d."""
    nat = F.inception_v3(modules=1, image=29, width=4, native=True)
    g = b200.graph(nat.doc, nat.blob)
    spec = b200.parse_spec(F.spec_fixture("int8_int32"))
    assert spec.classify_op("concat") == "float_only"
    assert spec.classify_op("avg_pool2d") == "float_only"
    sim = b200.insert_simulated_quantize(g, b200.generate_topology(g, spec))
    ops = [n["op"] for n in sim.to_json()["nodes"]]
    assert ops.count("concat") == 4 and ops.count("avg_pool2d") == 1
    mn = F.mobilenet_v2(blocks=MNV2, native=True)
    gm = b200.graph(mn.doc, mn.blob)
    topo = b200.generate_topology(gm, b200.parse_spec(F.spec_fixture("arm_vmlal_like")))
    dw = [n["id"] for n in mn.doc["nodes"] if n["attrs"].get("groups", 1) > 1]
    assert dw and all(i in topo.qv() for i in dw)
