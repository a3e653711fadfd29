"""Host-side parity on CPU: the B200 build's graph IR, hardware spec,
topology (Algorithm 1), simulated_quantize insertion and the four search
algorithms must reproduce the reference exactly — same canonical edge index,
same node ids, same decisions, same traces.  These run without a GPU (the
B200 library's host layers never touch the device)."""
import json

import numpy as np
import pytest

from paper_2103_14949_b200 import fixtures as F
from paper_2103_14949_b200 import quantc as Q

MODELS = {
    "small_cnn": lambda: F.small_cnn(),
    "chain": lambda: F.conv_add_pool_chain(),
    "resnet18": lambda: F.resnet(18, image=64, classes=10, width=8),
    "resnet50": lambda: F.resnet(50, image=64, classes=10, width=8),
    "deep_chain": lambda: F.deep_chain(20),
}


@pytest.mark.parametrize("name", list(MODELS))
@pytest.mark.parametrize("spec_name", list(F.SPECS))
def test_graph_topology_insertion_identical(b200, ref, name, spec_name):
    m = MODELS[name]()
    ga, gr = b200.graph(m.doc, m.blob), ref.graph(m.doc, m.blob)
    assert ga.validate() == gr.validate() == []
    assert ga.traversal_order() == gr.traversal_order()
    assert ga.edge_order() == gr.edge_order()
    sa, sr = b200.parse_spec(F.spec_fixture(spec_name)), ref.parse_spec(F.spec_fixture(spec_name))
    assert sa.serialize() == sr.serialize()
    try:
        tr = ref.generate_topology(gr, sr)
    except Q.TopologyError as e:
        with pytest.raises(Q.TopologyError) as ei:
            b200.generate_topology(ga, sa)
        assert str(ei.value) == str(e)
        return
    ta = b200.generate_topology(ga, sa)
    assert ta.dump() == tr.dump()
    assert ta.qv() == tr.qv()
    assert b200.simulated_edge_indices(ga, ta) == ref.simulated_edge_indices(gr, tr)
    assert b200.searchable_edge_indices(ta) == ref.searchable_edge_indices(tr)
    sima, simr = b200.insert_simulated_quantize(ga, ta), ref.insert_simulated_quantize(gr, tr)
    assert sima.to_json() == simr.to_json()
    assert sima.traversal_order() == simr.traversal_order()
    assert sima.validate() == simr.validate() == []


def test_spec_errors_identical(b200, ref):
    bad = [
        '{"ops": {"conv2d": [{"in": ["int8"], "out": "int32"}]}}',
        '{"ops": {"foo": [{"in": ["int8"], "out": "int32"}]}}',
        '{"ops": {"relu": [{"in": ["int7"], "out": "int32"}]}}',
        '{"ops": {"relu": [{"in": ["int8"], "out": "int8"}, {"in": ["int8"], "out": "int8"}]}}',
        '{"ops": {"relu": []}}',
        '[1, 2]',
        'not json',
    ]
    for text in bad:
        with pytest.raises(Q.SpecError) as er:
            ref.parse_spec(text)
        with pytest.raises(Q.SpecError) as ea:
            b200.parse_spec(text)
        if text != "not json":  # parser message text embeds nlohmann details
            assert str(ea.value) == str(er.value)
    assert b200.parse_spec("{}").classify_op("conv2d") == "float_only"


def test_fig3_spec_classification_and_matching(b200, ref):
    for q in (b200, ref):
        s = q.parse_spec(F.spec_fixture("fig3"))
        assert s.classify_op("global_avg_pool2d") == "float_only"
        assert s.classify_op("conv2d") == "integer_only"
        assert s.classify_op("add") == "mixed"
        assert s.candidate_dtypes("conv2d", 0) == ["int8", "int16"]
    for bits in ([8, 8], [6, 8], [9, 8], [16, 16], [17, 4]):
        for signs in ([1, 1], [0, 1]):
            ma = b200.parse_spec(F.spec_fixture("fig3")).match_signature("conv2d", bits, signs)
            mr = ref.parse_spec(F.spec_fixture("fig3")).match_signature("conv2d", bits, signs)
            assert ma == mr
    arm = b200.parse_spec(F.spec_fixture("arm_vmlal_like"))
    assert arm.match_signature("conv2d", [8, 8], [1, 1]) == (["int8", "int8"], "int16")
    assert arm.match_signature("conv2d", [9, 8], [1, 1]) == (["int16", "int16"], "int32")


def test_fig4_topology(b200):
    """SPEC acceptance 2: conv2d -> add -> global_avg_pool2d with the Fig. 3
    spec -> qv = {conv2d, add}, nqv = {global_avg_pool2d}."""
    m = F.conv_add_pool_chain()
    g = b200.graph(m.doc, m.blob)
    t = b200.generate_topology(g, b200.parse_spec(F.spec_fixture("fig3")))
    ops = {n["id"]: n["op"] for n in m.doc["nodes"]}
    q_ops = sorted(ops[i] for i in t.qv() if ops[i] not in ("input", "constant"))
    assert q_ops == ["add", "conv2d"]
    assert t.dump()["vertices"][str([i for i, o in ops.items() if o == "global_avg_pool2d"][0])] == "float"


def _space(n, lo=4, hi=8):
    return Q.SearchSpace(list(range(n)), [lo] * n, [hi] * n)


LOSSES = {
    "separable": lambda opt: (lambda c: float(sum(0.0 if b >= o else 1.0 + (o - b)
                                                  for b, o in zip(c, opt)))),
    "coupled": lambda opt: (lambda c: float(abs(c[0] - c[1]) * 0.1 + sum((b - o) ** 2 * 0.01
                                                                        for b, o in zip(c, opt)))),
    "constant": lambda opt: (lambda c: 0.5),
}


@pytest.mark.parametrize("loss_name", list(LOSSES))
def test_search_algorithms_identical(b200, ref, loss_name):
    opt = [6, 5, 7]
    loss = LOSSES[loss_name](opt)
    sp = _space(3)
    runs = [("greedy", dict(rounds=2, tol=0.0)), ("greedy", dict(rounds=1, tol=0.01)),
            ("anneal", dict(steps=300, t0=0.1, decay=0.99, seed=5)),
            ("random", dict(n=40, seed=9)), ("exhaustive", dict(cap=1000))]
    for method, kw in runs:
        ra = b200.search(method, sp, loss=loss, **kw)
        rr = ref.search(method, sp, loss=loss, **kw)
        assert (ra.best, ra.best_loss, ra.evaluations) == (rr.best, rr.best_loss, rr.evaluations)
        assert ra.trace == rr.trace
    if loss_name == "separable":
        ex = b200.search("exhaustive", sp, loss=loss, cap=1000)
        # strict acceptance never leaves all_hi on a flat loss;
        # a tolerance walks each edge down to its lossless optimum
        assert b200.search("greedy", sp, loss=loss, rounds=1).best == sp.all_hi()
        gr = b200.search("greedy", sp, loss=loss, rounds=1, tol=0.5)
        assert ex.evaluations == 125 and gr.best == ex.best == opt  # SPEC acceptance 3


def test_search_errors_identical(b200, ref):
    sp = _space(3)
    for method, kw in [("greedy", dict(rounds=0)), ("anneal", dict(steps=0)),
                       ("anneal", dict(steps=3, t0=0.0)), ("anneal", dict(steps=3, decay=1.5)),
                       ("random", dict(n=0)), ("exhaustive", dict(cap=10))]:
        with pytest.raises(Q.SearchError) as er:
            ref.search(method, sp, loss=lambda c: 0.0, **kw)
        with pytest.raises(Q.SearchError) as ea:
            b200.search(method, sp, loss=lambda c: 0.0, **kw)
        assert str(ea.value) == str(er.value)


def test_space_size(b200, ref):
    assert b200.space_size(_space(3)) == ref.space_size(_space(3)) == 125
    big = Q.SearchSpace(list(range(118)), [4] * 118, [8] * 118)
    assert b200.space_size(big) == ref.space_size(big) == 5 ** 118 > 4 ** 118  # SPEC accept. 9
    wide = Q.SearchSpace(list(range(40)), [4] * 40, [32] * 40)
    assert b200.space_size(wide) == 29 ** 40


def test_graph_errors_identical(b200, ref):
    m = F.small_cnn()
    doc = json.loads(json.dumps(m.doc))
    doc["edges"].append({"src": [99, 0], "dst": [2, 5]})
    ra = b200.graph(doc, m.blob).validate()
    rr = ref.graph(doc, m.blob).validate()
    assert ra == rr and ra
    cyc = {"nodes": [{"id": 0, "op": "input", "attrs": {"name": "x", "shape": [1, 4]}},
                     {"id": 1, "op": "relu", "attrs": {}}, {"id": 2, "op": "relu", "attrs": {}}],
           "edges": [{"src": [1, 0], "dst": [2, 0]}, {"src": [2, 0], "dst": [1, 0]}],
           "inputs": [0], "outputs": [[2, 0]]}
    assert b200.graph(cyc).validate() == ref.graph(cyc).validate()
    with pytest.raises(Q.GraphError) as ea:
        b200.graph(cyc).traversal_order()
    with pytest.raises(Q.GraphError) as er:
        ref.graph(cyc).traversal_order()
    assert str(ea.value) == str(er.value)
