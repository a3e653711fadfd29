"""BASELINE configs C3 and C5 as parity tests (bench.py measures C2/R50):

* C3 — MobileNetV2 under the ARM-style arm_vmlal_like spec ((i8, i8) -> i16
  and (i16, i16) -> i32 accumulation): calibration statistics, thresholds,
  losses and the greedy strategy, B200 vs the reference.
* C5 — Inception-v3-style strategy search: random and greedy search over
  bit-width candidates, B200 vs the reference.

Depthwise conv, concat and avg_pool are exact rewrites into the reference op
set (fixtures.py), so the unmodified reference runs the same graphs."""
import numpy as np
import pytest

from paper_2103_14949_b200 import fixtures as F

pytestmark = pytest.mark.gpu

MNV2_BLOCKS = [(1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 2, 2)]


def _pipe(q, model, data, spec_name, method="quantile", min_bit=4):
    g = q.graph(model.doc, model.blob)
    spec = q.parse_spec(F.spec_fixture(spec_name))
    topo = q.generate_topology(g, spec)
    sim = q.insert_simulated_quantize(g, topo)
    ds = q.dataset(data)
    edges = q.simulated_edge_indices(g, topo)
    st = q.collect_stats(g, ds, 2048, edges)
    thr = st.estimate_thresholds(method, quantile=0.999, kl_bits=8, pow2=False)
    ev = q.evaluator(sim, spec, topo, thr, st, ds, min_bit=min_bit)
    return dict(edges=edges, st=st, thr=thr, ev=ev)


def _same_stats(a, r):
    assert a["edges"] == r["edges"]
    for k in r["edges"]:
        ea, er = a["st"].get(k), r["st"].get(k)
        assert (ea["min"], ea["max"], ea["absmax"]) == (er["min"], er["max"], er["absmax"]), k
        np.testing.assert_array_equal(ea["counts"], er["counts"], err_msg=f"edge {k}")
    assert a["thr"] == r["thr"]


@pytest.fixture(scope="module")
def c3(b200, ref):
    m = F.mobilenet_v2(blocks=MNV2_BLOCKS)
    data = m.data(6)
    return _pipe(b200, m, data, "arm_vmlal_like", min_bit=14), \
        _pipe(ref, m, data, "arm_vmlal_like", min_bit=14)


def test_c3_mobilenet_arm_statistics_and_thresholds(c3):
    a, r = c3
    _same_stats(a, r)


def test_c3_mobilenet_arm_losses(c3):
    a, r = c3
    sp = r["ev"].space()
    rng = np.random.default_rng(3)
    cands = [sp.all_hi(), sp.all_lo()] + [
        [int(rng.integers(lo, hi + 1)) for lo, hi in zip(sp.lo, sp.hi)] for _ in range(4)]
    assert a["ev"].losses(cands).tolist() == r["ev"].losses(cands).tolist()
    for c in cands[:2]:
        assert a["ev"].strategy_for(c) == r["ev"].strategy_for(c)


def test_c3_mobilenet_arm_greedy_strategy(b200, ref, c3):
    a, r = c3
    ra = b200.search("greedy", a["ev"].space(), evaluator=a["ev"], rounds=1, tol=0.2)
    rr = ref.search("greedy", r["ev"].space(), evaluator=r["ev"], rounds=1, tol=0.2)
    assert (ra.best, ra.best_loss, ra.evaluations) == (rr.best, rr.best_loss, rr.evaluations)
    assert a["ev"].strategy_for(ra.best) == r["ev"].strategy_for(rr.best)


@pytest.fixture(scope="module")
def c5(b200, ref):
    m = F.inception_v3(modules=1, image=29, width=4)
    data = m.data(6)
    return _pipe(b200, m, data, "int8_int32", min_bit=4), \
        _pipe(ref, m, data, "int8_int32", min_bit=4)


def test_c5_inception_statistics_and_thresholds(c5):
    a, r = c5
    _same_stats(a, r)


@pytest.mark.parametrize("method,kw", [("random", dict(n=12, seed=5)),
                                       ("anneal", dict(steps=12, seed=2, t0=0.05)),
                                       ("greedy", dict(rounds=1, tol=0.1))])
def test_c5_inception_search_identical(b200, ref, c5, method, kw):
    a, r = c5
    ra = b200.search(method, a["ev"].space(), evaluator=a["ev"], **kw)
    rr = ref.search(method, r["ev"].space(), evaluator=r["ev"], **kw)
    assert (ra.best, ra.best_loss, ra.evaluations) == (rr.best, rr.best_loss, rr.evaluations)
    assert ra.trace == rr.trace
