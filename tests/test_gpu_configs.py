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
from paper_2103_14949_b200 import quantc as Q

F_I16 = Q.I16

pytestmark = pytest.mark.gpu

MNV2_BLOCKS = [(1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 2, 2)]


def _pipe(q, model, data, spec_name, method="quantile", min_bit=4, pow2=False):
    g = q.graph(model.doc, model.blob)
    spec = q.parse_spec(F.spec_fixture(spec_name))
    topo = q.generate_topology(g, spec)
    sim = q.insert_simulated_quantize(g, topo)
    ds = q.dataset(data)
    edges = q.simulated_edge_indices(g, topo)
    st = q.collect_stats(g, ds, 2048, edges)
    thr = st.estimate_thresholds(method, quantile=0.999, kl_bits=8, pow2=pow2)
    ev = q.evaluator(sim, spec, topo, thr, st, ds, min_bit=min_bit)
    return dict(edges=edges, st=st, thr=thr, ev=ev, sim=sim, ds=ds)


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
def c3_i16acc(b200, ref):
    """C3 at <= 8 bits with power-of-two thresholds: every conv binds the
    (i8, i8) -> i16 signature, so each conv output's sq clamps to the int16
    accumulator range (acc_scale = s_x * s_w) — on the fused tcgen05 engine."""
    m = F.mobilenet_v2(blocks=MNV2_BLOCKS)
    data = m.data(6)
    return _pipe(b200, m, data, "arm_vmlal_like", min_bit=4, pow2=True), \
        _pipe(ref, m, data, "arm_vmlal_like", min_bit=4, pow2=True)


def test_c3_int16_accumulation_on_fused_engine(b200, ref, cuda_lib, c3_i16acc):
    a, r = c3_i16acc
    _same_stats(a, r)
    sp = r["ev"].space()
    rng = np.random.default_rng(5)
    cands = [[8] * len(sp.lo), sp.all_lo(), [6] * len(sp.lo)] + [
        [int(rng.integers(lo, 9)) for lo in sp.lo] for _ in range(5)]
    # the bound signature really is (i8, i8) -> i16 with an int16 accumulator clamp
    bnd = r["ev"].bind(cands[0])
    assert any(p.acc_dtype == F_I16 for p in bnd.values())
    why = b200.fused_status(a["sim"], a["ev"].bind(cands[0]))
    assert why == "", why
    f0 = cuda_lib.counters()["fused_batches"]
    la = a["ev"].losses(cands)
    assert cuda_lib.counters()["fused_batches"] - f0 >= len(cands), "fused engine not used"
    np.testing.assert_array_equal(la, r["ev"].losses(cands))
    for c in cands[:3]:
        assert a["ev"].strategy_for(c) == r["ev"].strategy_for(c)
        ba = a["ev"].bind(c)
        for k, p in r["ev"].bind(c).items():
            assert ba[k].as_dict() == p.as_dict()
    # below the argmax: the fused fp32 scores equal the FP64 exact engine's
    for c in cands[:4]:
        bd = a["ev"].bind(c)
        cuda_lib.set_engine_mode("exact")
        ex = b200.predict_scores(a["sim"], a["ds"], bd)
        cuda_lib.set_engine_mode("auto")
        fu = b200.predict_scores(a["sim"], a["ds"], bd)
        assert ex.tobytes() == fu.tobytes()


def test_c3_int16_accumulation_greedy(b200, ref, c3_i16acc):
    a, r = c3_i16acc
    ra = b200.search("greedy", a["ev"].space(), evaluator=a["ev"], rounds=1, tol=0.2)
    rr = ref.search("greedy", r["ev"].space(), evaluator=r["ev"], rounds=1, tol=0.2)
    assert (ra.best, ra.best_loss, ra.evaluations, ra.trace) == \
        (rr.best, rr.best_loss, rr.evaluations, rr.trace)
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


@pytest.fixture(scope="module")
def c5_pow2(b200, ref):
    m = F.inception_v3(modules=1, image=29, width=4)
    data = m.data(6)
    return _pipe(b200, m, data, "int8_int32", min_bit=4, pow2=True), \
        _pipe(ref, m, data, "int8_int32", min_bit=4, pow2=True)


def test_c5_inception_pow2_on_fused_engine(b200, ref, cuda_lib, c5_pow2):
    """C5 with power-of-two thresholds: the whole search evaluation runs on
    the fused tcgen05 engine and equals the reference."""
    a, r = c5_pow2
    _same_stats(a, r)
    sp = r["ev"].space()
    rng = np.random.default_rng(9)
    cands = [sp.all_hi(), sp.all_lo()] + [
        [int(rng.integers(lo, hi + 1)) for lo, hi in zip(sp.lo, sp.hi)] for _ in range(6)]
    why = b200.fused_status(a["sim"], a["ev"].bind(cands[0]))
    assert why == "", why
    f0 = cuda_lib.counters()["fused_batches"]
    np.testing.assert_array_equal(a["ev"].losses(cands), r["ev"].losses(cands))
    assert cuda_lib.counters()["fused_batches"] - f0 >= len(cands)
    ra = b200.search_batched("random", a["ev"].space(), evaluator=a["ev"], n=12, seed=5)
    rr = ref.search("random", r["ev"].space(), evaluator=r["ev"], n=12, seed=5)
    assert (ra.best, ra.best_loss, ra.evaluations, ra.trace) == \
        (rr.best, rr.best_loss, rr.evaluations, rr.trace)
