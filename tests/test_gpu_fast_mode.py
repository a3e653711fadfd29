"""The reference's DEFAULT thresholds (ThresholdConfig.pow2 = false,
calibration.hpp:71-76) give non-power-of-two scales.  Under them:

* engine `auto` (default) runs the exact FP64 engine: bit-identical to the
  reference (every partial sum of the double accumulator reproduced in order);
* engine `fast` runs the fused int8 tcgen05 engine with fp32 epilogue math.
  Its integer GEMM sums q_x*q_w exactly, but the reference accumulates
  fl32(q_x*s_x) * fl32(q_w*s_w) in double, so a value sitting on a rounding
  boundary can land one code away.  STATED TOLERANCE (checked here on C1 and
  a ResNet-18 C2 slice): per candidate |loss_fast - loss_ref| <= 2/N; at the
  8-bit candidate (all_hi) top-1 predictions agree with the reference on
  >= 95% of the samples (at 4-6 bits a deep network's scores are dominated by
  quantization noise and one-code differences reorder near-ties, so only the
  loss is bounded there).  Greedy search: the same strategy on C1.  On C2
  the per-candidate bound holds on every candidate the reference greedy
  visits, but NOT the search result: one sample (1/N = 0.0625 at N = 16) is
  larger than the greedy tolerance, so a single flipped comparison changes
  the walk (measured: the fast strategy re-scored by the reference lands at
  loss 0.69 vs 0.44).  Strategy identity needs engine `auto` (exact)."""
import numpy as np
import pytest

from paper_2103_14949_b200 import fixtures as F

pytestmark = pytest.mark.gpu


def _pipe(q, model, data, method):
    g = q.graph(model.doc, model.blob)
    spec = q.parse_spec(F.spec_fixture("int8_int32"))
    topo = q.generate_topology(g, spec)
    sim = q.insert_simulated_quantize(g, topo)
    ds = q.dataset(data)
    st = q.collect_stats(g, ds, 2048, q.simulated_edge_indices(g, topo))
    thr = st.estimate_thresholds(method, quantile=0.99, kl_bits=8, pow2=False)
    return sim, ds, q.evaluator(sim, spec, topo, thr, st, ds), thr


@pytest.fixture
def fast_mode(cuda_lib):
    cuda_lib.set_engine_mode("fast")
    yield
    cuda_lib.set_engine_mode("auto")


@pytest.mark.parametrize("which", ["c1", "c2"])
def test_fast_mode_tolerance_vs_reference(b200, ref, fast_mode, which):
    if which == "c1":
        model, n, method = F.small_cnn(), 16, "kl"
    else:
        model, n, method = F.resnet(18, image=64, classes=100), 16, "quantile"
    data = model.data(n)
    sb, db, eb, tb = _pipe(b200, model, data, method)
    sr, dr, er, tr = _pipe(ref, model, data, method)
    assert tb == tr  # thresholds are host math on bit-identical statistics
    sp = eb.space()
    rng = np.random.default_rng(5)
    cands = [sp.all_hi(), sp.all_lo()] + [
        [int(rng.integers(lo, hi + 1)) for lo, hi in zip(sp.lo, sp.hi)] for _ in range(4)]
    # the fast engine really runs (non-pow2 scales are accepted in fast mode)
    assert b200.fused_status(sb, eb.bind(cands[0])) == ""
    lf, lr = eb.losses(cands), er.losses(cands)
    assert np.max(np.abs(lf - lr)) <= 2.0 / n + 1e-12, (lf, lr)
    c = sp.all_hi()
    pf = b200.predict_top1(sb, db, binding=eb.bind(c))
    pr = ref.predict_top1(sr, dr, binding=er.bind(c))
    assert np.mean(pf == pr) >= 0.95
    gr = ref.search("greedy", er.space(), evaluator=er, rounds=1, tol=0.02)
    if which == "c1":
        gf = b200.search("greedy", sp, evaluator=eb, rounds=1, tol=0.02)
        assert list(gf.best) == list(gr.best)
    else:
        visited = [rec[1] for rec in gr.trace["records"]]
        lv = eb.losses(visited)
        lrv = np.array([rec[2] for rec in gr.trace["records"]])
        assert np.max(np.abs(lv - lrv)) <= 2.0 / n + 1e-12
