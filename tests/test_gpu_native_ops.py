"""Op-set extension on the GPU: conv2d `groups`
(depthwise), avg_pool2d and concat run natively in the exact engine
(kernels/conv_f64.cu grouped GEMM + direct kernel, eltwise.cu avgpool /
concat).  Checked against

* the C restatement (array level, byte-exact),
* the compiled reference on the exactly rewritten graphs (fp32 outputs), and
* the graph oracle (tests/oracle_graph.py, pinned to the reference in
  test_native_ops.py) for calibration statistics and the sim-quant forward
  under the B200 evaluator's own bindings (C3 MobileNetV2 arm_vmlal_like,
  C5 Inception-v3 int8_int32)."""
import numpy as np
import pytest
import torch

from paper_2103_14949_b200 import fixtures as F
from tests import oracle_graph

pytestmark = pytest.mark.gpu

MNV2 = [(1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 2, 2)]


@pytest.mark.parametrize("n,c,h,o,k,s,p,g", [
    (2, 16, 9, 16, 3, 1, 1, 16),    # depthwise
    (2, 24, 10, 24, 3, 2, 1, 24),   # depthwise stride 2
    (1, 8, 7, 16, 3, 1, 1, 8),      # channel multiplier 2 (direct kernel)
    (2, 64, 6, 96, 3, 1, 1, 2),     # two groups through the GEMM kernel
    (1, 32, 5, 64, 1, 1, 0, 4),     # grouped 1x1
])
def test_grouped_conv_kernel_vs_port(cuda_lib, port, n, c, h, o, k, s, p, g):
    rng = np.random.default_rng(n * 1000 + c + g)
    x = rng.standard_normal((n, c, h, h)).astype(np.float32)
    w = rng.standard_normal((o, c // g, k, k)).astype(np.float32)
    b = rng.standard_normal(o).astype(np.float32)
    want = port.conv2d(x, w, b, (s, s), (p, p), groups=g)
    got = cuda_lib.conv2d_grouped_f64acc(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(),
                                         torch.from_numpy(b).cuda(), (s, s), (p, p), g)
    assert got.cpu().numpy().tobytes() == want.tobytes()


@pytest.mark.parametrize("k,s,p", [(3, 1, 1), (3, 2, 1), (2, 2, 0), (5, 1, 2)])
def test_avg_pool_kernel_vs_port(cuda_lib, port, k, s, p):
    x = np.random.default_rng(k + s).standard_normal((2, 5, 11, 11)).astype(np.float32)
    want = port.avg_pool2d(x, (k, k), (s, s), (p, p))
    got = cuda_lib.avg_pool2d(torch.from_numpy(x).cuda(), (k, k), (s, s), (p, p))
    assert got.cpu().numpy().tobytes() == want.tobytes()


def _pair(which):
    if which == "c5gap":
        # the bench's C5 layout: two modules (module 2 pools the concat of
        # module 1 directly) and a GAP head
        return (F.inception_v3(modules=2, image=35, width=4, head="gap"),
                F.inception_v3(modules=2, image=35, width=4, head="gap", native=True))
    if which == "c3":
        return F.mobilenet_v2(blocks=MNV2), F.mobilenet_v2(blocks=MNV2, native=True)
    return (F.inception_v3(modules=1, image=29, width=4),
            F.inception_v3(modules=1, image=29, width=4, native=True))


@pytest.mark.parametrize("which", ["c3", "c5"])
def test_native_fp32_equals_reference_on_rewrite(b200, ref, which):
    rw, nat = _pair(which)
    x = rw.data(3)
    for i in range(3):
        want = ref.eval_fp32(ref.graph(rw.doc, rw.blob), x[i])
        got = b200.eval_fp32(b200.graph(nat.doc, nat.blob), x[i])
        assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("which,spec_name", [("c3", "arm_vmlal_like"), ("c5", "int8_int32")])
def test_native_pipeline_vs_graph_oracle(b200, port, which, spec_name):
    _, nat = _pair(which)
    data = nat.data(6)
    xs = data.reshape(-1, *data.shape[2:])
    g = b200.graph(nat.doc, nat.blob)
    spec = b200.parse_spec(F.spec_fixture(spec_name))
    topo = b200.generate_topology(g, spec)
    sim = b200.insert_simulated_quantize(g, topo)
    ds = b200.dataset(data)
    edges = b200.simulated_edge_indices(g, topo)
    st = b200.collect_stats(g, ds, 2048, edges)
    # statistics: min / max / absmax and the 2048-bin histogram of every edge
    _, vals = oracle_graph.GraphOracle(port, nat.doc, nat.blob).run(xs, values=True)
    order = g.edge_order()
    consts = {n["id"] for n in nat.doc["nodes"] if n["op"] == "constant"}
    for k in edges:
        src = order[k][0]
        v = vals[src].astype(np.float64)
        e = st.get(k)
        assert (e["min"], e["max"]) == (v.min(), v.max()), k
        # the reference histograms every edge once per sample
        # (calibration.cpp:95-105): a constant's counts scale with N
        want = port.histogram(vals[src], e["absmax"], 2048) * (len(xs) if src in consts else 1)
        np.testing.assert_array_equal(e["counts"], want, err_msg=f"edge {k}")
    thr = st.estimate_thresholds("quantile", quantile=0.999, pow2=True)
    ev = b200.evaluator(sim, spec, topo, thr, st, ds, min_bit=8)
    sp = ev.space()
    orc = oracle_graph.GraphOracle(port, sim.to_json(), sim.blob())
    rng = np.random.default_rng(3)
    cands = [sp.all_hi(), sp.all_lo()] + [
        [int(rng.integers(lo, hi + 1)) for lo, hi in zip(sp.lo, sp.hi)] for _ in range(2)]
    refs, _ = oracle_graph.GraphOracle(port, nat.doc, nat.blob).predict(xs)
    np.testing.assert_array_equal(ev.reference_predictions(), refs)
    losses = ev.losses(cands)
    for c, loss in zip(cands, losses):
        bnd = ev.bind(c)
        want, scores = orc.predict(xs, bnd)
        np.testing.assert_array_equal(b200.predict_top1(sim, ds, binding=bnd), want)
        got = b200.predict_scores(sim, ds, binding=bnd)
        assert got.reshape(scores.shape).tobytes() == scores.tobytes()
        assert loss == 1.0 - float(np.sum(want == refs)) / len(refs)


@pytest.mark.parametrize("which,spec_name,min_bit", [("c3", "arm_vmlal_like", 4), ("c3", "int8_int32", 4),
                                                    ("c5", "int8_int32", 4), ("c5gap", "int8_int32", 4)])
def test_native_ops_on_fused_engine(b200, cuda_lib, which, spec_name, min_bit):
    """Native graphs under power-of-two thresholds run on the fused engine —
    C3 MobileNetV2's depthwise convs as a CUDA-core stage of int8 codes
    (fastplan Stage::kDw), C5 Inception's avg_pool2d over codes (Stage::kAvg)
    and concat as fp32 column placement plus one stage over the concatenated
    value (Stage::kCat) — and reproduce the exact FP64 engine, itself pinned
    to the reference on the rewritten graph, bit for bit: fp32 score bytes
    and losses of mixed-bit candidates."""
    _, nat = _pair(which)
    data = nat.data(6)
    g = b200.graph(nat.doc, nat.blob)
    spec = b200.parse_spec(F.spec_fixture(spec_name))
    topo = b200.generate_topology(g, spec)
    sim = b200.insert_simulated_quantize(g, topo)
    ds = b200.dataset(data)
    st = b200.collect_stats(g, ds, 2048, b200.simulated_edge_indices(g, topo))
    thr = st.estimate_thresholds("quantile", quantile=0.999, pow2=True)
    ev = b200.evaluator(sim, spec, topo, thr, st, ds, min_bit=min_bit)
    sp = ev.space()
    rng = np.random.default_rng(3)
    # the fused engine materialises int8 codes: bit widths <= 8 (for
    # arm_vmlal_like that binds the (i8, i8) -> i16 accumulation signature)
    his = [min(hi, 8) for hi in sp.hi]
    cands = [his, sp.all_lo()] + [
        [int(rng.integers(lo, hi + 1)) for lo, hi in zip(sp.lo, his)] for _ in range(4)]
    assert b200.fused_status(sim, ev.bind(cands[0])) == ""
    cuda_lib.set_engine_mode("exact")
    try:
        exact = ev.losses(cands)
        s_exact = [b200.predict_scores(sim, ds, ev.bind(c)) for c in cands[:3]]
    finally:
        cuda_lib.set_engine_mode("auto")
    f0 = cuda_lib.counters()["fused_batches"]
    fused = ev.losses(cands)
    assert cuda_lib.counters()["fused_batches"] - f0 >= len(cands)
    np.testing.assert_array_equal(exact, fused)
    for c, se in zip(cands[:3], s_exact):
        assert b200.predict_scores(sim, ds, ev.bind(c)).tobytes() == se.tobytes()
