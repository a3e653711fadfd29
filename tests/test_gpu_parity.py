"""GPU parity: the B200 implementation vs the reference oracle on identical
inputs, through the C ABI (include/quantc_capi.h) and the kernel ABI
(include/quantc_cuda.h).

Bar (BASELINE.json north_star): bit-exact for histogram counts, min/max,
integer outputs, predictions, losses and the selected strategy; KL values
within 1e-12 relative (log() may differ from glibc by 1 ulp); thresholds
bit-exact (they are absmax * i / B with the same integer i)."""
import numpy as np
import pytest
import torch

from paper_2103_14949_b200 import fixtures as F
from paper_2103_14949_b200 import quantc as Q

pytestmark = pytest.mark.gpu


def _pipeline(q, model, data, spec_name="int8_int32", method="quantile", pow2=False,
              quantile=0.999):
    g = q.graph(model.doc, model.blob)
    spec = q.parse_spec(F.spec_fixture(spec_name))
    topo = q.generate_topology(g, spec)
    sim = q.insert_simulated_quantize(g, topo)
    ds = q.dataset(data)
    edges = q.simulated_edge_indices(g, topo)
    st = q.collect_stats(g, ds, 2048, edges)
    thr = st.estimate_thresholds(method, quantile=quantile, kl_bits=8, pow2=pow2)
    ev = q.evaluator(sim, spec, topo, thr, st, ds)
    return dict(g=g, spec=spec, topo=topo, sim=sim, ds=ds, edges=edges, st=st, thr=thr, ev=ev)


@pytest.fixture(scope="module")
def small_cnn():
    m = F.small_cnn()
    return m, m.data(16)


def test_collect_stats_bit_exact(b200, ref, small_cnn):
    m, data = small_cnn
    a = _pipeline(b200, m, data)
    r = _pipeline(ref, m, data)
    assert a["edges"] == r["edges"]
    for k in r["edges"]:
        ea, er = a["st"].get(k), r["st"].get(k)
        assert ea["min"] == er["min"] and ea["max"] == er["max"], k
        assert ea["absmax"] == er["absmax"], k
        assert ea["sample_count"] == er["sample_count"]
        np.testing.assert_array_equal(ea["counts"], er["counts"], err_msg=f"edge {k}")


@pytest.mark.parametrize("method,pow2", [("max", False), ("quantile", False), ("kl", False),
                                         ("quantile", True), ("kl", True)])
def test_thresholds_and_losses_identical(b200, ref, small_cnn, method, pow2):
    m, data = small_cnn
    a = _pipeline(b200, m, data, method=method, pow2=pow2)
    r = _pipeline(ref, m, data, method=method, pow2=pow2)
    assert a["thr"] == r["thr"]
    np.testing.assert_array_equal(a["ev"].reference_predictions(),
                                  r["ev"].reference_predictions())
    sp = r["ev"].space()
    assert a["ev"].space() == sp
    rng = np.random.default_rng(0)
    cands = [sp.all_hi(), sp.all_lo()] + [
        [int(rng.integers(lo, hi + 1)) for lo, hi in zip(sp.lo, sp.hi)] for _ in range(6)]
    np.testing.assert_array_equal(a["ev"].losses(cands), r["ev"].losses(cands))
    for c in cands[:3]:
        assert a["ev"].bind(c).keys() == r["ev"].bind(c).keys()
        for k, p in r["ev"].bind(c).items():
            assert a["ev"].bind(c)[k].as_dict() == p.as_dict()
        assert a["ev"].strategy_for(c) == r["ev"].strategy_for(c)


def test_greedy_selects_identical_strategy(b200, ref, small_cnn):
    m, data = small_cnn
    out = []
    for q in (b200, ref):
        p = _pipeline(q, m, data, method="quantile", pow2=False)
        sp = p["ev"].space()
        res = q.search("greedy", sp, evaluator=p["ev"], rounds=2, tol=0.05)
        out.append((res.best, res.best_loss, res.evaluations, res.trace,
                    p["ev"].strategy_for(res.best)))
    assert out[0] == out[1]


def test_eval_fp32_resnet_block_bit_exact(b200, ref):
    m = F.resnet(18, image=32, classes=10, width=8)
    x = m.data(1)[0]
    ga, gr = b200.graph(m.doc, m.blob), ref.graph(m.doc, m.blob)
    ya, yr = b200.eval_fp32(ga, x), ref.eval_fp32(gr, x)
    assert ya.tobytes() == yr.tobytes()


def test_sim_quant_tensor_bit_exact(b200, ref):
    rng = np.random.default_rng(1)
    x = (rng.standard_normal(1 << 16) * rng.choice([0.01, 1, 100], 1 << 16)).astype(np.float32)
    for t, bit, sign, acc in [(1.0, 8, 1, Q.NONE), (0.37, 6, 1, Q.NONE), (3.3, 4, 1, Q.I16),
                              (2.0**-3, 8, 1, Q.I32), (5.0, 8, 0, Q.NONE)]:
        dt = Q.I8 if sign else Q.U8
        p = Q.QParams.make(t, bit, sign, dt, acc_dtype=acc, acc_scale=1e-3 if acc != Q.NONE else 0)
        if sign == 0:
            p.zero_point = 17
        assert b200.simulated_quantize(x, p).tobytes() == ref.simulated_quantize(x, p).tobytes()


def test_sim_quant_kernel_vs_port_many_tuples(cuda_lib, port):
    """SPEC acceptance 1: >= 10^4 (x, threshold, bit, sign) tuples, bit-exact."""
    rng = np.random.default_rng(2)
    for trial in range(40):
        t = float(np.exp(rng.uniform(-8, 8)))
        bit = int(rng.integers(2, 9))
        sign = int(rng.integers(0, 2))
        zp = 0 if sign else int(rng.integers(0, 1 << bit))
        x = (rng.standard_normal(4096) * t * rng.uniform(0.1, 3)).astype(np.float32)
        # near-tie values: exact half-integers of the grid
        s = t / 2.0 ** (bit - sign)
        x[:256] = ((rng.integers(-200, 200, 256) + 0.5) * s).astype(np.float32)
        p = Q.QParams.make(t, bit, sign, Q.I8 if sign else Q.U8, zero_point=zp)
        y = cuda_lib.sim_quant(torch.from_numpy(x).cuda(), p).cpu().numpy()
        expect = port.sim_quant(x, t, bit, sign, zp)
        assert y.tobytes() == expect.tobytes(), trial


def test_histogram_and_minmax_kernels(cuda_lib, port):
    rng = np.random.default_rng(3)
    x = rng.standard_normal(1_000_003).astype(np.float32)
    x[:5] = 0.0
    xt = torch.from_numpy(x).cuda()
    mm = cuda_lib.minmax(xt).cpu().numpy()
    assert mm[0] == float(x.min()) and mm[1] == float(x.max())
    absmax = max(abs(mm[0]), abs(mm[1]))
    for bins in (2048, 100, 7):
        c = cuda_lib.histogram(xt, absmax, bins).cpu().numpy()
        np.testing.assert_array_equal(c, port.histogram(x, absmax, bins))


def test_kl_sweep_kernel_matches_port(cuda_lib, port):
    rng = np.random.default_rng(4)
    hists = []
    for shape in range(12):
        if shape % 3 == 0:
            h = rng.integers(0, 1000, 2048)
        elif shape % 3 == 1:
            h = np.floor(1e6 * np.exp(-np.arange(2048) / rng.uniform(20, 400))).astype(np.int64)
        else:
            h = np.zeros(2048, np.int64)
            h[rng.integers(0, 2048, 50)] = rng.integers(1, 100, 50)
        hists.append(h)
    counts = torch.tensor(np.stack(hists), dtype=torch.int64).cuda()
    bi, bk = cuda_lib.kl_sweep(counts, 8)
    for e, h in enumerate(hists):
        i, kl = port.kl_best_index(h, 8)
        assert int(bi[e]) == i
        assert abs(float(bk[e]) - kl) <= 1e-12 * max(1.0, abs(kl))


def test_conv_f64_kernel_bit_exact(cuda_lib, port):
    rng = np.random.default_rng(5)
    for (N, Cc, H, W, O, K, s, pd) in [(2, 3, 17, 15, 16, 3, 1, 1), (1, 8, 12, 12, 70, 3, 2, 1),
                                       (3, 5, 9, 9, 130, 1, 1, 0), (1, 3, 30, 30, 8, 7, 2, 3)]:
        x = rng.standard_normal((N, Cc, H, W)).astype(np.float32)
        w = rng.standard_normal((O, Cc, K, K)).astype(np.float32)
        b = rng.standard_normal(O).astype(np.float32)
        y = cuda_lib.conv2d_f64acc(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(),
                                   torch.from_numpy(b).cuda(), (s, s), (pd, pd)).cpu().numpy()
        assert y.tobytes() == port.conv2d(x, w, b, (s, s), (pd, pd)).tobytes()


def test_tcgen05_gemm_exact_integer(cuda_lib):
    if not cuda_lib.tcgen05_available():
        pytest.fail("tcgen05 path not available on this device")
    rng = np.random.default_rng(6)
    for M, N, K in [(128, 64, 128), (300, 96, 256), (1000, 256, 640), (129, 300, 384)]:
        A = rng.integers(-128, 128, (M, K), dtype=np.int8)
        B = rng.integers(-128, 128, (N, K), dtype=np.int8)
        y = cuda_lib.gemm_s8(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), 1.0, None,
                             1).cpu().numpy().reshape(M, N)
        ref = A.astype(np.int64) @ B.astype(np.int64).T
        np.testing.assert_array_equal(y.astype(np.int64), ref)


def test_fast_engine_equals_exact_engine_pow2(b200, cuda_lib, small_cnn):
    """pow2 thresholds: tcgen05 int8 path is bit-identical to the FP64 path."""
    m, data = small_cnn
    p = _pipeline(b200, m, data, method="quantile", pow2=True)
    sp = p["ev"].space()
    cands = [sp.all_hi(), sp.all_lo(), [5] * len(sp.hi)]
    cuda_lib.set_engine_mode("exact")
    exact = p["ev"].losses(cands)
    g0 = cuda_lib.counters()["tcgen05_gemms"]
    cuda_lib.set_engine_mode("fast")
    fast = p["ev"].losses(cands)
    assert cuda_lib.counters()["tcgen05_gemms"] > g0
    cuda_lib.set_engine_mode("auto")
    np.testing.assert_array_equal(exact, fast)


@pytest.mark.parametrize("name,n", [("small_cnn", 16), ("resnet18", 8), ("resnet50", 4)])
def test_fused_engine_bit_exact_vs_exact_engine(b200, cuda_lib, name, n):
    """Engine v2 (fused NHWC int8 dataflow, tcgen05 implicit GEMM, fp32
    epilogue programs) must reproduce the FP64 exact engine bit for bit on
    power-of-two bindings: identical per-sample predictions and losses."""
    m = {"small_cnn": lambda: F.small_cnn(),
         "resnet18": lambda: F.resnet(18, image=64, classes=100),
         "resnet50": lambda: F.resnet(50, image=64, classes=100)}[name]()
    data = m.data(n)
    p = _pipeline(b200, m, data, method="quantile", pow2=True, quantile=0.99)
    sp = p["ev"].space()
    rng = np.random.default_rng(11)
    cands = [sp.all_hi(), sp.all_lo()] + [
        [int(rng.integers(lo, hi + 1)) for lo, hi in zip(sp.lo, sp.hi)] for _ in range(3)]
    cuda_lib.set_engine_mode("exact")
    exact = p["ev"].losses(cands)
    preds_exact = [b200.predict_top1(p["sim"], p["ds"], 0, p["ev"].bind(c)) for c in cands[:2]]
    cuda_lib.set_engine_mode("auto")
    f0 = cuda_lib.counters()["fused_batches"]
    fused = p["ev"].losses(cands)
    assert cuda_lib.counters()["fused_batches"] > f0, "fused engine was not used"
    preds_fused = [b200.predict_top1(p["sim"], p["ds"], 0, p["ev"].bind(c)) for c in cands[:2]]
    np.testing.assert_array_equal(exact, fused)
    for a, b in zip(preds_exact, preds_fused):
        np.testing.assert_array_equal(a, b)


def test_predict_top1_plan_cache(b200, ref, small_cnn):
    """predict_top1 keeps compiled plans resident across calls (keyed by
    graph identity): repeated and interleaved calls on two graphs, under
    several bindings, must still match the reference call for call."""
    m, data = small_cnn
    m2 = F.resnet(18, image=32, classes=10, width=8)
    data2 = m2.data(6)
    a, r = _pipeline(b200, m, data), _pipeline(ref, m, data)
    a2, r2 = _pipeline(b200, m2, data2), _pipeline(ref, m2, data2)
    sp, sp2 = r["ev"].space(), r2["ev"].space()
    cands = [sp.all_hi(), sp.all_lo(), sp.all_hi()]
    cands2 = [sp2.all_lo(), sp2.all_hi(), sp2.all_lo()]
    for c, c2 in zip(cands, cands2):
        np.testing.assert_array_equal(b200.predict_top1(a["sim"], a["ds"], 0, a["ev"].bind(c)),
                                      ref.predict_top1(r["sim"], r["ds"], 0, r["ev"].bind(c)))
        np.testing.assert_array_equal(b200.predict_top1(a2["sim"], a2["ds"], 0, a2["ev"].bind(c2)),
                                      ref.predict_top1(r2["sim"], r2["ds"], 0, r2["ev"].bind(c2)))
    # a graph rebuilt from the same document after the first is gone
    del a
    a3 = _pipeline(b200, m, data)
    np.testing.assert_array_equal(b200.predict_top1(a3["sim"], a3["ds"], 0, a3["ev"].bind(cands[1])),
                                  ref.predict_top1(r["sim"], r["ds"], 0, r["ev"].bind(cands[1])))


@pytest.mark.parametrize("name,n", [("small_cnn", 16), ("resnet18", 8), ("resnet50", 4)])
def test_fused_scores_bit_exact_vs_exact_engine(b200, cuda_lib, name, n):
    """Below the argmax: the fused engine's fp32 output rows (every class
    score) equal the FP64 exact engine's byte for byte, over bindings that mix
    bit-widths (so sq chains hit signed / non-negative / exact-ratio epilogue
    variants and half-way ties)."""
    m = {"small_cnn": lambda: F.small_cnn(),
         "resnet18": lambda: F.resnet(18, image=64, classes=100),
         "resnet50": lambda: F.resnet(50, image=64, classes=100)}[name]()
    data = m.data(n)
    p = _pipeline(b200, m, data, method="quantile", pow2=True, quantile=0.99)
    sp = p["ev"].space()
    rng = np.random.default_rng(21)
    cands = [sp.all_hi(), sp.all_lo()] + [
        [int(rng.integers(lo, hi + 1)) for lo, hi in zip(sp.lo, sp.hi)] for _ in range(4)]
    for c in cands:
        bnd = p["ev"].bind(c)
        cuda_lib.set_engine_mode("exact")
        exact = b200.predict_scores(p["sim"], p["ds"], bnd)
        cuda_lib.set_engine_mode("auto")
        f0 = cuda_lib.counters()["fused_batches"]
        fused = b200.predict_scores(p["sim"], p["ds"], bnd)
        assert cuda_lib.counters()["fused_batches"] > f0, "fused engine was not used"
        assert exact.shape == fused.shape
        assert exact.tobytes() == fused.tobytes(), (
            name, int((exact != fused).sum()), float(np.abs(exact - fused).max()))


def test_histogram_bin_edges_exact(cuda_lib, port):
    """Values on and one ulp around bin edges (the fp32 fast path defers
    these to the exact double binning): counts equal the restatement's."""
    rng = np.random.default_rng(31)
    for absmax, bins in [(6.0, 2048), (3.7, 2048), (1.0, 100), (0.001, 7)]:
        k = rng.integers(1, bins + 1, 20000)
        edge = (k * (absmax / bins)).astype(np.float32)
        x = np.concatenate([edge, np.nextafter(edge, np.float32(0)),
                            np.nextafter(edge, np.float32(np.inf)), -edge,
                            np.zeros(7, np.float32),
                            rng.uniform(-absmax, absmax, 50000).astype(np.float32)])
        x = np.clip(x, -absmax, absmax).astype(np.float32)
        c = cuda_lib.histogram(torch.from_numpy(x).cuda(), float(absmax), bins).cpu().numpy()
        np.testing.assert_array_equal(c, port.histogram(x, float(absmax), bins))


@pytest.mark.parametrize("name", ["small_cnn", "resnet18"])
def test_candidate_pairs_grouped_equal_single_calls(b200, cuda_lib, name):
    """losses(span) evaluates candidates two at a time through grouped tcgen05
    launches (FastPlan::predict_pair); every count must equal the one-
    candidate-per-call path."""
    model = F.small_cnn() if name == "small_cnn" else F.resnet(18, image=64, classes=10, width=16)
    p = _pipeline(b200, model, model.data(12), pow2=True)
    ev = p["ev"]
    sp = ev.space()
    rng = np.random.default_rng(11)
    cands = [sp.all_hi(), sp.all_lo()] + [
        [int(rng.integers(lo, hi + 1)) for lo, hi in zip(sp.lo, sp.hi)] for _ in range(7)]
    batched = ev.losses(cands).tolist()
    single = [ev.loss(c) for c in cands]
    assert batched == single


def _argmax_class(row):
    """Restatement of the reference argmax_class (interpreter.cpp:533-541)."""
    best = 0
    for i in range(1, len(row)):
        if row[i] > row[best]:
            best = i
    return best


@pytest.mark.parametrize("grouped", [0, 4])
def test_argmax_nan_and_ties_match_reference(cuda_lib, grouped):
    """NaN scores are never taken (except a NaN at index 0, which wins),
    ties keep the lowest index, +0 / -0 compare equal — per row, through the
    single and the grouped-candidate argmax kernels."""
    rng = np.random.default_rng(41)
    rows, cols = 64, 1000
    x = rng.standard_normal((rows, cols)).astype(np.float32)
    x[0, :] = np.nan                         # all NaN -> 0
    x[1, 0] = np.nan                         # NaN at 0 -> 0
    x[2, 5] = np.nan; x[2, 6] = 50.0         # NaN before the max
    x[3, :] = 1.0                            # all ties -> 0
    x[4, 700] = 9.0; x[4, 3] = 9.0           # tie -> lowest index
    x[5, :] = -np.inf; x[5, 900] = np.nan    # -inf everywhere -> 0
    x[6, :] = 0.0; x[6, 0] = -0.0; x[6, 17] = 0.0
    x[7, 1:] = np.nan                        # only index 0 is a number
    x[8, 999] = np.inf; x[8, 998] = np.nan
    x[9::7, rng.integers(0, cols, 8)] = np.nan  # scattered NaNs
    got = cuda_lib.argmax_rows(torch.from_numpy(x).cuda(), grouped=grouped).cpu().numpy()
    exp = np.array([_argmax_class(list(r)) for r in x])
    np.testing.assert_array_equal(got, exp)
