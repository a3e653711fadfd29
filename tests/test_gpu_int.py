"""GPU parity of the realized-graph integer path (SURVEY §8(a) conv2d/dense
int branches + requantize, reference interpreter.cpp:230-300 and :460-482):
the B200 eval_int — int8 x int8 -> int32 on tcgen05 with the zero-point /
bias / accumulator-clamp / requantize epilogue fused — against the
reference's own eval_int on the same graph, bit-exact, including the trap
mode's node / lowest flat index / value."""
import numpy as np
import pytest

from paper_2103_14949_b200 import fixtures as F
from paper_2103_14949_b200 import quantc as Q

pytestmark = pytest.mark.gpu

RQ = (1 << 30, 41, 7, -3)  # multiplier 2^30, shift 41, in_zp 7, out_zp -3
# general (non power-of-two) fixed-point multipliers, as requantize_params
# produces them for arbitrary scale ratios (SPEC.md realize module)
RQG = (1518500250, 41, 7, -3)        # ~ sqrt(1/2) * 2^31
RQG2 = (1900000001, 42, -5, 4)
RQG_MAX = (2147483647, 44, 1, -1)    # the largest multiplier

# case -> (probe config, backend that must run it: tc = tcgen05 kernel,
# simt = CUDA-core backend, generic = the int64 reference-order kernel)
CASES = {
    "3x3_pad": (dict(), "tc"),
    "3x3_zp0_pad": (dict(zp0=3, zp1=-2), "tc"),
    "3x3_rq": (dict(requant=RQ), "tc"),
    "3x3_zp_rq": (dict(zp0=-4, zp1=1, requant=RQ), "tc"),
    "u8_zp0_pad": (dict(dtype="uint8", zp0=100, requant=RQ), "tc"),
    "1x1": (dict(k=1, pad=0, c=64, o=40), "tc"),
    "1x1_s2": (dict(k=1, pad=0, stride=2, c=32, o=48, requant=RQ), "tc"),
    "3x3_s2": (dict(stride=2, c=24, o=20, h=15, w=15), "tc"),
    "7x7_s2": (dict(k=7, stride=2, pad=3, c=3, o=16, h=20, w=20), "tc"),
    "5x5_c200": (dict(k=5, pad=2, c=200, o=130, h=9, w=9, zp0=5, requant=RQ), "tc"),
    "dense": (dict(dense=True, c=300, o=70, n=5, requant=RQ), "tc"),
    # fused requantize -> relu -> requantize chains (realized-graph pattern)
    "rq_relu": (dict(requant=RQ, relu_zp=-3), "tc"),
    "rq_relu_rq": (dict(requant=RQ, relu_zp=2, requant2=(1 << 30, 31, 2, 5)), "tc"),
    "relu_acc": (dict(relu_zp=0), "tc"),
    "simt_rq_relu": (dict(acc="int16", requant=RQ, relu_zp=1), "simt"),
    "w_zp1_out_of_int8": (dict(zp1=-10, wlo=-128, whi=127), "generic"),
    # general multipliers: fused epilogue (tcgen05 / CUDA cores) and chains
    "3x3_rqg": (dict(requant=RQG), "tc"),
    "3x3_zp_rqg2": (dict(zp0=-4, zp1=1, requant=RQG2), "tc"),
    "dense_rqg_max": (dict(dense=True, c=300, o=70, n=5, requant=RQG_MAX), "tc"),
    "rqg_relu_rqg": (dict(requant=RQG, relu_zp=2, requant2=(1610612737, 32, 2, 5)), "tc"),
    "simt_rqg": (dict(acc="int16", requant=(1234567891, 39, 0, 0)), "simt"),
    "i16_rqg": (dict(dtype="int16", requant=(1300000007, 52, 0, 1)), "simt"),
    # int16-accumulator backend ((i8, i8) -> i16) on CUDA cores
    "acc_int16_saturate": (dict(acc="int16", dtype="uint8", zp0=100), "simt"),
    "acc_int16_rq": (dict(acc="int16", zp0=-3, zp1=2, requant=RQ, c=40, o=70), "simt"),
    "dense_zp_int16": (dict(dense=True, c=256, o=10, n=3, zp0=9, zp1=4, acc="int16"), "simt"),
    "dense_int16_acc_big": (dict(dense=True, c=1000, o=37, n=40, acc="int16"), "simt"),
    # int16 codes ((i16, i16) -> i32) on CUDA cores
    "i16_3x3": (dict(dtype="int16", c=20, o=33), "simt"),
    "i16_zp_rq_s2": (dict(dtype="int16", zp0=-700, zp1=5, stride=2, requant=(1 << 30, 50, 0, 1)),
                     "simt"),
    "i16_dense": (dict(dtype="int16", dense=True, c=77, o=12, n=2, zp0=40), "simt"),
    "i16_w_out_of_range": (dict(dtype="int16", zp1=-10, wlo=-32768, whi=32767), "generic"),
}


def _x(case, cfg, seed=1):
    n = cfg.get("n", 2)
    c = cfg.get("c", 16)
    shape = (n, c) if cfg.get("dense") else (n, c, cfg.get("h", 12), cfg.get("w", 12))
    x = np.random.default_rng(seed).normal(0, 2, shape).astype(np.float32)
    return np.abs(x) if cfg.get("dtype") == "uint8" else x


def _backend_counts(cuda_lib):
    c = cuda_lib.counters()
    return c["tcgen05_gemms"], c["simt_int_convs"]


@pytest.mark.parametrize("case", list(CASES))
def test_int_conv_bit_exact_vs_reference(b200, ref, cuda_lib, case):
    cfg, backend = CASES[case]
    doc, blob = F.int_conv_probe(**cfg)
    x = _x(case, cfg)
    yr, dtr = ref.eval_int(ref.graph(doc, blob), x)
    t0, s0 = _backend_counts(cuda_lib)
    yb, dtb = b200.eval_int(b200.graph(doc, blob), x)
    t1, s1 = _backend_counts(cuda_lib)
    assert dtb == dtr
    np.testing.assert_array_equal(yb, yr)
    ran = {"tc": t1 - t0, "simt": s1 - s0}
    if backend == "generic":
        assert ran == {"tc": 0, "simt": 0}
    else:
        assert ran[backend] == 1 and sum(ran.values()) == 1, ran


@pytest.mark.parametrize("case", ["acc_int16_saturate", "dense_zp_int16", "i16_3x3"])
def test_int_conv_trap_matches_reference(b200, ref, case):
    cfg = CASES[case][0]
    doc, blob = F.int_conv_probe(**cfg)
    x = _x(case, cfg)
    with pytest.raises(Q.OverflowError_) as er:
        ref.eval_int(ref.graph(doc, blob), x, trap=True)
    with pytest.raises(Q.OverflowError_) as eb:
        b200.eval_int(b200.graph(doc, blob), x, trap=True)
    assert (eb.value.node, eb.value.flat_index, eb.value.value) == (
        er.value.node, er.value.flat_index, er.value.value)


def _realized(ref, b200, model, spec_name, n):
    data = model.data(n)
    g = ref.graph(model.doc, model.blob)
    spec = ref.parse_spec(F.spec_fixture(spec_name))
    topo = ref.generate_topology(g, spec)
    sim = ref.insert_simulated_quantize(g, topo)
    ds = ref.dataset(data)
    st = ref.collect_stats(g, ds, 2048, ref.simulated_edge_indices(g, topo))
    thr = st.estimate_thresholds("quantile", quantile=0.999, pow2=True)
    ev = ref.evaluator(sim, spec, topo, thr, st, ds)
    strat = ev.strategy_for(ev.space().all_hi())
    R = b200.realize(sim.copy_to(b200), strat, b200.parse_spec(F.spec_fixture(spec_name)))
    return R, data


@pytest.mark.parametrize("name,spec_name", [
    ("small_cnn", "int8_int32"), ("small_cnn", "x86_vnni_like"),
    ("small_cnn", "arm_vmlal_like"), ("resnet18", "int8_int32"),
])
def test_realized_model_eval_int_bit_exact(b200, ref, name, spec_name):
    model = F.small_cnn() if name == "small_cnn" else F.resnet(18, image=32, classes=10,
                                                                 width=8)
    R, data = _realized(ref, b200, model, spec_name, 3)
    Rr = R.copy_to(ref)
    for x in data:
        yr, dtr = ref.eval_int(Rr, x)
        yb, dtb = b200.eval_int(R, x)
        assert dtb == dtr
        np.testing.assert_array_equal(yb, yr)


def test_standalone_requantize_general_multipliers(cuda_lib, port, b200):
    """qcu_requantize (kernels/intops.cu) with multipliers from
    requantize_params of random ratios vs the restatement of
    fixed_point_rescale (reference interpreter.cpp:32-37, :464-482)."""
    import torch
    rng = np.random.default_rng(17)
    x = rng.integers(-(1 << 31), (1 << 31) - 1, 1 << 16, dtype=np.int64).astype(np.int32)
    x[:8] = [0, 1, -1, (1 << 31) - 1, -(1 << 31), 12345, -12345, 7]
    for trial in range(24):
        ratio = float(np.exp2(rng.uniform(-24, 2)))
        mult, shift = b200.requantize_params(ratio, 1.0)
        assert mult != 1 << 30 or ratio == 2.0 ** round(np.log2(ratio))
        in_zp, out_zp = int(rng.integers(-20, 20)), int(rng.integers(-20, 20))
        qmin, qmax = (-128, 127) if trial % 2 else (-32768, 32767)
        y = cuda_lib.requantize(torch.from_numpy(x).cuda(), mult, shift, in_zp, out_zp, qmin,
                                qmax).cpu().numpy()
        np.testing.assert_array_equal(y, port.requantize(x, mult, shift, in_zp, out_zp, qmin,
                                                         qmax))


@pytest.mark.parametrize("name", ["small_cnn", "resnet18"])
def test_realized_general_thresholds_eval_int_bit_exact(b200, ref, name):
    """Realized graphs under NON-power-of-two thresholds (the reference's
    default, calibration.hpp:71-76): realize() emits general fixed-point
    multipliers, and the B200 eval_int equals the reference's eval_int."""
    model = F.small_cnn() if name == "small_cnn" else F.resnet(18, image=32, classes=10,
                                                                 width=8)
    data = model.data(3)
    g = ref.graph(model.doc, model.blob)
    spec = ref.parse_spec(F.spec_fixture("int8_int32"))
    topo = ref.generate_topology(g, spec)
    sim = ref.insert_simulated_quantize(g, topo)
    ds = ref.dataset(data)
    st = ref.collect_stats(g, ds, 2048, ref.simulated_edge_indices(g, topo))
    thr = st.estimate_thresholds("quantile", quantile=0.99, pow2=False)
    ev = ref.evaluator(sim, spec, topo, thr, st, ds)
    strat = ev.strategy_for(ev.space().all_hi())
    R = b200.realize(sim.copy_to(b200), strat, b200.parse_spec(F.spec_fixture("int8_int32")))
    mults = [nd["attrs"]["multiplier"] for nd in R.to_json()["nodes"]
             if nd["op"] == "requantize"]
    assert any(m != 1 << 30 for m in mults), "no general multiplier was emitted"
    Rr = R.copy_to(ref)
    for x in data:
        yr, dtr = ref.eval_int(Rr, x)
        yb, dtb = b200.eval_int(R, x)
        assert dtb == dtr
        np.testing.assert_array_equal(yb, yr)
