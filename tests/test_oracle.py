"""Pins the oracle before trusting it (CPU only).

1. The plain-C restatement (oracle/quantc_oracle.c) against the committed
   known answers produced by the compiled reference (tests/golden/) and
   against SPEC.md's worked examples.
2. The restatement against the compiled reference itself on random inputs.
"""
import json
import os

import numpy as np
import pytest

from paper_2103_14949_b200 import fixtures as F
from paper_2103_14949_b200 import quantc as Q

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


def test_spec_examples_hold_in_golden():
    cs = {(t, b, s): v for t, b, s, v in GOLD["compute_scale"]}
    assert cs[(1.0, 8, 1)] == 2.0**-7 and cs[(6.0, 6, 1)] == 0.1875 and cs[(1.0, 8, 0)] == 2.0**-8
    qb = {(b, s): (lo, hi) for b, s, lo, hi in GOLD["quant_bounds"]}
    assert qb[(8, 1)] == (-128, 127) and qb[(6, 1)] == (-32, 31) and qb[(8, 0)] == (0, 255)
    sq = {(x, t, b): v for x, t, b, v in GOLD["sim_quant_value"]}
    assert sq[(0.5, 1.0, 8)] == 0.5
    assert sq[(2.0, 1.0, 8)] == 0.9921875
    assert sq[(0.004, 1.0, 8)] == 0.0078125
    rp = dict((a, b) for a, b in GOLD["round_pow2"])
    assert rp[3.2] == 4.0 and rp[2.0] == 2.0 and rp[1.5] == 2.0
    assert GOLD["quantile_1_100"] == 99.0
    # the KL estimator is degenerate -> absmax * 2^b / B
    assert GOLD["kl_all_mass_bin0"] == 5.0 * 256 / 2048


def test_port_sim_quant_matches_golden(port):
    for x, t, bit, sign, zp, acc, acc_scale, want in GOLD["sim_quant_tuples"]:
        lo_hi = None
        if acc:
            lo_hi = (-32768 * acc_scale, 32767 * acc_scale)
        got = port.sim_quant(np.array([x], np.float32), t, bit, sign, zp, acc=lo_hi)[0]
        assert np.float32(got).tobytes() == np.float32(want).tobytes(), (x, t, bit, sign)


def test_port_kl_matches_golden(port):
    for h, absmax, tb, want in GOLD["kl_random"]:
        i, _ = port.kl_best_index(np.array(h, np.int64), tb)
        assert absmax * (i / len(h)) == want


def test_port_quantile_matches_golden(port):
    assert port.quantile(np.ones(100, np.int64), 100.0, 0.99) == GOLD["quantile_1_100"]


def test_port_vs_reference_sim_quant_random(port, ref):
    rng = np.random.default_rng(7)
    n = 0
    while n < 10_000:
        t = float(np.exp(rng.uniform(-5, 5)))
        bit = int(rng.integers(2, 9))
        x = (rng.standard_normal(500) * t * 2).astype(np.float32)
        p = Q.QParams.symmetric(t, bit)
        assert port.sim_quant(x, t, bit).tobytes() == ref.simulated_quantize(x, p).tobytes()
        n += x.size


def test_port_vs_reference_conv(port, ref):
    """fp32 conv with sequential double accumulation, through a 1-node graph."""
    rng = np.random.default_rng(8)
    gb = F.GraphBuilder()
    x = gb.input("data", [2, 3, 9, 7])
    w = rng.standard_normal((5, 3, 3, 3)).astype(np.float32)
    b = rng.standard_normal(5).astype(np.float32)
    y = gb.op("conv2d", [x, gb.constant(w), gb.constant(b)], strides=[2, 1], padding=[1, 1])
    gb.output(y)
    doc, blob = gb.build()
    xin = rng.standard_normal((2, 3, 9, 7)).astype(np.float32)
    got = ref.eval_fp32(ref.graph(doc, blob), xin)
    assert got.tobytes() == port.conv2d(xin, w, b, (2, 1), (1, 1)).tobytes()


def test_port_vs_reference_histogram_and_int_ops(port, ref):
    """overflow probe of SPEC.md interpreter examples: 127*127*256 int16."""
    doc, blob = F.overflow_dense(256, 127, "int16")
    g = ref.graph(doc, blob)
    x = np.full((1, 256), 127.0, np.float32)
    out, dt = ref.eval_int(g, x, trap=False)
    assert dt == Q.I16 and (out == 32767).all()
    with pytest.raises(Q.OverflowError_) as ei:
        ref.eval_int(g, x, trap=True)
    assert ei.value.flat_index == 0
    # same via the C restatement
    y, first = port.conv2d_int(np.full((1, 256, 1, 1), 127, np.int32),
                               np.full((4, 256, 1, 1), 127, np.int32), None, (1, 1), (0, 0),
                               0, 0, -32768, 32767)
    assert first == 0 and (y == 32767).all()


def test_port_requantize_examples(port):
    # SPEC.md realize examples: ratio 0.5 -> (2^30, 31); ratio 0.75 -> (1610612736, 31)
    x = np.array([-7, -3, -1, 0, 1, 3, 7, 1000, -1000], np.int32)
    y = port.requantize(x, 1 << 30, 31, 0, 0, -128, 127)
    np.testing.assert_array_equal(y, [-4, -2, -1, 0, 1, 2, 4, 127, -128])  # half away
    y = port.requantize(x, 1610612736, 31, 0, 0, -128, 127)
    np.testing.assert_array_equal(y, np.clip(np.sign(x) * np.floor(np.abs(x) * 0.75 + 0.5), -128, 127))
