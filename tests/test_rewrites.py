"""The exact rewrites that express configs C3/C5 in the reference op set
(fixtures.py: depthwise -> block-diagonal conv, concat -> placement convs +
add, avg_pool -> constant depthwise conv, relu6 -> clip) reproduce the
original ops bit for bit, run on the compiled reference (oracle/_ref)."""
import numpy as np

from paper_2103_14949_b200 import fixtures as F


def _const(gb, blob, nid):
    node = gb.nodes[nid]
    pl = node["payload"]
    n = int(np.prod(pl["shape"]))
    return np.frombuffer(blob, np.float32, n, pl["offset"]).reshape(pl["shape"])


def _depthwise_ref(x, w, b, stride, pad):
    # reference conv semantics per channel: double accumulation in (kh, kw)
    # order over in-bounds taps, + bias, one rounding to float
    n, c, h, wd = x.shape
    k = w.shape[-1]
    oh, ow = (h + 2 * pad - k) // stride + 1, (wd + 2 * pad - k) // stride + 1
    y = np.zeros((n, c, oh, ow), np.float32)
    for ch in range(c):
        for i in range(oh):
            for j in range(ow):
                acc = 0.0
                for a in range(k):
                    for bb in range(k):
                        ih, iw = i * stride - pad + a, j * stride - pad + bb
                        if 0 <= ih < h and 0 <= iw < wd:
                            acc += float(x[0, ch, ih, iw]) * float(w[ch, ch, a, bb])
                y[0, ch, i, j] = np.float32(acc + float(b[ch]))
    return y


def test_depthwise_rewrite_is_exact(ref):
    gb = F.GraphBuilder()
    wts = F._Weights(1)
    x = gb.input("data", [1, 5, 7, 7])
    d = F._depthwise(gb, wts, x, 3, stride=2)
    gb.output(d)
    doc, blob = gb.build()
    xin = np.random.default_rng(0).standard_normal((1, 5, 7, 7)).astype(np.float32)
    y = ref.eval_fp32(ref.graph(doc, blob), xin)
    conv = gb.nodes[d]
    srcs = [e["src"][0] for e in gb.edges if e["dst"][0] == d]
    w, b = _const(gb, blob, srcs[1]), _const(gb, blob, srcs[2])
    assert conv["attrs"]["strides"] == [2, 2]
    np.testing.assert_array_equal(y.reshape(1, 5, 4, 4), _depthwise_ref(xin, w, b, 2, 1))


def test_concat_and_avgpool_rewrites_are_exact(ref):
    gb = F.GraphBuilder()
    wts = F._Weights(2)
    x = gb.input("data", [1, 3, 6, 6])
    a = gb.op("relu", [F._conv(gb, wts, x, 4, 3, pad=1)])
    b = F._conv(gb, wts, x, 2, 1)
    p = F._avg_pool(gb, x)
    cat = F._concat(gb, [a, b, p])
    gb.output(cat)
    doc, blob = gb.build()
    g = ref.graph(doc, blob)
    xin = np.random.default_rng(1).standard_normal((1, 3, 6, 6)).astype(np.float32)
    va = ref.eval_fp32_values(g, xin, [a]).reshape(1, 4, 6, 6)
    vb = ref.eval_fp32_values(g, xin, [b]).reshape(1, 2, 6, 6)
    vp = ref.eval_fp32_values(g, xin, [p]).reshape(1, 3, 6, 6)
    vc = ref.eval_fp32_values(g, xin, [cat]).reshape(1, 9, 6, 6)
    np.testing.assert_array_equal(vc, np.concatenate([va, vb, vp], axis=1))
    # avg pool: double sum of the in-bounds taps / 9 (count_include_pad)
    xp = np.pad(xin.astype(np.float64), ((0, 0), (0, 0), (1, 1), (1, 1)))
    ninth = float(np.float32(1.0 / 9))
    exp = np.zeros_like(vp)
    for c in range(3):
        for i in range(6):
            for j in range(6):
                acc = 0.0
                for u in range(3):
                    for v in range(3):
                        ih, iw = i - 1 + u, j - 1 + v
                        if 0 <= ih < 6 and 0 <= iw < 6:
                            acc += xp[0, c, ih + 1, iw + 1] * ninth
                exp[0, c, i, j] = np.float32(acc)
    np.testing.assert_array_equal(vp, exp)


def test_c3_c5_models_run_on_reference(ref):
    for m in (F.mobilenet_v2(blocks=[(1, 16, 1, 1), (6, 24, 2, 2)]),
              F.inception_v3(modules=1, image=29, width=4)):
        g = ref.graph(m.doc, m.blob)
        y = ref.eval_fp32(g, m.data(1)[0])
        assert np.isfinite(y).all() and y.size == 10
