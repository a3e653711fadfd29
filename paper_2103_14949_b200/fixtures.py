"""Synthetic models, datasets and hardware specs (the reference's fixtures
module, declared in fixtures.hpp:26-60 but never implemented there).

Graphs are emitted in the C-ABI graph format (include/quantc_capi.h: JSON +
little-endian payload blob) so the identical bytes feed this repo's B200
implementation and the reference oracle.  Weights: conv He-normal
N(0, sqrt(2/fan_in)), dense N(0, sqrt(1/fan_in)), bias N(0, 0.01) with BN
pre-folded (SPEC.md graph-ir non-goals); inputs N(0, 1).  Seeds are explicit.

Config map (BASELINE.json:configs):
  [0] small_cnn          2x conv3x3-relu + dense, 16 x [1,3,32,32]
  [1] resnet(18)         224x224
  [3] resnet(50)         224x224 (the bench workload)
  [2]/[4] mobilenet_v2 / inception_v3: op-set rewrites, SURVEY.md §7 (not in round 1)
"""
from __future__ import annotations

import json
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

# ---- hardware specs (fixtures.hpp:35-40, SPEC.md fixtures module) ----------

def _sig(ins, out):
    return {"in": list(ins), "out": out}


SPECS: Dict[str, dict] = {
    # Fig. 3: add {f32, i32}, conv2d {i16xi16->i32, i8xi8->i16}, f32 pooling
    "fig3": {"ops": {
        "add": [_sig(["float32", "float32"], "float32"), _sig(["int32", "int32"], "int32")],
        "conv2d": [_sig(["int16", "int16"], "int32"), _sig(["int8", "int8"], "int16")],
        "global_avg_pool2d": [_sig(["float32"], "float32")],
    }},
    # uint8 activations x int8 weights -> int32 (x86 VNNI style)
    "x86_vnni_like": {"ops": {
        "conv2d": [_sig(["uint8", "int8"], "int32")],
        "dense": [_sig(["uint8", "int8"], "int32")],
    }},
    # int8 x int8 -> int16 accumulation and int16 x int16 -> int32 (ARM vmlal)
    "arm_vmlal_like": {"ops": {
        "conv2d": [_sig(["int8", "int8"], "int16"), _sig(["int16", "int16"], "int32")],
        "dense": [_sig(["int8", "int8"], "int16"), _sig(["int16", "int16"], "int32")],
    }},
    # int8 x int8 -> int32 mac ops, int8 elementwise (the headline spec)
    "int8_int32": {"ops": {
        "conv2d": [_sig(["int8", "int8"], "int32")],
        "dense": [_sig(["int8", "int8"], "int32")],
        "add": [_sig(["int8", "int8"], "int32")],
        "relu": [_sig(["int8"], "int8")],
        "max_pool2d": [_sig(["int8"], "int8")],
        "clip": [_sig(["int8"], "int8")],
    }},
}


def spec_fixture(name: str) -> str:
    if name not in SPECS:
        raise KeyError(f"unknown spec fixture {name!r}")
    return json.dumps(SPECS[name])


# ---- graph builder ----------------------------------------------------------

class GraphBuilder:
    """Builds the C-ABI graph document (nodes/edges/inputs/outputs + blob)."""

    def __init__(self):
        self.nodes: List[dict] = []
        self.edges: List[dict] = []
        self.inputs: List[int] = []
        self.outputs: List[List[int]] = []
        self.blob = bytearray()
        self.shapes: Dict[int, Tuple[int, ...]] = {}
        self._next = 0

    def _new(self, op: str, attrs: Optional[dict] = None, payload=None) -> int:
        nid = self._next
        self._next += 1
        node = {"id": nid, "op": op, "attrs": attrs or {}}
        if payload is not None:
            node["payload"] = payload
        self.nodes.append(node)
        return nid

    def input(self, name: str, shape: Sequence[int]) -> int:
        nid = self._new("input", {"name": name, "shape": list(shape)})
        self.inputs.append(nid)
        self.shapes[nid] = tuple(shape)
        return nid

    def constant(self, arr: np.ndarray, dtype: str = "float32") -> int:
        if dtype == "float32":
            data = np.ascontiguousarray(arr, dtype=np.float32)
        else:
            data = np.ascontiguousarray(arr, dtype=np.int32)
        off = len(self.blob)
        self.blob += data.tobytes()
        nid = self._new("constant", {}, {"dtype": dtype, "shape": list(data.shape),
                                          "offset": off})
        self.shapes[nid] = tuple(data.shape)
        return nid

    def op(self, op: str, inputs: Sequence[int], **attrs) -> int:
        nid = self._new(op, attrs)
        for port, src in enumerate(inputs):
            self.edges.append({"src": [src, 0], "dst": [nid, port]})
        self.shapes[nid] = self._infer(op, [self.shapes[i] for i in inputs], attrs)
        return nid

    def output(self, nid: int):
        self.outputs.append([nid, 0])

    @staticmethod
    def _infer(op, ins, attrs):
        if op == "conv2d":
            (n, c, h, w), (o, _, kh, kw) = ins[0], ins[1]
            s = attrs.get("strides", [1, 1])
            p = attrs.get("padding", [0, 0])
            return (n, o, (h + 2 * p[0] - kh) // s[0] + 1, (w + 2 * p[1] - kw) // s[1] + 1)
        if op == "dense":
            return (ins[0][0], ins[1][0])
        if op == "concat":
            return (ins[0][0], sum(i[1] for i in ins), ins[0][2], ins[0][3])
        if op in ("max_pool2d", "avg_pool2d"):
            n, c, h, w = ins[0]
            k = attrs["pool_size"]
            s = attrs.get("strides", k)
            p = attrs.get("padding", [0, 0])
            return (n, c, (h + 2 * p[0] - k[0]) // s[0] + 1, (w + 2 * p[1] - k[1]) // s[1] + 1)
        if op == "global_avg_pool2d":
            return (ins[0][0], ins[0][1], 1, 1)
        if op == "flatten":
            return (ins[0][0], int(np.prod(ins[0][1:])))
        return ins[0]

    def build(self) -> Tuple[dict, bytes]:
        doc = {"nodes": self.nodes, "edges": self.edges, "inputs": self.inputs,
               "outputs": self.outputs}
        return doc, bytes(self.blob)


class Model:
    """A synthetic model: graph document + blob + calibration data."""

    def __init__(self, name, doc, blob, sample_shape, gb: GraphBuilder):
        self.name, self.doc, self.blob = name, doc, blob
        self.sample_shape = tuple(sample_shape)
        self.builder = gb

    def data(self, n: int, seed: int = 9) -> np.ndarray:
        rng = np.random.default_rng(seed)
        return rng.standard_normal((n,) + self.sample_shape, dtype=np.float32)

    def macs_per_sample(self) -> int:
        gb = self.builder
        total = 0
        for node in gb.nodes:
            if node["op"] not in ("conv2d", "dense"):
                continue
            srcs = [e["src"][0] for e in gb.edges if e["dst"][0] == node["id"]]
            wshape = gb.shapes[srcs[1]]
            oshape = gb.shapes[node["id"]]
            if node["op"] == "conv2d":
                total += int(np.prod(oshape[1:])) * int(np.prod(wshape[1:]))
            else:
                total += oshape[1] * wshape[1]
        return total


# ---- weight helpers ---------------------------------------------------------

class _Weights:
    def __init__(self, seed: int):
        self.rng = np.random.default_rng(seed)

    def conv(self, o, c, kh, kw, gain=1.0):
        fan_in = c * kh * kw
        return (self.rng.standard_normal((o, c, kh, kw), dtype=np.float32)
                * np.float32(gain * np.sqrt(2.0 / fan_in)))

    def dense(self, m, k):
        return self.rng.standard_normal((m, k), dtype=np.float32) * np.float32(np.sqrt(1.0 / k))

    def bias(self, n):
        return self.rng.standard_normal((n,), dtype=np.float32) * np.float32(0.01)


def _conv(gb, wts, x, o, k, stride=1, pad=0, gain=1.0, bias=True):
    c = gb.shapes[x][1]
    w = gb.constant(wts.conv(o, c, k, k, gain))
    ins = [x, w]
    if bias:
        ins.append(gb.constant(wts.bias(o)))
    return gb.op("conv2d", ins, strides=[stride, stride], padding=[pad, pad])


# ---- models ----------------------------------------------------------------

def small_cnn(seed: int = 7, image: int = 32, channels: int = 16, classes: int = 10) -> Model:
    """BASELINE config 0: 2x (conv3x3 pad 1 + relu) + flatten + dense."""
    gb = GraphBuilder()
    wts = _Weights(seed)
    x = gb.input("data", [1, 3, image, image])
    h = gb.op("relu", [_conv(gb, wts, x, channels, 3, pad=1)])
    h = gb.op("relu", [_conv(gb, wts, h, channels, 3, pad=1)])
    f = gb.op("flatten", [h])
    k = gb.shapes[f][1]
    y = gb.op("dense", [f, gb.constant(wts.dense(classes, k)), gb.constant(wts.bias(classes))])
    gb.output(y)
    doc, blob = gb.build()
    return Model("small_cnn", doc, blob, [1, 3, image, image], gb)


def conv_add_pool_chain(seed: int = 5, image: int = 8) -> Model:
    """Fig. 4 chain: conv2d -> add(constant) -> global_avg_pool2d (fixtures.hpp:54-56)."""
    gb = GraphBuilder()
    wts = _Weights(seed)
    x = gb.input("data", [1, 3, image, image])
    c = _conv(gb, wts, x, 4, 3, pad=1, bias=False)
    cst = gb.constant(wts.rng.standard_normal(gb.shapes[c], dtype=np.float32))
    a = gb.op("add", [c, cst])
    p = gb.op("global_avg_pool2d", [a])
    gb.output(p)
    doc, blob = gb.build()
    return Model("conv_add_pool_chain", doc, blob, [1, 3, image, image], gb)


def deep_chain(searchable_edges: int, seed: int = 3, width: int = 8) -> Model:
    """dense/relu chain with `searchable_edges` quantizable edges under int8_int32
    (fixtures.hpp:50-52): each dense contributes 2 (data, weight), each relu 1."""
    gb = GraphBuilder()
    wts = _Weights(seed)
    h = gb.input("data", [1, width])
    remaining = searchable_edges
    while remaining > 0:
        if remaining >= 2:
            h = gb.op("dense", [h, gb.constant(wts.dense(width, width))])
            remaining -= 2
        if remaining >= 1:
            h = gb.op("relu", [h])
            remaining -= 1
    gb.output(h)
    doc, blob = gb.build()
    return Model(f"deep_chain_{searchable_edges}", doc, blob, [1, width], gb)


def resnet(depth: int = 50, seed: int = 42, image: int = 224, classes: int = 1000,
           width: int = 64, residual_gain: float = 0.3, batch: int = 1) -> Model:
    """BN-folded ResNet-18/34/50/101 (torchvision topology) built from the closed
    op set: conv2d(+bias) / relu / max_pool2d / add / global_avg_pool2d /
    flatten / dense.  `residual_gain` scales the last conv of every residual
    branch (a folded BN gamma < 1) so activations stay O(1) with depth.
    `batch` > 1 declares a batched input [batch, 3, image, image] (one eval_int
    call over many images; predict_top1 samples stay [1, 3, H, W])."""
    cfg = {18: ("basic", [2, 2, 2, 2]), 34: ("basic", [3, 4, 6, 3]),
           50: ("bottleneck", [3, 4, 6, 3]), 101: ("bottleneck", [3, 4, 23, 3])}
    kind, blocks = cfg[depth]
    gb = GraphBuilder()
    wts = _Weights(seed)
    x = gb.input("data", [batch, 3, image, image])
    h = gb.op("relu", [_conv(gb, wts, x, width, 7, stride=2, pad=3)])
    h = gb.op("max_pool2d", [h], pool_size=[3, 3], strides=[2, 2], padding=[1, 1])
    expansion = 4 if kind == "bottleneck" else 1
    in_c = width
    for stage, n in enumerate(blocks):
        planes = width * (2 ** stage)
        for b in range(n):
            stride = 2 if (b == 0 and stage > 0) else 1
            if kind == "basic":
                y = gb.op("relu", [_conv(gb, wts, h, planes, 3, stride, 1)])
                y = _conv(gb, wts, y, planes, 3, 1, 1, gain=residual_gain)
            else:
                y = gb.op("relu", [_conv(gb, wts, h, planes, 1)])
                y = gb.op("relu", [_conv(gb, wts, y, planes, 3, stride, 1)])
                y = _conv(gb, wts, y, planes * expansion, 1, gain=residual_gain)
            out_c = planes * expansion
            if stride != 1 or in_c != out_c:
                sc = _conv(gb, wts, h, out_c, 1, stride, 0)
            else:
                sc = h
            h = gb.op("relu", [gb.op("add", [y, sc])])
            in_c = out_c
    p = gb.op("global_avg_pool2d", [h])
    f = gb.op("flatten", [p])
    y = gb.op("dense", [f, gb.constant(wts.dense(classes, in_c)), gb.constant(wts.bias(classes))])
    gb.output(y)
    doc, blob = gb.build()
    return Model(f"resnet{depth}", doc, blob, [batch, 3, image, image], gb)


# ---- exact rewrites of ops outside the reference op set --------
#
# The reference has no grouped/depthwise conv, concat or avg_pool2d
# (graph.cpp:17-35).  Configs C3 (MobileNetV2) and C5 (Inception-v3) are built
# from exact rewrites so the unmodified reference runs them:
#   depthwise KxK      -> conv2d with block-diagonal weights (off-diagonal
#                         taps are 0: x*0 adds a signed zero to a nonzero or
#                         +0 double accumulator, so the sum is unchanged)
#   concat(a, b, ...)  -> sum of 1x1 "placement" convs (identity blocks),
#                         one nonzero term per output channel
#   avg_pool KxK       -> depthwise conv with constant 1/(K*K) weights
#                         (count_include_pad semantics)
#   relu6              -> clip(0, 6)

# native=True emits the op-set extension instead (conv2d groups=C,
# avg_pool2d, concat: include/quantc/graph.hpp), with the same weights drawn
# from the same RNG stream, so the native and rewritten graphs compute
# bit-identical fp32 values (tests/test_gpu_native_ops.py).

def _depthwise(gb, wts, x, k, stride=1, pad=None, gain=1.0, bias=True, native=False):
    c = gb.shapes[x][1]
    pad = k // 2 if pad is None else pad
    dw = wts.rng.standard_normal((c, k, k), dtype=np.float32) * np.float32(gain * np.sqrt(2.0 / (k * k)))
    if native:
        w = dw.reshape(c, 1, k, k).copy()
    else:
        w = np.zeros((c, c, k, k), np.float32)
        for i in range(c):
            w[i, i] = dw[i]
    ins = [x, gb.constant(w)]
    if bias:
        ins.append(gb.constant(wts.bias(c)))
    if native:
        return gb.op("conv2d", ins, strides=[stride, stride], padding=[pad, pad], groups=c)
    return gb.op("conv2d", ins, strides=[stride, stride], padding=[pad, pad])


def _avg_pool(gb, x, k=3, stride=1, pad=1, native=False):
    if native:
        return gb.op("avg_pool2d", [x], pool_size=[k, k], strides=[stride, stride], padding=[pad, pad])
    c = gb.shapes[x][1]
    w = np.zeros((c, c, k, k), np.float32)
    for i in range(c):
        w[i, i] = np.float32(1.0 / (k * k))
    return gb.op("conv2d", [x, gb.constant(w)], strides=[stride, stride], padding=[pad, pad])


def _concat(gb, xs, native=False):
    if native:
        return gb.op("concat", list(xs), axis=1)
    total = sum(gb.shapes[x][1] for x in xs)
    out, off = None, 0
    for x in xs:
        c = gb.shapes[x][1]
        p = np.zeros((total, c, 1, 1), np.float32)
        for i in range(c):
            p[off + i, i, 0, 0] = 1.0
        y = gb.op("conv2d", [x, gb.constant(p)], strides=[1, 1], padding=[0, 0])
        out = y if out is None else gb.op("add", [out, y])
        off += c
    return out


def _relu6(gb, x):
    return gb.op("clip", [x], a_min=0.0, a_max=6.0)


def mobilenet_v2(seed: int = 11, image: int = 32, classes: int = 10, width: float = 0.25,
                 blocks=None, native: bool = False) -> Model:
    """BASELINE config C3: MobileNetV2 (inverted residuals, relu6, linear
    bottlenecks) with depthwise convs rewritten exactly (see above), for the
    arm_vmlal_like int16-accumulation spec.  `blocks` = (t, c, n, s) rows;
    the default is the paper's table at width `width`."""
    cfg = blocks or [(1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 3, 2), (6, 64, 4, 2),
                     (6, 96, 3, 1), (6, 160, 3, 2), (6, 320, 1, 1)]

    def ch(c):
        return max(8, int(round(c * width / 8)) * 8)

    gb = GraphBuilder()
    wts = _Weights(seed)
    x = gb.input("data", [1, 3, image, image])
    h = _relu6(gb, _conv(gb, wts, x, ch(32), 3, stride=2, pad=1))
    in_c = ch(32)
    for t, c, n, s in cfg:
        out_c = ch(c)
        for i in range(n):
            stride = s if i == 0 else 1
            y = h
            if t != 1:
                y = _relu6(gb, _conv(gb, wts, y, in_c * t, 1))
            y = _relu6(gb, _depthwise(gb, wts, y, 3, stride, native=native))
            y = _conv(gb, wts, y, out_c, 1, gain=0.5)  # linear bottleneck
            h = gb.op("add", [h, y]) if (stride == 1 and in_c == out_c) else y
            in_c = out_c
    h = _relu6(gb, _conv(gb, wts, h, max(ch(1280), 64), 1))
    p = gb.op("global_avg_pool2d", [h])
    f = gb.op("flatten", [p])
    y = gb.op("dense", [f, gb.constant(wts.dense(classes, gb.shapes[f][1])),
                        gb.constant(wts.bias(classes))])
    gb.output(y)
    doc, blob = gb.build()
    return Model("mobilenet_v2" + ("_native" if native else ""), doc, blob, [1, 3, image, image], gb)


def inception_v3(seed: int = 13, image: int = 35, classes: int = 10, width: int = 8,
                 modules: int = 2, head: str = "flatten", native: bool = False) -> Model:
    """BASELINE config C5: an Inception-v3-style network (stem, Inception-A
    modules with 1x1 / 1x1-3x3 / 1x1-3x3-3x3 / avgpool-1x1 branches, a
    grid-reduction module, Inception-C-style 1x3/3x1 factorised branches) with
    concat and avg_pool rewritten exactly (see above).  head "gap" is the
    paper's global-average-pool classifier; "flatten" (default) keeps the
    spatial map so random inputs give varied top-1 predictions, which the
    search's agreement loss needs."""
    gb = GraphBuilder()
    wts = _Weights(seed)

    def cbr(x, o, kh, kw=None, stride=1, ph=None, pw=None):
        kw = kh if kw is None else kw
        c = gb.shapes[x][1]
        w = gb.constant(wts.conv(o, c, kh, kw))
        ph = kh // 2 if ph is None else ph
        pw = kw // 2 if pw is None else pw
        y = gb.op("conv2d", [x, w, gb.constant(wts.bias(o))], strides=[stride, stride],
                  padding=[ph, pw])
        return gb.op("relu", [y])

    x = gb.input("data", [1, 3, image, image])
    h = cbr(x, 2 * width, 3, stride=2, ph=0, pw=0)
    h = cbr(h, 2 * width, 3)
    h = cbr(h, 4 * width, 3)
    for _ in range(modules):  # Inception-A
        b1 = cbr(h, 4 * width, 1)
        b2 = cbr(cbr(h, 3 * width, 1), 4 * width, 3)
        b3 = cbr(cbr(cbr(h, 4 * width, 1), 6 * width, 3), 6 * width, 3)
        b4 = cbr(_avg_pool(gb, h, native=native), 2 * width, 1)
        h = _concat(gb, [b1, b2, b3, b4], native=native)
    # grid reduction: 3x3 stride 2 | 1x1-3x3-3x3 stride 2 | max pool
    r1 = cbr(h, 8 * width, 3, stride=2, ph=0, pw=0)
    r2 = cbr(cbr(h, 4 * width, 1), 6 * width, 3, stride=2, ph=0, pw=0)
    r3 = gb.op("max_pool2d", [h], pool_size=[3, 3], strides=[2, 2], padding=[0, 0])
    h = _concat(gb, [r1, r2, r3], native=native)
    # Inception-C-style: 1x1 | 1x1 -> (1x3, 3x1)
    c1 = cbr(h, 8 * width, 1)
    c2 = cbr(h, 6 * width, 1)
    c2 = _concat(gb, [cbr(c2, 4 * width, 1, 3), cbr(c2, 4 * width, 3, 1)], native=native)
    h = _concat(gb, [c1, c2], native=native)
    if head == "gap":
        f = gb.op("flatten", [gb.op("global_avg_pool2d", [h])])
    else:
        # a linear 1x1 projection with zero-sum rows removes the relu
        # features' common mode
        w = wts.conv(2 * width, gb.shapes[h][1], 1, 1)
        w -= w.mean(axis=1, keepdims=True)
        f = gb.op("flatten", [gb.op("conv2d", [h, gb.constant(w)], strides=[1, 1],
                                    padding=[0, 0])])
    y = gb.op("dense", [f, gb.constant(wts.dense(classes, gb.shapes[f][1])),
                        gb.constant(wts.bias(classes))])
    gb.output(y)
    doc, blob = gb.build()
    return Model("inception_v3" + ("_native" if native else ""), doc, blob, [1, 3, image, image], gb)


def overflow_dense(k: int = 256, value: int = 127, acc: str = "int16") -> Tuple[dict, bytes]:
    """Realized int8 dense probe from SPEC.md interpreter examples: quantize ->
    dense(int8, weights all `value`) with `acc` accumulator. 127*127*256 exceeds
    int16, so saturate -> 32767 and trap -> OverflowError at the dense node."""
    gb = GraphBuilder()
    x = gb.input("data", [1, k])
    q = gb.op("quantize", [x], scale=1.0, zero_point=0, q_min=-128, q_max=127,
              out_dtype="int8")
    w = gb.constant(np.full((4, k), value, np.int32), dtype="int8")
    d = gb.op("dense", [q, w], acc_dtype=acc)
    gb.output(d)
    return gb.build()


def int_conv_probe(n=2, c=16, h=12, w=12, o=24, k=3, stride=1, pad=1, dtype="int8",
                   zp0=0, zp1=0, acc="int32", requant=None, dense=False, seed=0,
                   wlo=None, whi=None, relu_zp=None, requant2=None) -> Tuple[dict, bytes]:
    """Realized-graph integer conv2d/dense probe (SPEC.md realize output
    shapes): quantize(x) -> conv2d / dense(int weights, int32 bias, zero
    points, acc dtype) [-> requantize(multiplier, shift, zero points)].
    Exercises every IntEpi path of the tcgen05 integer kernel: signed /
    unsigned data, nonzero zp0 with padding, zp1 folding, accumulator
    saturation (int16 acc), and a fused requantize."""
    rng = np.random.default_rng(seed)
    lo, hi = {"int8": (-128, 127), "uint8": (0, 255), "int16": (-32768, 32767)}[dtype]
    # default weight range: values of the data's width whose w - zp1 fits it
    wl, wh = (-32768, 32767) if dtype == "int16" else (-128, 127)
    wlo = max(wl, wl + zp1) if wlo is None else wlo
    whi = min(wh, wh + zp1) if whi is None else whi
    wdt = "int16" if dtype == "int16" else "int8"
    gb = GraphBuilder()
    shape = [n, c] if dense else [n, c, h, w]
    x = gb.input("data", shape)
    q = gb.op("quantize", [x], scale=1.0 / (4096 if dtype == "int16" else 32), zero_point=zp0,
              q_min=lo, q_max=hi, out_dtype=dtype)
    if dense:
        wt = gb.constant(rng.integers(wlo, whi + 1, (o, c)), dtype=wdt)
    else:
        wt = gb.constant(rng.integers(wlo, whi + 1, (o, c, k, k)), dtype=wdt)
    b = gb.constant(rng.integers(-5000, 5000, (o,)), dtype="int32")
    attrs = dict(acc_dtype=acc, in_zero_points=[zp0, zp1])
    if dense:
        y = gb.op("dense", [q, wt, b], **attrs)
    else:
        y = gb.op("conv2d", [q, wt, b], strides=[stride, stride], padding=[pad, pad], **attrs)
    if requant is not None:
        mult, shift, in_zp, out_zp = requant
        y = gb.op("requantize", [y], multiplier=mult, shift=shift, in_zero_point=in_zp,
                  zero_point=out_zp, q_min=-128, q_max=127, out_dtype="int8")
    if relu_zp is not None:  # relu int: max(x, zero_point)
        y = gb.op("relu", [y], zero_point=relu_zp)
    if requant2 is not None:
        mult, shift, in_zp, out_zp = requant2
        y = gb.op("requantize", [y], multiplier=mult, shift=shift, in_zero_point=in_zp,
                  zero_point=out_zp, q_min=-128, q_max=127, out_dtype="int8")
    gb.output(y)
    return gb.build()
