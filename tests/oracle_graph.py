"""Graph-level CPU oracle: a node-by-node interpreter of a graph document
(Graph.to_json() + blob) with an optional SimBinding, restating the reference
executor (interpreter.cpp:75-179 run_all / eval_node, :196-430 op semantics,
:519-556 predict_top1) on the plain-C arithmetic port (oracle/quantc_oracle.c).

It also covers the op-set extension the reference cannot run (SURVEY §8(f)
rank 2): conv2d with `groups`, avg_pool2d and concat, with the semantics of
their exact rewrites into the reference op set (fixtures.py _depthwise /
_avg_pool / _concat, proven on the compiled reference in test_rewrites.py).

TEST INFRASTRUCTURE: a checker for tests/, never the thing measured.  Samples
are evaluated batch-stacked; every op is per sample or per element, so this
equals the reference's per-sample loop.
"""
from collections import defaultdict, deque

import numpy as np

_DT_RANGE = {1: (-128, 127), 2: (0, 255), 3: (-32768, 32767), 4: (-(2 ** 31), 2 ** 31 - 1)}


def _payload(node, blob):
    pl = node.get("payload") or node["attrs"].get("payload")
    shape = pl["shape"]
    n = int(np.prod(shape)) if shape else 1
    if pl.get("dtype", "float32") == "float32":
        return np.frombuffer(blob, np.float32, n, pl["offset"]).reshape(shape).copy()
    width = {"int8": 1, "uint8": 1, "int16": 2, "int32": 4}[pl["dtype"]]
    raw = np.frombuffer(blob, {1: np.int8, 2: np.int16, 4: np.int32}[width], n, pl["offset"])
    if pl["dtype"] == "uint8":
        raw = raw.view(np.uint8)
    return raw.astype(np.int32).reshape(shape)


class GraphOracle:
    def __init__(self, port, doc, blob):
        self.port = port
        self.doc = doc
        self.blob = blob
        self.nodes = {n["id"]: n for n in doc["nodes"]}
        self.ins = defaultdict(dict)
        for e in doc["edges"]:
            self.ins[e["dst"][0]][e["dst"][1]] = e["src"][0]
        # any topological order: every node is a pure function of its inputs
        indeg = {i: len(self.ins[i]) for i in self.nodes}
        outs = defaultdict(list)
        for e in doc["edges"]:
            outs[e["src"][0]].append(e["dst"][0])
        ready = deque(sorted(i for i, d in indeg.items() if d == 0))
        self.order = []
        while ready:
            i = ready.popleft()
            self.order.append(i)
            for j in outs[i]:
                indeg[j] -= 1
                if indeg[j] == 0:
                    ready.append(j)
        self.consts = {i: _payload(n, blob) for i, n in self.nodes.items() if n["op"] == "constant"}

    # simulate.cpp:64-87 through the C port; binding entries are quantc.QParams
    def _sq(self, nid, x, binding):
        n = self.nodes[nid]
        p = binding.get(nid) if binding else None
        if p is None:
            a = n["attrs"]
            passthrough = a.get("passthrough", True)
            thr, bit, sign, zp = a.get("threshold", 1.0), a.get("bit", 8), a.get("sign", 1), a.get("zero_point", 0)
            has_acc, lo, hi = False, 0.0, 0.0
        else:
            passthrough, thr, bit, sign, zp = bool(p.passthrough), p.threshold, p.bit, p.sign, p.zero_point
            has_acc = p.acc_dtype >= 1 and p.acc_scale > 0.0
            lo, hi = ((float(_DT_RANGE[p.acc_dtype][0]) * p.acc_scale,
                       float(_DT_RANGE[p.acc_dtype][1]) * p.acc_scale) if has_acc else (0.0, 0.0))
        return self.port.sim_quant(x, thr, bit, sign, zp, passthrough, (lo, hi) if has_acc else None)

    def run(self, x, binding=None, values=False):
        """x: [N, C, H, W] (or [N, K]) fp32 samples stacked; returns the graph's
        first output, batch-stacked (and every node's value with values=True)."""
        v = {}
        for nid in self.order:
            n = self.nodes[nid]
            op, a = n["op"], n["attrs"]
            src = [v[self.ins[nid][p]] for p in sorted(self.ins[nid])]
            if op == "input":
                y = np.ascontiguousarray(x, np.float32)
            elif op == "constant":
                y = self.consts[nid]
            elif op == "simulated_quantize":
                y = self._sq(nid, src[0], binding)
            elif op in ("conv2d", "avg_pool2d"):
                st, pd = a.get("strides", None), a.get("padding", [0, 0])
                if op == "conv2d":
                    st = st or [1, 1]
                    w = src[1]
                    b = src[2] if len(src) > 2 else None
                    y = self.port.conv2d(src[0], w, b, tuple(st), tuple(pd), groups=a.get("groups", 1))
                else:
                    k = a["pool_size"]
                    y = self.port.avg_pool2d(src[0], k, tuple(st or k), tuple(pd))
            elif op == "dense":
                d, w = src[0], src[1]
                b = src[2] if len(src) > 2 else None
                y = self.port.conv2d(d.reshape(d.shape[0], d.shape[1], 1, 1),
                                     w.reshape(w.shape[0], w.shape[1], 1, 1), b).reshape(d.shape[0], -1)
            elif op == "add":
                y = (src[0] + src[1]).astype(np.float32)  # float + float, one rounding
            elif op == "relu":
                y = np.where(src[0] < 0, np.float32(0), src[0]).astype(np.float32)
            elif op == "clip":
                lo, hi = np.float32(a["a_min"]), np.float32(a["a_max"])
                s = src[0]
                y = np.where(s < lo, lo, np.where(hi < s, hi, s)).astype(np.float32)
            elif op == "max_pool2d":
                k = a["pool_size"]
                st, pd = a.get("strides", k), a.get("padding", [0, 0])
                s = src[0]
                n_, c_, h_, w_ = s.shape
                oh, ow = (h_ + 2 * pd[0] - k[0]) // st[0] + 1, (w_ + 2 * pd[1] - k[1]) // st[1] + 1
                y = np.full((n_, c_, oh, ow), -np.inf, np.float32)
                for u in range(k[0]):
                    for t in range(k[1]):
                        for i in range(oh):
                            ih = i * st[0] - pd[0] + u
                            if not 0 <= ih < h_:
                                continue
                            for j in range(ow):
                                iw = j * st[1] - pd[1] + t
                                if 0 <= iw < w_:
                                    y[:, :, i, j] = np.maximum(y[:, :, i, j], s[:, :, ih, iw])
            elif op == "global_avg_pool2d":
                y = self.port.global_avg_pool2d(src[0])
            elif op == "flatten":
                y = src[0].reshape(src[0].shape[0], -1)
            elif op == "concat":
                y = np.concatenate(src, axis=1)
            else:
                raise NotImplementedError(op)
            v[nid] = y
        out = self.doc["outputs"][0]
        y = v[out[0] if isinstance(out, list) else out]
        return (y, v) if values else y

    def predict(self, x, binding=None):
        """predict_top1 (interpreter.cpp:533-556): strict '>' argmax over each
        sample's whole output."""
        y = self.run(x, binding).reshape(x.shape[0], -1)
        return np.argmax(y, axis=1).astype(np.int64), y
