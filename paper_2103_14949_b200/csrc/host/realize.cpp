// realize.cpp — realization helpers declared by reference realize.hpp:17-62.
// The reference ships no implementation; these follow SPEC.md's realize
// module (:593-672).  Full graph lowering (realize()) is SURVEY §8(f) rank 1.
#include "quantc/realize.hpp"

#include <algorithm>
#include <cmath>
#include <set>
#include <map>

#include "quantc/simulate.hpp"

namespace quantc {

double RequantParams::value() const { return std::ldexp(static_cast<double>(multiplier), -shift); }

double EdgeDecision::scale() const { return compute_scale(threshold, bit, sign); }

RequantParams requantize_params(double s_in, double s_out) {
  if (!(s_in > 0.0) || !(s_out > 0.0)) throw RealizeError("requantize_params needs positive scales");
  int e = 0;
  const double m = std::frexp(s_in / s_out, &e);  // ratio = m * 2^e, m in [0.5, 1)
  int64_t mult = std::llround(std::ldexp(m, 31));
  int shift = 31 - e;
  if (mult == (int64_t{1} << 31)) {
    mult >>= 1;
    --shift;
  }
  RequantParams r;
  r.multiplier = static_cast<int32_t>(mult);
  r.shift = shift;
  return r;
}

DType choose_storage_dtype(int bit, const std::vector<DType>& candidates, int sign) {
  const DType* best = nullptr;
  for (const DType& d : candidates) {
    if (d.is_float() || max_bits(d) < bit) continue;
    if (sign == 1 && !d.is_signed()) continue;
    if (sign == 0 && d.is_signed()) continue;
    if (!best || d.width() < best->width()) best = &d;
  }
  if (!best) {
    throw RealizeError("no candidate dtype can hold " + std::to_string(bit) + " effective bits");
  }
  return *best;
}

std::pair<int64_t, int64_t> rewrite_clip(double min_f, double max_f, double s_out,
                                         int64_t zero_point, DType storage) {
  int64_t lo = std::llround(min_f / s_out) + zero_point;
  int64_t hi = std::llround(max_f / s_out) + zero_point;
  lo = std::clamp(lo, storage.min_value(), storage.max_value());
  hi = std::clamp(hi, storage.min_value(), storage.max_value());
  return {lo, hi};
}

namespace {

// Realized value of a sim-graph output: where it lives in the new graph and,
// for integers, the grid it is on (value = (q - zp) * scale).
struct Dom {
  PortRef ref;
  bool integer = false;
  double scale = 1.0;
  double threshold = 0.0;  // of the sq that produced it (add: unified-scale choice)
  int64_t zp = 0;
  DType dtype = f32;
  bool folded_const = false;  // a constant quantized at realize time (weights)
};

class Lowering {
 public:
  Lowering(const Graph& g, const Strategy& st, const HardwareSpec& spec)
      : g_(g), st_(st), spec_(spec), next_id_(g.max_node_id() + 1) {}

  Graph run() {
    for (NodeId id : traversal_order(g_)) {
      try {
        lower(g_.node(id));
      } catch (const RealizeError&) {
        throw;
      } catch (const std::exception& e) {
        throw RealizeError("realize: node " + std::to_string(id) + " (" +
                           op_name(g_.node(id).op) + "): " + e.what());
      }
    }
    std::vector<PortRef> outs;
    for (const PortRef& o : g_.outputs()) outs.push_back(dom_.at(o.node).ref);
    std::vector<NodeId> inputs = g_.inputs();
    return Graph(std::move(nodes_), std::move(edges_), std::move(inputs), std::move(outs));
  }

 private:
  NodeId emit(Node n, const std::vector<PortRef>& ins) {
    const NodeId id = n.id;
    for (size_t p = 0; p < ins.size(); ++p) {
      if (ins[p].node >= 0) edges_.push_back(Edge{ins[p], PortRef{id, static_cast<int>(p)}});
    }
    nodes_.push_back(std::move(n));
    return id;
  }
  Node fresh(OpKind op) {
    Node n;
    n.id = next_id_++;
    n.op = op;
    return n;
  }
  // producers of a node's data ports, in port order (unfed ports -> -1)
  std::vector<NodeId> producers(NodeId id) const {
    std::vector<NodeId> out;
    for (const Edge* e : g_.in_edges(id)) out.push_back(e ? e->src.node : -1);
    return out;
  }
  const EdgeDecision* decision(const Node& sq) const {
    if (sq.attr_or<bool>("boundary", false)) return nullptr;
    const int e = sq.attr_or<int>("edge_index", -1);
    auto it = st_.edges.find(e);
    return it == st_.edges.end() ? nullptr : &it->second;
  }

  // integer codes of `d` moved onto the grid (s, zp, dtype, bounds)
  Dom to_grid(const Dom& d, const EdgeDecision& dec) {
    const double s = dec.scale();
    const QuantBounds qb = quant_bounds(dec.bit, dec.sign);
    Dom out;
    out.integer = true;
    out.scale = s;
    out.threshold = dec.threshold;
    out.zp = dec.zero_point;
    out.dtype = dec.storage_dtype;
    if (!d.integer) {
      Node q = fresh(OpKind::kQuantize);
      q.attrs["scale"] = s;
      q.attrs["zero_point"] = dec.zero_point;
      q.attrs["q_min"] = qb.qmin;
      q.attrs["q_max"] = qb.qmax;
      q.attrs["out_dtype"] = dec.storage_dtype.name();
      out.ref = PortRef{emit(std::move(q), {d.ref}), 0};
      return out;
    }
    if (d.scale == s && d.zp == dec.zero_point && d.dtype == dec.storage_dtype) {
      out.ref = d.ref;  // already there
      return out;
    }
    const RequantParams rp = requantize_params(d.scale, s);
    Node r = fresh(OpKind::kRequantize);
    r.attrs["multiplier"] = static_cast<int64_t>(rp.multiplier);
    r.attrs["shift"] = rp.shift;
    r.attrs["in_zero_point"] = d.zp;
    r.attrs["zero_point"] = dec.zero_point;
    r.attrs["q_min"] = qb.qmin;
    r.attrs["q_max"] = qb.qmax;
    r.attrs["out_dtype"] = dec.storage_dtype.name();
    out.ref = PortRef{emit(std::move(r), {d.ref}), 0};
    return out;
  }

  Dom as_float(const Dom& d) {
    if (!d.integer) return d;
    Node q = fresh(OpKind::kDequantize);
    q.attrs["scale"] = d.scale;
    q.attrs["zero_point"] = d.zp;
    Dom out;
    out.ref = PortRef{emit(std::move(q), {d.ref}), 0};
    return out;
  }

  // weight edge: fold sq into an integer constant (SPEC: "constant-input
  // quantize ops are constant-folded")
  Dom fold(const Node& c, const EdgeDecision& dec) {
    const double s = dec.scale();
    const QuantBounds qb = quant_bounds(dec.bit, dec.sign);
    auto w = c.payload->floats();
    std::vector<int32_t> codes(w.size());
    for (size_t i = 0; i < w.size(); ++i) {
      const int64_t q = std::llround(static_cast<double>(w[i]) / s) + dec.zero_point;
      codes[i] = static_cast<int32_t>(std::clamp(q, qb.qmin, qb.qmax));
    }
    Node k = fresh(OpKind::kConstant);
    k.payload = Tensor::from_ints(dec.storage_dtype, c.payload->shape(), std::move(codes));
    Dom out;
    out.integer = true;
    out.folded_const = true;
    out.scale = s;
    out.threshold = dec.threshold;
    out.zp = dec.zero_point;
    out.dtype = dec.storage_dtype;
    out.ref = PortRef{emit(std::move(k), {}), 0};
    return out;
  }

  DType acc_dtype(OpKind op, const std::vector<Dom>& ins, const std::vector<const EdgeDecision*>& decs) {
    std::vector<int> bits, signs;
    for (size_t i = 0; i < ins.size(); ++i) {
      bits.push_back(decs[i] ? decs[i]->bit : max_bits(ins[i].dtype));
      signs.push_back(decs[i] ? decs[i]->sign : (ins[i].dtype.is_signed() ? 1 : 0));
    }
    const auto sigs = spec_.signatures(op);
    const Signature* sig = match_signature(sigs, bits, signs);
    if (!sig) {
      throw RealizeError("no hardware signature of " + op_name(op) +
                         " is consistent with the strategy's bit widths");
    }
    return sig->out_dtype;
  }

  void lower(const Node& n) {
    switch (n.op) {
      case OpKind::kInput: {
        Node c = n;
        dom_[n.id].ref = PortRef{emit(std::move(c), {}), 0};
        return;
      }
      case OpKind::kConstant:
        // emitted lazily: folded by a weight sq, quantized as a bias, or
        // copied for a float consumer (lower_operands)
        consts_.insert(n.id);
        return;
      case OpKind::kSimulatedQuantize: {
        const NodeId src = producers(n.id).at(0);
        const EdgeDecision* dec = decision(n);
        const Node& p = g_.node(src);
        if (p.op == OpKind::kConstant) {
          dom_[n.id] = dec ? fold(p, *dec) : float_const(p);
          return;
        }
        const Dom& d = dom_.at(src);
        dom_[n.id] = dec ? to_grid(d, *dec) : as_float(d);
        sq_dec_[n.id] = dec;
        return;
      }
      default:
        lower_op(n);
    }
  }

  Dom float_const(const Node& c) {
    auto it = const_copy_.find(c.id);
    if (it != const_copy_.end()) return it->second;
    Node k = c;
    Dom d;
    d.ref = PortRef{emit(std::move(k), {}), 0};
    const_copy_[c.id] = d;
    return d;
  }

  Dom operand(NodeId src) {
    if (consts_.count(src)) return float_const(g_.node(src));
    return dom_.at(src);
  }

  void lower_op(const Node& n) {
    const auto prod = producers(n.id);
    std::vector<Dom> ins;
    std::vector<const EdgeDecision*> decs;
    for (NodeId s : prod) {
      ins.push_back(s >= 0 ? operand(s) : Dom{});
      auto it = sq_dec_.find(s);
      decs.push_back(it == sq_dec_.end() ? nullptr : it->second);
    }
    Node out = n;
    Dom res;
    switch (n.op) {
      case OpKind::kConv2d:
      case OpKind::kDense: {
        const Dom& d = ins.at(0);
        const Dom& w = ins.at(1);
        if (d.integer != w.integer) {
          throw RealizeError(op_name(n.op) + " node " + std::to_string(n.id) +
                             " has one quantized and one float operand");
        }
        if (!d.integer) break;  // stays a float op
        const DType acc = acc_dtype(n.op, {d, w}, {decs[0], decs[1]});
        out.attrs["acc_dtype"] = acc.name();
        out.attrs["in_zero_points"] = std::vector<int64_t>{d.zp, w.zp};
        std::vector<PortRef> refs{d.ref, w.ref};
        if (ins.size() > 2 && prod[2] >= 0) {
          // bias quantized to the accumulator at s_data * s_weight
          const Node& b = g_.node(prod[2]);
          const double sb = d.scale * w.scale;
          auto bf = b.payload->floats();
          std::vector<int32_t> bq(bf.size());
          for (size_t i = 0; i < bf.size(); ++i) {
            const int64_t q = std::llround(static_cast<double>(bf[i]) / sb);
            bq[i] = static_cast<int32_t>(std::clamp(q, acc.min_value(), acc.max_value()));
          }
          Node k = fresh(OpKind::kConstant);
          k.payload = Tensor::from_ints(acc, b.payload->shape(), std::move(bq));
          refs.push_back(PortRef{emit(std::move(k), {}), 0});
        }
        res.integer = true;
        res.scale = d.scale * w.scale;
        res.zp = 0;
        res.dtype = acc;
        res.ref = PortRef{emit(std::move(out), refs), 0};
        dom_[n.id] = res;
        return;
      }
      case OpKind::kAdd: {
        const Dom& a = ins.at(0);
        const Dom& b = ins.at(1);
        if (a.integer != b.integer) {
          throw RealizeError("add node " + std::to_string(n.id) + " mixes quantized and float inputs");
        }
        if (!a.integer) break;
        // unified scale: the input with the larger threshold (SPEC realize)
        const int keep = b.threshold > a.threshold ? 1 : 0;
        const Dom& u = ins[static_cast<size_t>(keep)];
        const Dom& other = ins[static_cast<size_t>(1 - keep)];
        EdgeDecision target;
        target.threshold = u.threshold;
        target.zero_point = u.zp;
        target.storage_dtype = u.dtype;
        target.bit = decs[static_cast<size_t>(keep)] ? decs[static_cast<size_t>(keep)]->bit : max_bits(u.dtype);
        target.sign = decs[static_cast<size_t>(keep)] ? decs[static_cast<size_t>(keep)]->sign
                                                      : (u.dtype.is_signed() ? 1 : 0);
        Dom moved = to_grid(other, target);
        std::vector<Dom> both(2);
        both[static_cast<size_t>(keep)] = u;
        both[static_cast<size_t>(1 - keep)] = moved;
        const DType acc = acc_dtype(n.op, both, {decs[static_cast<size_t>(keep)],
                                                 decs[static_cast<size_t>(keep)]});
        out.attrs["acc_dtype"] = acc.name();
        res.integer = true;
        res.scale = u.scale;
        res.threshold = u.threshold;
        res.zp = both[0].zp + both[1].zp;
        res.dtype = acc;
        res.ref = PortRef{emit(std::move(out), {both[0].ref, both[1].ref}), 0};
        dom_[n.id] = res;
        return;
      }
      case OpKind::kRelu:
        if (ins.at(0).integer) out.attrs["zero_point"] = ins[0].zp;
        res = ins[0];
        res.ref = PortRef{emit(std::move(out), {ins[0].ref}), 0};
        dom_[n.id] = res;
        return;
      case OpKind::kClip:
        if (ins.at(0).integer) {
          const auto qc = rewrite_clip(n.attr<double>("a_min"), n.attr<double>("a_max"), ins[0].scale,
                                       ins[0].zp, ins[0].dtype);
          out.attrs["q_min"] = qc.first;
          out.attrs["q_max"] = qc.second;
        }
        res = ins[0];
        res.ref = PortRef{emit(std::move(out), {ins[0].ref}), 0};
        dom_[n.id] = res;
        return;
      case OpKind::kMaxPool2d:
      case OpKind::kFlatten:
        res = ins.at(0);
        res.ref = PortRef{emit(std::move(out), {ins[0].ref}), 0};
        dom_[n.id] = res;
        return;
      default:
        break;
    }
    // float op: every operand as a float value
    std::vector<PortRef> refs;
    for (size_t i = 0; i < ins.size(); ++i) {
      refs.push_back(prod[i] >= 0 ? as_float(ins[i]).ref : PortRef{-1, 0});
    }
    res = Dom{};
    res.ref = PortRef{emit(std::move(out), refs), 0};
    dom_[n.id] = res;
  }

  const Graph& g_;
  const Strategy& st_;
  const HardwareSpec& spec_;
  NodeId next_id_;
  std::vector<Node> nodes_;
  std::vector<Edge> edges_;
  std::map<NodeId, Dom> dom_;
  std::map<NodeId, const EdgeDecision*> sq_dec_;
  std::set<NodeId> consts_;
  std::map<NodeId, Dom> const_copy_;
};

}  // namespace

// SPEC.md realize module (:629-640): lower the simulated graph bound with
// `strategy` into an integer graph — weights folded to integer constants,
// quantize at fp32->int boundaries, requantize for int->int scale changes
// (requantize_params), add inputs on the larger-threshold scale, clip bounds
// via rewrite_clip, dequantize at int->fp32 boundaries, accumulator dtypes
// from the matched hardware signatures, biases quantized at s_data*s_weight.
Graph realize(const Graph& sim_g, const Strategy& strategy, const HardwareSpec& spec) {
  Graph out = Lowering(sim_g, strategy, spec).run();
  auto v = validate_graph(out);
  if (!v.empty()) throw RealizeError("realized graph is invalid: " + v.front().message);
  if (out.contains_op(OpKind::kSimulatedQuantize)) {
    throw RealizeError("realized graph still contains simulated_quantize nodes");
  }
  return out;
}

}  // namespace quantc
