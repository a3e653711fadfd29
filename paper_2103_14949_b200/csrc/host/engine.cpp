// engine.cpp — GPU graph executor (see engine.hpp).
//
// Op semantics follow reference interpreter.cpp:113-482 node by node; every
// kernel it launches is documented with the reference lines it reproduces.
#include "engine.hpp"

#include <algorithm>
#include <chrono>
#include <map>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <limits>
#include <list>
#include <mutex>
#include <stdexcept>

#include "quantc/device.hpp"
#include "quantc/simulate.hpp"

namespace quantc::engine {

namespace {

cudaStream_t S() { return static_cast<cudaStream_t>(device::stream()); }

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

int64_t i64(const Json& j) { return j.get<int64_t>(); }

struct Attr2 {
  int a, b;
};
Attr2 pair_attr(const Node& n, const char* key, Attr2 dflt) {
  if (!n.has_attr(key)) return dflt;
  auto v = n.attr<std::vector<int64_t>>(key);
  if (v.size() != 2) throw EvalError(std::string(key) + " must be 2d at node " + std::to_string(n.id));
  return {static_cast<int>(v[0]), static_cast<int>(v[1])};
}

bool is_pow2(double t) {
  if (!(t > 0.0) || !std::isfinite(t)) return false;
  int e = 0;
  return std::frexp(t, &e) == 0.5;
}

// per-sample output shape inference (mirrors validate_graph's rules)
std::vector<int64_t> infer_shape(const Node& n, const std::vector<const std::vector<int64_t>*>& in) {
  auto need = [&](size_t i) -> const std::vector<int64_t>& {
    if (i >= in.size() || !in[i]) {
      throw EvalError(op_name(n.op) + " node " + std::to_string(n.id) + " missing input " +
                      std::to_string(i));
    }
    return *in[i];
  };
  switch (n.op) {
    case OpKind::kInput:
      return n.attr<std::vector<int64_t>>("shape");
    case OpKind::kConstant:
      return n.payload->shape();
    case OpKind::kConv2d: {
      const auto &d = need(0), &w = need(1);
      const int64_t groups = n.attr_or<int64_t>("groups", 1);
      if (d.size() != 4 || w.size() != 4 || groups < 1 || w[0] % groups != 0 ||
          d[1] != w[1] * groups) {
        throw EvalError("conv2d shape mismatch at node " + std::to_string(n.id));
      }
      Attr2 st = pair_attr(n, "strides", {1, 1}), pd = pair_attr(n, "padding", {0, 0});
      return {d[0], w[0], (d[2] + 2 * pd.a - w[2]) / st.a + 1, (d[3] + 2 * pd.b - w[3]) / st.b + 1};
    }
    case OpKind::kDense: {
      const auto &d = need(0), &w = need(1);
      if (d.size() != 2 || w.size() != 2 || d[1] != w[1]) {
        throw EvalError("dense shape mismatch at node " + std::to_string(n.id));
      }
      return {d[0], w[0]};
    }
    case OpKind::kAdd: {
      const auto &a = need(0), &b = need(1);
      if (a != b) throw EvalError("add operand shapes differ at node " + std::to_string(n.id));
      return a;
    }
    case OpKind::kMaxPool2d: {
      const auto& d = need(0);
      auto k = n.attr<std::vector<int64_t>>("pool_size");
      Attr2 st = pair_attr(n, "strides", {static_cast<int>(k[0]), static_cast<int>(k[1])});
      Attr2 pd = pair_attr(n, "padding", {0, 0});
      return {d[0], d[1], (d[2] + 2 * pd.a - k[0]) / st.a + 1, (d[3] + 2 * pd.b - k[1]) / st.b + 1};
    }
    case OpKind::kGlobalAvgPool2d: {
      const auto& d = need(0);
      return {d[0], d[1], 1, 1};
    }
    case OpKind::kAvgPool2d: {
      const auto& d = need(0);
      auto k = n.attr<std::vector<int64_t>>("pool_size");
      Attr2 st = pair_attr(n, "strides", {static_cast<int>(k[0]), static_cast<int>(k[1])});
      Attr2 pd = pair_attr(n, "padding", {0, 0});
      return {d[0], d[1], (d[2] + 2 * pd.a - k[0]) / st.a + 1, (d[3] + 2 * pd.b - k[1]) / st.b + 1};
    }
    case OpKind::kConcat: {
      std::vector<int64_t> out = need(0);
      for (size_t i = 1; i < in.size(); ++i) {
        const auto& d = need(i);
        if (d.size() != 4 || out.size() != 4 || d[0] != out[0] || d[2] != out[2] || d[3] != out[3]) {
          throw EvalError("concat operand shapes differ at node " + std::to_string(n.id));
        }
        out[1] += d[1];
      }
      return out;
    }
    case OpKind::kFlatten: {
      const auto& d = need(0);
      int64_t rest = 1;
      for (size_t i = 1; i < d.size(); ++i) rest *= d[i];
      return {d[0], rest};
    }
    default:
      return need(0);
  }
}

}  // namespace

std::shared_ptr<void> device_alloc(size_t bytes) { return device_alloc_on(S(), bytes); }

std::shared_ptr<void> device_alloc_on(void* stream, size_t bytes) {
  void* p = nullptr;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (bytes == 0) bytes = 16;
  cuda_ok(cudaMallocAsync(&p, bytes, s), "cudaMallocAsync");
  return std::shared_ptr<void>(p, [s](void* q) { cudaFreeAsync(q, s); });
}

QParams qparams_of(const Node& n, const SimBinding* binding) {
  if (binding) {
    auto it = binding->find(n.id);
    if (it != binding->end()) return it->second;
  }
  // reference interpreter.cpp:47-63 (qparams_from_attrs)
  QParams p;
  p.passthrough = n.attr_or<bool>("passthrough", true);
  if (!p.passthrough) {
    p.threshold = n.attr<double>("threshold");
    p.bit = n.attr<int>("bit");
    p.sign = n.attr<int>("sign");
    p.zero_point = n.attr_or<int64_t>("zero_point", 0);
    p.in_dtype = parse_dtype(n.attr_or<std::string>("in_dtype", "int8"));
    p.out_dtype = parse_dtype(n.attr_or<std::string>("out_dtype", p.in_dtype.name()));
  }
  if (n.has_attr("acc_dtype")) {
    p.acc_dtype = parse_dtype(n.attr<std::string>("acc_dtype"));
    p.acc_scale = n.attr<double>("acc_scale");
  }
  return p;
}

kern::SqParams resolve_sq(const QParams& p) {
  // check_params (reference simulate.cpp:47-60)
  if (!p.passthrough) {
    if (!(p.threshold > 0.0)) throw std::invalid_argument("QParams: threshold must be positive");
    if (p.bit < 2) throw std::invalid_argument("QParams: bit must be >= 2");
    if (p.in_dtype.is_integer()) {
      if (p.bit > max_bits(p.in_dtype)) {
        throw std::invalid_argument("QParams: bit exceeds storage dtype width");
      }
      if (p.sign != (p.in_dtype.is_signed() ? 1 : 0)) {
        throw std::invalid_argument("QParams: sign incompatible with storage dtype");
      }
    }
  }
  kern::SqParams k{};
  k.has_acc = p.acc_dtype.has_value() && p.acc_scale > 0.0;
  if (k.has_acc) {
    k.lo = static_cast<double>(p.acc_dtype->min_value()) * p.acc_scale;
    k.hi = static_cast<double>(p.acc_dtype->max_value()) * p.acc_scale;
  }
  k.passthrough = p.passthrough ? 1 : 0;
  if (!p.passthrough) {
    k.s = compute_scale(p.threshold, p.bit, p.sign);
    QuantBounds b = quant_bounds(p.bit, p.sign);
    k.qmin = static_cast<double>(b.qmin);
    k.qmax = static_cast<double>(b.qmax);
    k.zp = static_cast<double>(p.zero_point);
    k.inv_s = 1.0 / k.s;
    k.exact_div = std::isfinite(k.inv_s) && k.inv_s != 0.0 ? 0 : 1;
  }
  return k;
}

DevTensor upload(const Tensor& t) {
  DevTensor d;
  d.dtype = t.dtype();
  d.shape = t.shape();
  d.batched = false;
  const size_t bytes = static_cast<size_t>(t.numel()) * 4;
  d.buf = device_alloc(bytes);
  const void* src = t.dtype().is_float() ? static_cast<const void*>(t.floats().data())
                                         : static_cast<const void*>(t.ints().data());
  if (bytes) cuda_ok(cudaMemcpyAsync(d.buf.get(), src, bytes, cudaMemcpyHostToDevice, S()), "upload");
  return d;
}

Tensor download(const DevTensor& d, int batch) {
  std::vector<int64_t> shape = d.shape;
  if (d.batched && !shape.empty()) shape[0] *= batch;
  const int64_t n = shape_numel(shape);
  if (d.dtype.is_float()) {
    std::vector<float> h(static_cast<size_t>(n));
    if (n) cuda_ok(cudaMemcpyAsync(h.data(), d.buf.get(), n * 4, cudaMemcpyDeviceToHost, S()), "download");
    device::synchronize();
    return Tensor::from_floats(shape, std::move(h));
  }
  std::vector<int32_t> h(static_cast<size_t>(n));
  if (n) cuda_ok(cudaMemcpyAsync(h.data(), d.buf.get(), n * 4, cudaMemcpyDeviceToHost, S()), "download");
  device::synchronize();
  return Tensor::from_ints(d.dtype, shape, std::move(h));
}

// ---- plan cache -------------------------------------------------------------------

struct PlanLease::Entry {
  uint64_t uid = 0;
  std::mutex m;
  std::unique_ptr<Plan> plan;
};

PlanLease lease_plan(const Graph& g) {
  static std::mutex mu;
  static std::list<std::shared_ptr<PlanLease::Entry>> lru;  // most recent first
  static const size_t cap = [] {
    const char* e = std::getenv("QUANTC_PLAN_CACHE");
    return e ? static_cast<size_t>(std::max(0, std::atoi(e))) : size_t{2};
  }();
  PlanLease l;
  if (cap == 0) {
    l.own_ = std::make_unique<Plan>(g);
    l.plan_ = l.own_.get();
    return l;
  }
  std::shared_ptr<PlanLease::Entry> e;
  {
    std::lock_guard<std::mutex> lk(mu);
    for (auto it = lru.begin(); it != lru.end(); ++it) {
      if ((*it)->uid == g.uid()) {
        e = *it;
        lru.erase(it);
        break;
      }
    }
    if (!e) {
      e = std::make_shared<PlanLease::Entry>();
      e->uid = g.uid();
    }
    lru.push_front(e);
    while (lru.size() > cap) lru.pop_back();  // leased entries stay alive with their lease
  }
  auto lock = std::make_shared<std::unique_lock<std::mutex>>(e->m);
  if (!e->plan) e->plan = std::make_unique<Plan>(g);
  l.entry_ = e;
  l.lock_ = lock;
  l.plan_ = e->plan.get();
  return l;
}

// ---- Plan ----------------------------------------------------------------------

Plan::Plan(const Graph& g) : g_(g) {
  const std::vector<NodeId> order = traversal_order(g);
  steps_.resize(order.size());
  shapes_.resize(order.size());
  batched_.assign(order.size(), 0);
  for (size_t i = 0; i < order.size(); ++i) index_[order[i]] = static_cast<int>(i);
  for (size_t i = 0; i < order.size(); ++i) {
    Step& st = steps_[i];
    st.node = &g.node(order[i]);
    for (const Edge* e : g.in_edges(order[i])) {
      st.in.push_back(e ? index_.at(e->src.node) : -1);
      if (e) steps_[static_cast<size_t>(index_.at(e->src.node))].uses++;
    }
  }
  for (const PortRef& o : g.outputs()) {
    auto it = index_.find(o.node);
    if (it != index_.end()) steps_[static_cast<size_t>(it->second)].uses++;
  }
  // shapes, batchedness, constants, liveness peak
  int64_t live = 0;
  std::vector<int> remaining(steps_.size());
  for (size_t i = 0; i < steps_.size(); ++i) remaining[i] = steps_[i].uses;
  for (size_t i = 0; i < steps_.size(); ++i) {
    const Step& st = steps_[i];
    std::vector<const std::vector<int64_t>*> ins;
    bool any_batched = st.node->op == OpKind::kInput;
    for (int p : st.in) {
      ins.push_back(p >= 0 ? &shapes_[static_cast<size_t>(p)] : nullptr);
      if (p >= 0 && batched_[static_cast<size_t>(p)]) any_batched = true;
    }
    if (st.node->op == OpKind::kConstant) {
      if (!st.node->payload) throw EvalError("constant node missing payload");
      constants_[static_cast<int>(i)] = upload(*st.node->payload);
    }
    try {
      shapes_[i] = infer_shape(*st.node, ins);
    } catch (const EvalError&) {
      throw;
    } catch (const std::exception& e) {
      throw EvalError(std::string("shape inference failed at node ") +
                      std::to_string(st.node->id) + ": " + e.what());
    }
    batched_[i] = any_batched ? 1 : 0;
    if (any_batched && st.node->op != OpKind::kInput && st.node->op != OpKind::kFlatten) {
      live += shape_numel(shapes_[i]) * 4;
      peak_bytes_ = std::max(peak_bytes_, live);
    }
    for (int p : st.in) {
      if (p < 0) continue;
      if (--remaining[static_cast<size_t>(p)] == 0 && batched_[static_cast<size_t>(p)] &&
          steps_[static_cast<size_t>(p)].node->op != OpKind::kInput &&
          steps_[static_cast<size_t>(p)].node->op != OpKind::kFlatten) {
        live -= shape_numel(shapes_[static_cast<size_t>(p)]) * 4;
      }
    }
  }
  // im2col / code buffers of the fast path need headroom
  peak_bytes_ = peak_bytes_ * 2 + (1 << 20);
  device::synchronize();
}

int Plan::batch_for(int64_t n_samples) const {
  const int64_t budget = static_cast<int64_t>(device::memory_budget_bytes());
  int64_t b = std::max<int64_t>(1, budget / std::max<int64_t>(1, peak_bytes_));
  b = std::min<int64_t>(b, 1024);
  return static_cast<int>(std::min<int64_t>(b, std::max<int64_t>(1, n_samples)));
}

// ---- run -------------------------------------------------------------------------

namespace {

struct Runner {
  const Plan& plan;
  const RunSpec& spec;
  std::vector<DevTensor> vals;
  std::vector<int> remaining;
  std::vector<char> keep;
  std::vector<char> fast_conv;        // conv/dense step uses the tcgen05 path
  std::vector<char> codes_only;       // sq step feeding a fast conv emits codes only
  std::vector<std::shared_ptr<void>> codes;  // int8 codes per sq step
  std::vector<int> code_cpad;
  std::vector<int> code_kpad;
  std::vector<kern::SqParams> sqp;
  std::vector<QParams> qp;
  std::shared_ptr<void> trap;
  std::vector<char> done;  // computed by a fused producer (requantize after an int conv)

  Runner(const Plan& p, const RunSpec& s) : plan(p), spec(s) {
    const size_t n = p.steps().size();
    vals.resize(n);
    done.assign(n, 0);
    remaining.resize(n);
    keep.assign(n, 0);
    fast_conv.assign(n, 0);
    codes_only.assign(n, 0);
    codes.resize(n);
    code_cpad.assign(n, 0);
    code_kpad.assign(n, 0);
    sqp.resize(n);
    qp.resize(n);
    for (size_t i = 0; i < n; ++i) remaining[i] = p.steps()[i].uses;
    for (int k : s.keep) keep[static_cast<size_t>(k)] = 1;
  }

  int64_t N(int step) const { return plan.batched(step) ? spec.batch : 1; }

  const DevTensor& in(int step, int port) {
    const auto& st = plan.steps()[static_cast<size_t>(step)];
    if (port >= static_cast<int>(st.in.size()) || st.in[static_cast<size_t>(port)] < 0) {
      throw EvalError(op_name(st.node->op) + " node " + std::to_string(st.node->id) +
                      " missing input " + std::to_string(port));
    }
    return vals[static_cast<size_t>(st.in[static_cast<size_t>(port)])];
  }

  DevTensor out_like(int step, DType dt) {
    DevTensor d;
    d.dtype = dt;
    d.shape = plan.shape(step);
    d.batched = plan.batched(step);
    d.buf = device_alloc(static_cast<size_t>(d.numel(spec.batch)) * 4);
    return d;
  }

  unsigned long long* trap_ptr() {
    if (spec.mode != OverflowMode::kTrap) return nullptr;
    if (!trap) trap = device_alloc(8);
    unsigned long long init = ~0ull;
    cuda_ok(cudaMemcpyAsync(trap.get(), &init, 8, cudaMemcpyHostToDevice, S()), "trap init");
    return static_cast<unsigned long long*>(trap.get());
  }
  int64_t trapped() {
    unsigned long long h = ~0ull;
    cuda_ok(cudaMemcpyAsync(&h, trap.get(), 8, cudaMemcpyDeviceToHost, S()), "trap read");
    device::synchronize();
    return h == ~0ull ? -1 : static_cast<int64_t>(h);
  }

  DType acc_dtype_of(const Node& n) const {
    if (!n.has_attr("acc_dtype")) {
      throw EvalError("node " + std::to_string(n.id) + " (" + op_name(n.op) +
                      ") missing accumulator dtype annotation");
    }
    return parse_dtype(n.attr<std::string>("acc_dtype"));
  }

  void require_int_regime(const Node& n) {
    if (!spec.integer_regime) {
      throw EvalError("op " + op_name(n.op) + " (node " + std::to_string(n.id) +
                      ") is not supported in the fp32 regime");
    }
  }

  // ---- fast-path planning: decide per conv/dense whether its two MAC
  // operands are int8-grid sq outputs the tcgen05 kernel can consume.
  void plan_fast() {
    if (!spec.allow_fast || spec.integer_regime || !kern::gemm_s8_tcgen05_available()) return;
    const auto mode = device::engine_mode();
    if (mode == device::EngineMode::kExact) return;
    const auto& steps = plan.steps();
    for (size_t i = 0; i < steps.size(); ++i) {
      const auto& st = steps[i];
      if (st.node->op == OpKind::kSimulatedQuantize) {
        qp[i] = qparams_of(*st.node, spec.binding);
        sqp[i] = resolve_sq(qp[i]);
      }
    }
    for (size_t i = 0; i < steps.size(); ++i) {
      const auto& st = steps[i];
      if (st.node->op != OpKind::kConv2d && st.node->op != OpKind::kDense) continue;
      if (st.node->attr_or<int64_t>("groups", 1) != 1) continue;  // grouped: FP64 / int64 kernels
      if (st.in.size() < 2 || st.in[0] < 0 || st.in[1] < 0) continue;
      const int d = st.in[0], w = st.in[1];
      const auto &sd = steps[static_cast<size_t>(d)], &sw = steps[static_cast<size_t>(w)];
      if (sd.node->op != OpKind::kSimulatedQuantize || sw.node->op != OpKind::kSimulatedQuantize) continue;
      if (sd.uses != 1 || sw.uses != 1 || keep[static_cast<size_t>(d)] || keep[static_cast<size_t>(w)]) continue;
      if (!plan.batched(d) || plan.batched(w)) continue;
      if (st.in.size() > 2 && st.in[2] >= 0 && plan.batched(st.in[2])) continue;
      bool ok = true;
      for (int s : {d, w}) {
        const QParams& q = qp[static_cast<size_t>(s)];
        ok = ok && !q.passthrough && q.sign == 1 && q.zero_point == 0 && q.bit <= 8;
        if (mode == device::EngineMode::kAuto) ok = ok && is_pow2(q.threshold);
      }
      // the producer of the sq inputs must be float tensors
      if (!ok) continue;
      fast_conv[i] = 1;
      codes_only[static_cast<size_t>(d)] = 1;
      codes_only[static_cast<size_t>(w)] = 1;
    }
  }

  void release_inputs(int step) {
    for (int p : plan.steps()[static_cast<size_t>(step)].in) {
      if (p < 0) continue;
      if (--remaining[static_cast<size_t>(p)] == 0 && !keep[static_cast<size_t>(p)]) {
        vals[static_cast<size_t>(p)] = DevTensor{};
        codes[static_cast<size_t>(p)].reset();
      }
    }
  }

  void exec(int i);
  void exec_conv(int i, bool dense);
  bool exec_conv_int_tc(int i, bool dense, const kern::ConvShape& cs, const DevTensor& d,
                        const DevTensor& w, const DevTensor* b, DType acc,
                        const std::vector<int64_t>& zps);
  bool exec_conv_int_simt(int i, const kern::ConvShape& cs, const DevTensor& d,
                          const DevTensor& w, const DevTensor* b, DType acc,
                          const std::vector<int64_t>& zps);
  std::vector<int> fused_chain(int i, bool allow_add = false) const;
  DType chain_dtype(const std::vector<int>& chain, DType acc) const;
  void fill_posts(kern::IntEpi& ie, int i, const std::vector<int>& chain) const;
  void finish_int(int i, const std::vector<int>& chain, const DevTensor& y, const kern::ConvShape& cs,
                  const DevTensor& d, const DevTensor& w, const DevTensor* b,
                  const std::vector<int64_t>& zps);
  void exec_conv_fast(int i, bool dense);
  void exec_sq(int i);
  void exec_sq_codes(int i);
};

// Realized-graph int8 x int8 conv/dense on tcgen05 (SURVEY §8(a) a7/a8 with
// the a9 requantize fused): codes packed NHWC, weights packed K-major with
// zp1 folded (when w - zp1 fits int8), the exact int32 tensor-core sum,
// and the IntEpi epilogue (zp0 correction, bias, accumulator clamp / trap,
// requantize of a sole requantize consumer).  Returns false when the layer
// does not qualify (the int64 CUDA-core kernel then runs).
bool Runner::exec_conv_int_tc(int i, bool dense, const kern::ConvShape& cs, const DevTensor& d,
                              const DevTensor& w, const DevTensor* b, DType acc,
                              const std::vector<int64_t>& zps) {
  static const bool off = [] {
    const char* e = std::getenv("QUANTC_INT_TC");
    return e && std::string(e) == "0";
  }();
  if (off || !kern::gemm_s8_tcgen05_available()) return false;
  // 8-bit (or narrower) data codes; the weights' range is checked on device
  if (!d.dtype.is_integer() || d.dtype.width() > 8 || !w.dtype.is_integer()) return false;
  if (acc.width() > 32) return false;
  // the int16-accumulator signature is the CUDA-core backend's
  // (exec_conv_int_simt) unless QUANTC_INT16_ON_TC=1
  static const bool i16_on_tc = [] {
    const char* e = std::getenv("QUANTC_INT16_ON_TC");
    return e && std::string(e) == "1";
  }();
  if (acc.width() <= 16 && !i16_on_tc) return false;

  const int taps = cs.KH * cs.KW;
  const int ld = (cs.C + 15) / 16 * 16;
  const bool direct = dense || (taps == 1 && cs.sh == 1 && cs.sw == 1 && cs.ph == 0 &&
                                cs.pw == 0 && ld == cs.C);
  if (!direct && taps > 63) return false;
  const int Ktrue = direct ? ld : taps * ld;
  const int Kpad = (Ktrue + 127) / 128 * 128;
  if (static_cast<int64_t>(Ktrue) * 255 * 128 >= (int64_t{1} << 31)) return false;  // int32 TMEM sum
  // weights: w - zp1 as int8 codes [O][Kpad] and their per-row sums
  // packed weights: once per plan and layer (the range check reads one flag)
  auto key = std::make_pair(i, 0);
  auto wit = plan.int_weights.find(key);
  if (wit == plan.int_weights.end()) {
    Plan::IntWeights iw;
    iw.codes = device_alloc(static_cast<size_t>(cs.O) * Kpad + 16);
    iw.wsum = device_alloc(static_cast<size_t>(cs.O) * 4 + 16);
    int* bad = reinterpret_cast<int*>(static_cast<int8_t*>(iw.wsum.get()) + static_cast<size_t>(cs.O) * 4);
    cuda_ok(cudaMemsetAsync(iw.wsum.get(), 0, static_cast<size_t>(cs.O) * 4 + 16, S()), "wsum");
    kern::pack_i32_weights(w.i(), static_cast<int8_t*>(iw.codes.get()), static_cast<int32_t*>(iw.wsum.get()),
                           bad, cs.O, cs.C, taps, ld, Kpad, zps.at(1), S());
    int hbad = 0;
    cuda_ok(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, S()), "pack flag");
    device::synchronize();
    iw.ok = hbad == 0;
    wit = plan.int_weights.emplace(key, iw).first;
  }
  if (!wit->second.ok) return false;
  const std::shared_ptr<void>& wcodes = wit->second.codes;
  const std::shared_ptr<void>& wsum = wit->second.wsum;
  // data codes NHWC.  The reference skips padded taps, i.e. they add
  // (zp0 - zp0) * w = 0; with zp0 != 0 the border is materialised as zp0 so
  // that acc - zp0 * wsum stays exact, otherwise the gather's zero fill is.
  const bool pad_fill = zps.at(0) != 0 && (cs.ph != 0 || cs.pw != 0);
  const int pph = pad_fill ? cs.ph : 0, ppw = pad_fill ? cs.pw : 0;
  const int HP = cs.H + 2 * pph, WP = cs.W + 2 * ppw;
  std::shared_ptr<void> xcodes;
  if (d.codes && d.codes_ld == ld && !pad_fill) {
    xcodes = d.codes;  // the producer's epilogue already wrote them
  } else {
    xcodes = device_alloc(static_cast<size_t>(cs.N) * HP * WP * ld + 64);
    kern::pack_i32_nhwc(d.i(), static_cast<uint8_t*>(xcodes.get()), cs.N, cs.C, cs.H, cs.W, pph,
                        ppw, ld, static_cast<int32_t>(zps.at(0)), S());
  }
  const std::vector<int> chain = fused_chain(i, true);
  const int last = chain.empty() ? i : chain.back();
  const DType ydt = chain_dtype(chain, acc);
  DevTensor y = out_like(last, ydt);
  // side output of the final values' code bytes when an integer conv/dense
  // consumes them (its input pack is then skipped)
  int64_t code_rows = 0;
  int code_ld = 0;
  if (ydt.width() <= 8 && !keep[static_cast<size_t>(last)]) {
    const auto& steps = plan.steps();
    for (size_t j = static_cast<size_t>(last) + 1; j < steps.size(); ++j) {
      const auto& sj = steps[j];
      const OpKind op = sj.node->op;
      if ((op == OpKind::kConv2d || op == OpKind::kDense) && !sj.in.empty() && sj.in[0] == last) {
        code_rows = static_cast<int64_t>(cs.N) * cs.OH * cs.OW;
        code_ld = (cs.O + 15) / 16 * 16;
        break;
      }
    }
  }
  if (code_rows > 0 && !dense) {
    y.codes = device_alloc(static_cast<size_t>(code_rows) * code_ld + 64);
    y.codes_ld = code_ld;
  }
  kern::TcConvSpec sp{};
  sp.x = static_cast<const int8_t*>(xcodes.get());
  sp.w = static_cast<const int8_t*>(wcodes.get());
  sp.M = static_cast<int64_t>(cs.N) * cs.OH * cs.OW;
  sp.O = cs.O;
  sp.Kpad = Kpad;
  sp.gather = direct ? 0 : 1;
  sp.Ktrue = Ktrue;
  sp.lda = ld;
  sp.Nimg = cs.N;
  sp.H = HP;
  sp.W = WP;
  sp.C = cs.C;
  sp.ld = ld;
  sp.KH = cs.KH;
  sp.KW = cs.KW;
  sp.sh = cs.sh;
  sp.sw = cs.sw;
  sp.ph = cs.ph - pph;
  sp.pw = cs.pw - ppw;
  sp.OH = cs.OH;
  sp.OW = cs.OW;
  sp.prog = kern::ProgArgs{nullptr, 0, kern::kShapeInt};
  kern::IntEpi& ie = sp.iepi;
  ie.y = y.i();
  ie.bias = b ? b->i() : nullptr;
  ie.zp0 = zps.at(0);
  ie.wsum = ie.zp0 != 0 ? static_cast<const int32_t*>(wsum.get()) : nullptr;
  ie.trap = trap_ptr();
  ie.acc_min = acc.min_value();
  ie.acc_max = acc.max_value();
  ie.OHW = cs.OH * cs.OW;
  ie.a_unsigned = d.dtype.is_signed() ? 0 : 1;
  ie.codes = static_cast<uint8_t*>(y.codes.get());
  ie.codes_ld = y.codes_ld;
  fill_posts(ie, i, chain);
  {
    static const bool off32 = std::getenv("QUANTC_NO_INT_FAST32") != nullptr;
    bool f32ok = !off32;
    for (int k = 0; k < ie.n_post; ++k) {
      const kern::IntEpi::Post& p = ie.post[k];
      if (p.kind == kern::kPostRequantize) {
        f32ok = f32ok && p.mult == (1 << 30) && p.shift >= 30 && p.shift < 61 &&
                std::abs(p.in_zp) < (1 << 16) && std::abs(p.out_zp) < (1 << 16);
      } else if (p.kind == kern::kPostAdd) {
        // the other operand of the add at chain position k
        const int run = k == 0 ? i : chain[static_cast<size_t>(k - 1)];
        const auto& in = plan.steps()[static_cast<size_t>(chain[static_cast<size_t>(k)])].in;
        const int other = in[0] == run ? in[1] : in[0];
        f32ok = f32ok && vals[static_cast<size_t>(other)].dtype.width() <= 16;
      } else if (p.kind == kern::kPostRelu) {
        f32ok = f32ok && std::abs(p.out_zp) < (1 << 16);
      }
    }
    ie.fast32 = f32ok ? 1 : 0;
  }
  kern::tc_conv(sp, S());
  device::counters().tcgen05_gemms++;
  finish_int(i, chain, y, cs, d, w, b, zps);
  return true;
}

// the sole-consumer chain after integer conv/dense step i that the
// epilogue absorbs: up to three requantize / relu steps, each the only
// consumer of the previous value and not a kept (output) value
std::vector<int> Runner::fused_chain(int i, bool allow_add) const {
  std::vector<int> chain;
  if (!spec.integer_regime) return chain;
  static const bool no_add = std::getenv("QUANTC_NO_INT_ADD_FUSION") != nullptr;
  const auto& steps = plan.steps();
  int cur = i;
  DType cur_dt = acc_dtype_of(*steps[static_cast<size_t>(i)].node);
  bool added = false;
  while (static_cast<int>(chain.size()) < kern::kMaxIntPosts) {
    if (steps[static_cast<size_t>(cur)].uses != 1 || keep[static_cast<size_t>(cur)]) break;
    int next = -1;
    for (size_t j = static_cast<size_t>(cur) + 1; j < steps.size(); ++j) {
      const auto& sj = steps[j];
      if (std::find(sj.in.begin(), sj.in.end(), cur) != sj.in.end()) {
        next = static_cast<int>(j);
        break;
      }
    }
    if (next < 0) break;
    const auto& sn = steps[static_cast<size_t>(next)];
    const OpKind op = sn.node->op;
    if (op == OpKind::kAdd && allow_add && !no_add && sn.in.size() == 2 && !added) {
      // an integer add whose other operand is already computed (an earlier
      // step), of the same batched shape, and whose accumulator provably
      // cannot overflow given both operands' dtypes (no trap to report)
      const int other = sn.in[0] == cur ? sn.in[1] : sn.in[0];
      if (other < 0 || other >= i || sn.in[0] == sn.in[1]) break;
      const DevTensor& ov = vals[static_cast<size_t>(other)];
      if (!ov.buf || !ov.dtype.is_integer() || ov.batched != plan.batched(cur) ||
          ov.per_numel() != shape_numel(plan.shape(cur))) {
        break;
      }
      const DType add_acc = acc_dtype_of(*sn.node);
      const int64_t lo = cur_dt.min_value() + ov.dtype.min_value();
      const int64_t hi = cur_dt.max_value() + ov.dtype.max_value();
      if (lo < add_acc.min_value() || hi > add_acc.max_value()) break;
      chain.push_back(next);
      cur = next;
      cur_dt = add_acc;
      added = true;  // one add per chain (the epilogue prefetches one operand)
      continue;
    }
    if (op != OpKind::kRequantize && op != OpKind::kRelu) break;
    if (sn.in.size() != 1) break;
    chain.push_back(next);
    cur = next;
    if (op == OpKind::kRequantize) cur_dt = parse_dtype(sn.node->attr<std::string>("out_dtype"));
  }
  return chain;
}

// dtype of the chain's last value (requantize: out_dtype; relu: its input's)
DType Runner::chain_dtype(const std::vector<int>& chain, DType acc) const {
  DType dt = acc;
  for (int j : chain) {
    const Node& n = *plan.steps()[static_cast<size_t>(j)].node;
    if (n.op == OpKind::kRequantize) dt = parse_dtype(n.attr<std::string>("out_dtype"));
    if (n.op == OpKind::kAdd) dt = parse_dtype(n.attr<std::string>("acc_dtype"));
  }
  return dt;
}

void Runner::fill_posts(kern::IntEpi& ie, int i, const std::vector<int>& chain) const {
  ie.n_post = 0;
  int run = i;  // the step whose value the chain element consumes
  for (int j : chain) {
    const Node& n = *plan.steps()[static_cast<size_t>(j)].node;
    kern::IntEpi::Post& p = ie.post[ie.n_post++];
    p = kern::IntEpi::Post{};
    if (n.op == OpKind::kRelu) {
      p.kind = kern::kPostRelu;
      p.out_zp = static_cast<int32_t>(n.attr_or<int64_t>("zero_point", 0));
    } else if (n.op == OpKind::kAdd) {
      // the operand that is not the chain's running value
      const auto& in = plan.steps()[static_cast<size_t>(j)].in;
      const int other = in[0] == run ? in[1] : in[0];
      p.kind = kern::kPostAdd;
      p.other = vals[static_cast<size_t>(other)].i();
    } else {
      p.kind = kern::kPostRequantize;
      const int64_t mult = n.attr<int64_t>("multiplier");
      const int shift = n.attr<int>("shift");
      if (mult < INT32_MIN || mult > INT32_MAX || shift < -32768 || shift > 32767) {
        throw EvalError("requantize multiplier/shift out of range at node " + std::to_string(n.id));
      }
      p.mult = static_cast<int32_t>(mult);
      p.shift = static_cast<int16_t>(shift);
      p.in_zp = static_cast<int32_t>(n.attr_or<int64_t>("in_zero_point", 0));
      p.out_zp = static_cast<int32_t>(n.attr_or<int64_t>("zero_point", 0));
      p.q_min = static_cast<int32_t>(n.attr<int64_t>("q_min"));
      p.q_max = static_cast<int32_t>(n.attr<int64_t>("q_max"));
    }
    run = j;
  }
}

// trap check (OverflowError at the lowest flat index, value recomputed
// exactly) and publication of the integer conv's (or fused requantize's) value
void Runner::finish_int(int i, const std::vector<int>& chain, const DevTensor& y, const kern::ConvShape& cs,
                        const DevTensor& d, const DevTensor& w, const DevTensor* b,
                        const std::vector<int64_t>& zps) {
  if (trap) {
    const int64_t flat = trapped();
    if (flat >= 0) {
      const Node& n = *plan.steps()[static_cast<size_t>(i)].node;
      const int64_t v = kern::conv2d_int_value_at(d.i(), w.i(), b ? b->i() : nullptr, cs, zps[0],
                                                  zps[1], flat, S());
      throw OverflowError(n.id, flat, v);
    }
  }
  for (int j : chain) done[static_cast<size_t>(j)] = 1;
  vals[static_cast<size_t>(chain.empty() ? i : chain.back())] = y;
}

static kern::IntEpi int_epi(const DevTensor& y, const DevTensor* b, const void* wsum,
                            unsigned long long* trap, DType acc, const kern::ConvShape& cs,
                            const std::vector<int64_t>& zps) {
  kern::IntEpi ie{};
  ie.y = y.i();
  ie.bias = b ? b->i() : nullptr;
  ie.zp0 = zps.at(0);
  ie.wsum = ie.zp0 != 0 ? static_cast<const int32_t*>(wsum) : nullptr;
  ie.trap = trap;
  ie.acc_min = acc.min_value();
  ie.acc_max = acc.max_value();
  ie.OHW = cs.OH * cs.OW;
  return ie;
}

// CUDA-core backend (conv_simt.cu): int16 codes, or the int16 accumulator
bool Runner::exec_conv_int_simt(int i, const kern::ConvShape& cs, const DevTensor& d,
                                const DevTensor& w, const DevTensor* b, DType acc,
                                const std::vector<int64_t>& zps) {
  static const bool off = [] {
    const char* e = std::getenv("QUANTC_INT_SIMT");
    return e && std::string(e) == "0";
  }();
  if (off || !d.dtype.is_integer() || !w.dtype.is_integer()) return false;
  if (d.dtype.width() > 16 || acc.width() > 32) return false;
  const bool i16 = d.dtype.width() > 8;
  const bool u8 = !i16 && !d.dtype.is_signed();
  const int per = i16 ? 2 : 4;
  const int Cw = (cs.C + per - 1) / per;
  const int taps = cs.KH * cs.KW;
  const int64_t K = static_cast<int64_t>(taps) * Cw;
  if (!i16 && K * 4 * 255 * 128 >= (int64_t{1} << 31)) return false;  // dp4a int32 sum
  auto key = std::make_pair(i, 1);
  auto wit = plan.int_weights.find(key);
  if (wit == plan.int_weights.end()) {
    Plan::IntWeights iw;
    iw.codes = device_alloc(static_cast<size_t>(K) * cs.O * 4);
    iw.wsum = device_alloc(static_cast<size_t>(cs.O) * 4 + 16);
    int* bad = reinterpret_cast<int*>(static_cast<int8_t*>(iw.wsum.get()) + static_cast<size_t>(cs.O) * 4);
    cuda_ok(cudaMemsetAsync(iw.wsum.get(), 0, static_cast<size_t>(cs.O) * 4 + 16, S()), "wsum");
    kern::pack_weight_words(w.i(), static_cast<uint32_t*>(iw.codes.get()),
                            static_cast<int32_t*>(iw.wsum.get()), bad, cs.O, cs.C, taps, Cw, i16,
                            zps.at(1), S());
    int hbad = 0;
    cuda_ok(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, S()), "pack flag");
    device::synchronize();
    iw.ok = hbad == 0;
    wit = plan.int_weights.emplace(key, iw).first;
  }
  if (!wit->second.ok) return false;
  const std::shared_ptr<void>& wwords = wit->second.codes;
  const std::shared_ptr<void>& wsum = wit->second.wsum;
  const int HP = cs.H + 2 * cs.ph, WP = cs.W + 2 * cs.pw;
  auto xwords = device_alloc(static_cast<size_t>(cs.N) * HP * WP * Cw * 4 + 16);
  kern::pack_words(d.i(), static_cast<uint32_t*>(xwords.get()), cs.N, cs.C, cs.H, cs.W, cs.ph,
                   cs.pw, Cw, i16, static_cast<int32_t>(zps.at(0)), S());
  const std::vector<int> chain = fused_chain(i);
  DevTensor y = out_like(chain.empty() ? i : chain.back(), chain_dtype(chain, acc));
  kern::SimtConvSpec sp{};
  sp.x = static_cast<const uint32_t*>(xwords.get());
  sp.w = static_cast<const uint32_t*>(wwords.get());
  sp.N = cs.N;
  sp.HP = HP;
  sp.WP = WP;
  sp.Cw = Cw;
  sp.O = cs.O;
  sp.KH = cs.KH;
  sp.KW = cs.KW;
  sp.sh = cs.sh;
  sp.sw = cs.sw;
  sp.OH = cs.OH;
  sp.OW = cs.OW;
  sp.i16 = i16;
  sp.u8 = u8;
  sp.ie = int_epi(y, b, wsum.get(), trap_ptr(), acc, cs, zps);
  fill_posts(sp.ie, i, chain);
  kern::conv_int_simt(sp, S());
  device::counters().simt_int_convs++;
  finish_int(i, chain, y, cs, d, w, b, zps);
  return true;
}

void Runner::exec_sq(int i) {
  const Node& n = *plan.steps()[static_cast<size_t>(i)].node;
  const DevTensor& x = in(i, 0);
  if (!x.dtype.is_float()) throw std::invalid_argument("simulated_quantize needs a float32 tensor");
  QParams p = qparams_of(n, spec.binding);
  kern::SqParams k = resolve_sq(p);
  if (p.passthrough && !p.acc_dtype.has_value()) {  // identity (simulate.cpp:83)
    DevTensor a = x;
    a.shape = plan.shape(i);
    vals[static_cast<size_t>(i)] = a;
    return;
  }
  DevTensor y = out_like(i, f32);
  kern::sim_quant(x.f(), y.f(), x.numel(spec.batch), k, S());
  vals[static_cast<size_t>(i)] = y;
}

void Runner::exec_sq_codes(int i) {
  const DevTensor& x = in(i, 0);
  if (!x.dtype.is_float()) throw std::invalid_argument("simulated_quantize needs a float32 tensor");
  const kern::SqParams& k = sqp[static_cast<size_t>(i)];
  const auto& shape = plan.shape(i);
  if (plan.batched(i)) {
    // data operand: NCHW (or [rows, K]) -> NHWC codes, channels padded to 16
    const int n0 = static_cast<int>(shape[0] * spec.batch);
    const int C = static_cast<int>(shape[1]);
    const int H = shape.size() == 4 ? static_cast<int>(shape[2]) : 1;
    const int W = shape.size() == 4 ? static_cast<int>(shape[3]) : 1;
    const int Cpad = (C + 15) / 16 * 16;
    auto buf = device_alloc(static_cast<size_t>(n0) * H * W * Cpad);
    kern::sim_quant_codes_nhwc(x.f(), nullptr, static_cast<int8_t*>(buf.get()), n0, C, H, W,
                               Cpad, k, S());
    codes[static_cast<size_t>(i)] = buf;
    code_cpad[static_cast<size_t>(i)] = Cpad;
  }
  // weights are converted by the consumer (needs the data Cpad); keep the
  // float input reachable via vals
  DevTensor alias = x;
  vals[static_cast<size_t>(i)] = alias;
}

void Runner::exec_conv_fast(int i, bool dense) {
  const auto& st = plan.steps()[static_cast<size_t>(i)];
  const int d = st.in[0], w = st.in[1];
  const DevTensor& wt = vals[static_cast<size_t>(w)];  // float weights (pre-sq)
  const auto& dshape = plan.shape(d);
  const auto& wshape = plan.shape(w);
  const auto& oshape = plan.shape(i);
  const int Nimg = static_cast<int>(dshape[0] * spec.batch);
  const int C = static_cast<int>(dshape[1]);
  const int H = dense ? 1 : static_cast<int>(dshape[2]);
  const int W = dense ? 1 : static_cast<int>(dshape[3]);
  const int O = static_cast<int>(wshape[0]);
  const int KH = dense ? 1 : static_cast<int>(wshape[2]);
  const int KW = dense ? 1 : static_cast<int>(wshape[3]);
  const int OH = dense ? 1 : static_cast<int>(oshape[2]);
  const int OW = dense ? 1 : static_cast<int>(oshape[3]);
  Attr2 strd = dense ? Attr2{1, 1} : pair_attr(*st.node, "strides", {1, 1});
  Attr2 pad = dense ? Attr2{0, 0} : pair_attr(*st.node, "padding", {0, 0});
  const int Cpad = code_cpad[static_cast<size_t>(d)];
  const int Kraw = KH * KW * Cpad;
  const int Kpad = (Kraw + 127) / 128 * 128;
  const int64_t M = static_cast<int64_t>(Nimg) * OH * OW;

  // weight codes [O][Kpad] in (kh, kw, c) order
  auto wcodes = device_alloc(static_cast<size_t>(O) * Kpad);
  kern::weights_to_codes(wt.f(), static_cast<int8_t*>(wcodes.get()), O, C, KH, KW, Cpad, Kpad,
                         sqp[static_cast<size_t>(w)], S());
  const int8_t* A = static_cast<const int8_t*>(codes[static_cast<size_t>(d)].get());
  std::shared_ptr<void> cols;
  const bool direct = KH == 1 && KW == 1 && strd.a == 1 && strd.b == 1 && pad.a == 0 &&
                      pad.b == 0 && Cpad == Kpad;
  if (!direct) {
    cols = device_alloc(static_cast<size_t>(M) * Kpad);
    kern::im2col_s8(A, static_cast<int8_t*>(cols.get()), Nimg, H, W, Cpad, KH, KW, OH, OW,
                    strd.a, strd.b, pad.a, pad.b, Kpad, S());
    A = static_cast<const int8_t*>(cols.get());
  }
  DevTensor y = out_like(i, f32);
  kern::GemmEpilogue ep{};
  ep.y = y.f();
  ep.bias = (st.in.size() > 2 && st.in[2] >= 0) ? vals[static_cast<size_t>(st.in[2])].f() : nullptr;
  ep.scale = sqp[static_cast<size_t>(d)].s * sqp[static_cast<size_t>(w)].s;
  ep.OHW = OH * OW;
  const bool prof = device::profile_enabled();
  if (prof) device::profile_gemm_begin();
  kern::gemm_s8_tcgen05(A, static_cast<const int8_t*>(wcodes.get()), static_cast<int>(M), O, Kpad,
                        ep, S());
  if (prof) device::profile_gemm_end(2.0 * static_cast<double>(M) * O * C * KH * KW);
  device::counters().tcgen05_gemms++;
  vals[static_cast<size_t>(i)] = y;
}

void Runner::exec_conv(int i, bool dense) {
  const auto& st = plan.steps()[static_cast<size_t>(i)];
  const Node& n = *st.node;
  const DevTensor& d = in(i, 0);
  const DevTensor& w = in(i, 1);
  const DevTensor* b = (st.in.size() > 2 && st.in[2] >= 0) ? &in(i, 2) : nullptr;
  if (w.batched || (b && b->batched)) {
    throw EvalError("B200 engine: per-sample (non-constant) conv2d/dense weights are unsupported "
                    "at node " + std::to_string(n.id));
  }
  const auto& ds = plan.shape(st.in[0]);
  const auto& ws = plan.shape(st.in[1]);
  const auto& os = plan.shape(i);
  kern::ConvShape cs{};
  cs.N = static_cast<int>(ds[0] * N(st.in[0]));
  if (dense) {
    cs.C = static_cast<int>(ds[1]);
    cs.H = cs.W = cs.KH = cs.KW = cs.OH = cs.OW = cs.sh = cs.sw = 1;
    cs.ph = cs.pw = 0;
    cs.O = static_cast<int>(ws[0]);
  } else {
    Attr2 strd = pair_attr(n, "strides", {1, 1}), pad = pair_attr(n, "padding", {0, 0});
    cs.C = static_cast<int>(ds[1]);
    cs.H = static_cast<int>(ds[2]);
    cs.W = static_cast<int>(ds[3]);
    cs.O = static_cast<int>(ws[0]);
    cs.KH = static_cast<int>(ws[2]);
    cs.KW = static_cast<int>(ws[3]);
    cs.OH = static_cast<int>(os[2]);
    cs.OW = static_cast<int>(os[3]);
    cs.sh = strd.a;
    cs.sw = strd.b;
    cs.ph = pad.a;
    cs.pw = pad.b;
    cs.G = static_cast<int>(n.attr_or<int64_t>("groups", 1));
  }
  if (d.dtype.is_float()) {
    if (!w.dtype.is_float() || (b && !b->dtype.is_float())) {
      throw EvalError(std::string(dense ? "dense" : "conv2d") +
                      " mixed float/integer operands at node " + std::to_string(n.id));
    }
    DevTensor y = out_like(i, f32);
    kern::conv2d_f64acc(d.f(), w.f(), b ? b->f() : nullptr, y.f(), cs, S());
    device::counters().f64_convs++;
    vals[static_cast<size_t>(i)] = y;
    return;
  }
  DType acc = acc_dtype_of(n);
  auto zps = n.attr_or<std::vector<int64_t>>("in_zero_points", {0, 0});
  // grouped integer convs run on the exact int64 kernel
  if (kern::conv_groups(cs) == 1 && exec_conv_int_tc(i, dense, cs, d, w, b, acc, zps)) return;
  if (kern::conv_groups(cs) == 1 && exec_conv_int_simt(i, cs, d, w, b, acc, zps)) return;
  DevTensor y = out_like(i, acc);
  unsigned long long* trap = trap_ptr();
  kern::conv2d_int(d.i(), w.i(), b ? b->i() : nullptr, y.i(), cs, zps[0], zps[1],
                   acc.min_value(), acc.max_value(), trap, S());
  if (trap) {
    int64_t flat = trapped();
    if (flat >= 0) {
      int64_t v = kern::conv2d_int_value_at(d.i(), w.i(), b ? b->i() : nullptr, cs, zps[0],
                                            zps[1], flat, S());
      throw OverflowError(n.id, flat, v);
    }
  }
  vals[static_cast<size_t>(i)] = y;
}

void Runner::exec(int i) {
  if (done[static_cast<size_t>(i)]) return;  // produced by a fused producer
  const auto& st = plan.steps()[static_cast<size_t>(i)];
  const Node& n = *st.node;
  switch (n.op) {
    case OpKind::kInput: {
      const auto& ins = plan.graph().inputs();
      auto it = std::find(ins.begin(), ins.end(), n.id);
      if (it == ins.end()) throw EvalError("missing input tensor: " + n.attr_or<std::string>("name", ""));
      const size_t k = static_cast<size_t>(it - ins.begin());
      if (k >= spec.inputs.size() || !spec.inputs[k]) {
        throw EvalError("missing input tensor: " + n.attr_or<std::string>("name", ""));
      }
      DevTensor t;
      t.dtype = f32;
      t.shape = plan.shape(i);
      t.batched = true;
      t.buf = std::shared_ptr<void>(const_cast<float*>(spec.inputs[k]), [](void*) {});
      vals[static_cast<size_t>(i)] = t;
      return;
    }
    case OpKind::kConstant:
      vals[static_cast<size_t>(i)] = plan.constant(i);
      return;
    case OpKind::kConv2d:
    case OpKind::kDense:
      if (fast_conv[static_cast<size_t>(i)]) {
        exec_conv_fast(i, n.op == OpKind::kDense);
      } else {
        exec_conv(i, n.op == OpKind::kDense);
      }
      return;
    case OpKind::kAdd: {
      const DevTensor& a = in(i, 0);
      const DevTensor& b = in(i, 1);
      if (a.per_numel() != b.per_numel()) {
        throw EvalError("add operand shapes differ at node " + std::to_string(n.id));
      }
      if (a.dtype.is_float() != b.dtype.is_float()) {
        throw EvalError("add mixes float and integer operands at node " + std::to_string(n.id));
      }
      const int64_t total = static_cast<int64_t>(plan.batched(i) ? spec.batch : 1) *
                            shape_numel(plan.shape(i));
      if (a.dtype.is_float()) {
        DevTensor y = out_like(i, f32);
        kern::add_f32(a.f(), a.numel(spec.batch), b.f(), b.numel(spec.batch), y.f(), total, S());
        vals[static_cast<size_t>(i)] = y;
      } else {
        DType acc = acc_dtype_of(n);
        DevTensor y = out_like(i, acc);
        unsigned long long* trap = trap_ptr();
        kern::add_int(a.i(), a.numel(spec.batch), b.i(), b.numel(spec.batch), y.i(), total,
                      acc.min_value(), acc.max_value(), trap, S());
        if (trap) {
          int64_t flat = trapped();
          if (flat >= 0) {
            int32_t av = 0, bv = 0;
            cuda_ok(cudaMemcpy(&av, a.i() + flat % a.numel(spec.batch), 4, cudaMemcpyDeviceToHost), "trap");
            cuda_ok(cudaMemcpy(&bv, b.i() + flat % b.numel(spec.batch), 4, cudaMemcpyDeviceToHost), "trap");
            throw OverflowError(n.id, flat, static_cast<int64_t>(av) + bv);
          }
        }
        vals[static_cast<size_t>(i)] = y;
      }
      return;
    }
    case OpKind::kRelu: {
      const DevTensor& x = in(i, 0);
      DevTensor y = out_like(i, x.dtype);
      if (x.dtype.is_float()) {
        kern::relu_f32(x.f(), y.f(), x.numel(spec.batch), S());
      } else {
        kern::relu_int(x.i(), y.i(), x.numel(spec.batch),
                       static_cast<int32_t>(n.attr_or<int64_t>("zero_point", 0)), S());
      }
      vals[static_cast<size_t>(i)] = y;
      return;
    }
    case OpKind::kClip: {
      const DevTensor& x = in(i, 0);
      DevTensor y = out_like(i, x.dtype);
      if (x.dtype.is_float()) {
        kern::clip_f32(x.f(), y.f(), x.numel(spec.batch), static_cast<float>(n.attr<double>("a_min")),
                       static_cast<float>(n.attr<double>("a_max")), S());
      } else {
        kern::clip_int(x.i(), y.i(), x.numel(spec.batch),
                       static_cast<int32_t>(n.attr<int64_t>("q_min")),
                       static_cast<int32_t>(n.attr<int64_t>("q_max")), S());
      }
      vals[static_cast<size_t>(i)] = y;
      return;
    }
    case OpKind::kMaxPool2d: {
      const DevTensor& x = in(i, 0);
      const auto& xs = plan.shape(st.in[0]);
      const auto& os = plan.shape(i);
      auto k = n.attr<std::vector<int64_t>>("pool_size");
      Attr2 strd = pair_attr(n, "strides", {static_cast<int>(k[0]), static_cast<int>(k[1])});
      Attr2 pad = pair_attr(n, "padding", {0, 0});
      DevTensor y = out_like(i, x.dtype);
      const int Nn = static_cast<int>(xs[0] * N(st.in[0]));
      if (x.dtype.is_float()) {
        kern::maxpool_f32(x.f(), y.f(), Nn, static_cast<int>(xs[1]), static_cast<int>(xs[2]),
                          static_cast<int>(xs[3]), static_cast<int>(os[2]), static_cast<int>(os[3]),
                          static_cast<int>(k[0]), static_cast<int>(k[1]), strd.a, strd.b, pad.a,
                          pad.b, S());
      } else {
        kern::maxpool_int(x.i(), y.i(), Nn, static_cast<int>(xs[1]), static_cast<int>(xs[2]),
                          static_cast<int>(xs[3]), static_cast<int>(os[2]), static_cast<int>(os[3]),
                          static_cast<int>(k[0]), static_cast<int>(k[1]), strd.a, strd.b, pad.a,
                          pad.b, S());
      }
      vals[static_cast<size_t>(i)] = y;
      return;
    }
    case OpKind::kGlobalAvgPool2d: {
      const DevTensor& x = in(i, 0);
      if (!x.dtype.is_float()) {
        throw EvalError("integer global_avg_pool2d is not supported (node " + std::to_string(n.id) + ")");
      }
      const auto& xs = plan.shape(st.in[0]);
      DevTensor y = out_like(i, f32);
      kern::gap_f32(x.f(), y.f(), static_cast<int>(xs[0] * N(st.in[0]) * xs[1]),
                    static_cast<int>(xs[2] * xs[3]), S());
      vals[static_cast<size_t>(i)] = y;
      return;
    }
    case OpKind::kFlatten: {
      DevTensor a = in(i, 0);
      a.shape = plan.shape(i);
      vals[static_cast<size_t>(i)] = a;
      return;
    }
    case OpKind::kAvgPool2d: {
      const DevTensor& x = in(i, 0);
      if (!x.dtype.is_float()) {
        throw EvalError("integer avg_pool2d is not supported (node " + std::to_string(n.id) + ")");
      }
      const auto& xs = plan.shape(st.in[0]);
      const auto& os = plan.shape(i);
      auto k = n.attr<std::vector<int64_t>>("pool_size");
      Attr2 strd = pair_attr(n, "strides", {static_cast<int>(k[0]), static_cast<int>(k[1])});
      Attr2 pad = pair_attr(n, "padding", {0, 0});
      DevTensor y = out_like(i, f32);
      kern::avgpool_f32(x.f(), y.f(), static_cast<int>(xs[0] * N(st.in[0])), static_cast<int>(xs[1]),
                        static_cast<int>(xs[2]), static_cast<int>(xs[3]), static_cast<int>(os[2]),
                        static_cast<int>(os[3]), static_cast<int>(k[0]), static_cast<int>(k[1]),
                        strd.a, strd.b, pad.a, pad.b, S());
      vals[static_cast<size_t>(i)] = y;
      return;
    }
    case OpKind::kConcat: {
      // every operand is [n, c_i, H, W] per sample: copy each into its channel
      // range of the [n, sum c_i, H, W] output (batched operands only; an
      // unbatched operand broadcasts over the batch)
      const DevTensor& x0 = in(i, 0);
      DevTensor y = out_like(i, x0.dtype);
      const auto& os = plan.shape(i);
      const int64_t hw = os[2] * os[3];
      const int64_t outer = os[1] * hw;
      const int rows = static_cast<int>(os[0] * N(i));
      int64_t off = 0;
      for (size_t p = 0; p < st.in.size(); ++p) {
        const DevTensor& x = in(i, static_cast<int>(p));
        if (x.dtype.is_float() != x0.dtype.is_float()) {
          throw EvalError("concat mixes float and integer operands at node " + std::to_string(n.id));
        }
        const int64_t inner = plan.shape(st.in[p])[1] * hw;
        if (plan.batched(st.in[p]) || N(i) == 1) {
          kern::concat_words(x.buf.get(), y.buf.get(), rows, inner, outer, off, S());
        } else {
          for (int r = 0; r < rows; ++r) {
            kern::concat_words(x.buf.get(), static_cast<uint32_t*>(y.buf.get()) + r * outer, 1,
                               inner, outer, off, S());
          }
        }
        off += inner;
      }
      vals[static_cast<size_t>(i)] = y;
      return;
    }
    case OpKind::kSimulatedQuantize:
      if (codes_only[static_cast<size_t>(i)]) {
        exec_sq_codes(i);
      } else {
        exec_sq(i);
      }
      return;
    case OpKind::kQuantize: {
      require_int_regime(n);
      const DevTensor& x = in(i, 0);
      if (!x.dtype.is_float()) throw EvalError("quantize input must be float32");
      DevTensor y = out_like(i, parse_dtype(n.attr<std::string>("out_dtype")));
      kern::quantize_f32_int(x.f(), y.i(), x.numel(spec.batch), n.attr<double>("scale"),
                             n.attr_or<int64_t>("zero_point", 0), n.attr<int64_t>("q_min"),
                             n.attr<int64_t>("q_max"), S());
      vals[static_cast<size_t>(i)] = y;
      return;
    }
    case OpKind::kDequantize: {
      require_int_regime(n);
      const DevTensor& x = in(i, 0);
      if (!x.dtype.is_integer()) throw EvalError("dequantize input must be integer");
      DevTensor y = out_like(i, f32);
      kern::dequantize_int_f32(x.i(), y.f(), x.numel(spec.batch), n.attr<double>("scale"),
                               n.attr_or<int64_t>("zero_point", 0), S());
      vals[static_cast<size_t>(i)] = y;
      return;
    }
    case OpKind::kRequantize: {
      require_int_regime(n);
      const DevTensor& x = in(i, 0);
      if (!x.dtype.is_integer()) throw EvalError("requantize input must be integer");
      DevTensor y = out_like(i, parse_dtype(n.attr<std::string>("out_dtype")));
      kern::requantize_int(x.i(), y.i(), x.numel(spec.batch), n.attr<int64_t>("multiplier"),
                           n.attr<int>("shift"), n.attr_or<int64_t>("in_zero_point", 0),
                           n.attr_or<int64_t>("zero_point", 0), n.attr<int64_t>("q_min"),
                           n.attr<int64_t>("q_max"), S());
      vals[static_cast<size_t>(i)] = y;
      return;
    }
  }
  throw EvalError("bad op kind");
}

}  // namespace

std::vector<DevTensor> run(const Plan& plan, const RunSpec& spec) {
  // QUANTC_STEP_PROF=<ms>: report steps whose host-side work exceeds <ms>
  // (default 5) and a per-op-kind host-time summary at the end
  static const double sprof = [] {
    const char* e = std::getenv("QUANTC_STEP_PROF");
    if (!e) return -1.0;
    const double v = std::atof(e);
    return v > 0.0 ? v : 5.0;
  }();
  Runner r(plan, spec);
  r.plan_fast();
  const int n = static_cast<int>(plan.steps().size());
  std::map<std::string, std::pair<double, int>> by_op;
  for (int i = 0; i < n; ++i) {
    if (sprof < 0.0) {
      r.exec(i);
      if (spec.on_value) spec.on_value(i, r.vals[static_cast<size_t>(i)]);
      r.release_inputs(i);
      continue;
    }
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    const auto t0 = std::chrono::steady_clock::now();
    r.exec(i);
    const auto t1 = std::chrono::steady_clock::now();
    if (spec.on_value) spec.on_value(i, r.vals[static_cast<size_t>(i)]);
    const auto t2 = std::chrono::steady_clock::now();
    r.release_inputs(i);
    const auto t3 = std::chrono::steady_clock::now();
    const std::string op = op_name(plan.steps()[static_cast<size_t>(i)].node->op);
    by_op[op].first += ms(t0, t3);
    by_op[op].second += 1;
    if (ms(t0, t3) > sprof) {
      std::fprintf(stderr, "  step %d op %s: exec %.2f hook %.2f release %.2f ms\n", i, op.c_str(),
                   ms(t0, t1), ms(t1, t2), ms(t2, t3));
    }
  }
  if (sprof >= 0.0) {
    for (const auto& [op, v] : by_op) {
      std::fprintf(stderr, "  host %-20s %8.2f ms over %d steps\n", op.c_str(), v.first, v.second);
    }
  }
  std::vector<DevTensor> out;
  for (int k : spec.keep) out.push_back(r.vals[static_cast<size_t>(k)]);
  return out;
}

}  // namespace quantc::engine
