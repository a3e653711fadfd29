// interpreter.cpp — the reference executor API on the GPU engine
// (reference interpreter.cpp:487-603).
#include "quantc/interpreter.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "dataset.hpp"
#include "engine.hpp"
#include "quantc/device.hpp"

namespace quantc {

OverflowError::OverflowError(NodeId node_, int64_t flat_index_, int64_t value_)
    : EvalError("accumulator overflow at node " + std::to_string(node_) + ", element " +
                std::to_string(flat_index_) + " (value " + std::to_string(value_) + ")"),
      node(node_),
      flat_index(flat_index_),
      value(value_) {}

namespace {

cudaStream_t S() { return static_cast<cudaStream_t>(device::stream()); }

// one graph input as a host view: the reference FeedMap's tensors, or the
// caller's buffer straight from the C-ABI (no intermediate Tensor copies)
struct HostInput {
  const float* data;
  std::vector<int64_t> shape;
};

// host inputs -> one-sample device inputs, with the reference's checks
// (interpreter.cpp:115-125)
std::vector<std::shared_ptr<void>> upload_inputs(const Graph& g, const std::vector<HostInput>& in) {
  std::vector<std::shared_ptr<void>> bufs;
  for (size_t k = 0; k < g.inputs().size(); ++k) {
    const Node& n = g.node(g.inputs()[k]);
    const std::string name = n.attr_or<std::string>("name", "");
    auto shape = n.attr<std::vector<int64_t>>("shape");
    if (in[k].shape != shape) {
      throw EvalError("input " + name + " has shape " + shape_to_string(in[k].shape) +
                      ", expected " + shape_to_string(shape));
    }
    const size_t bytes = static_cast<size_t>(shape_numel(shape)) * 4;
    auto buf = engine::device_alloc(bytes);
    static const bool no_staging = std::getenv("QUANTC_NO_STAGED_INPUT") != nullptr;
    if (bytes >= (size_t{4} << 20) && !no_staging && !device::host_pinned(in[k].data, bytes)) {
      gpu::staged_h2d(buf.get(), in[k].data, bytes);  // pageable caller buffer, tens of MB
    } else if (bytes) {
      if (cudaMemcpyAsync(buf.get(), in[k].data, bytes, cudaMemcpyHostToDevice, S()) != cudaSuccess) {
        throw DeviceError("input upload failed");
      }
    }
    bufs.push_back(buf);
  }
  return bufs;
}

std::vector<HostInput> feed_views(const Graph& g, const FeedMap& feed) {
  std::vector<HostInput> v;
  for (NodeId id : g.inputs()) {
    const Node& n = g.node(id);
    const std::string name = n.attr_or<std::string>("name", "");
    auto it = feed.find(name);
    if (it == feed.end()) throw EvalError("missing input tensor: " + name);
    if (!it->second.dtype().is_float()) {
      throw EvalError("B200 engine: graph inputs must be float32 (input " + name + ")");
    }
    v.push_back(HostInput{it->second.floats().data(), it->second.shape()});
  }
  return v;
}

std::vector<std::shared_ptr<void>> feed_inputs(const Graph& g, const FeedMap& feed) {
  return upload_inputs(g, feed_views(g, feed));
}

std::vector<Tensor> run_single(const Graph& g, const std::vector<HostInput>& in,
                               const SimBinding* binding, bool integer_regime, OverflowMode mode) {
  // weights stay resident across calls on the same graph (plan cache)
  const engine::PlanLease lease = engine::lease_plan(g);
  const engine::Plan& plan = lease.plan();
  // grow the allocator pool once for the run's activations (many growth
  // steps during the run stall the host for up to seconds)
  device::pool_reserve(static_cast<size_t>(plan.per_sample_bytes_peak()) * 2);
  static const bool hprof = std::getenv("QUANTC_HOST_PROF") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  const auto t0 = now();
  auto bufs = upload_inputs(g, in);
  const auto t1 = now();
  engine::RunSpec spec;
  spec.batch = 1;
  for (auto& b : bufs) spec.inputs.push_back(static_cast<const float*>(b.get()));
  spec.binding = binding;
  spec.integer_regime = integer_regime;
  spec.mode = mode;
  for (const PortRef& o : g.outputs()) spec.keep.push_back(plan.step_of(o.node));
  auto vals = engine::run(plan, spec);
  const auto t2 = now();
  std::vector<Tensor> outs;
  for (size_t k = 0; k < vals.size(); ++k) {
    if (!vals[k].buf) throw EvalError("graph output was never computed");
    outs.push_back(engine::download(vals[k], 1));
  }
  if (hprof) {
    std::fprintf(stderr, "run_single ms: upload %.2f run(host) %.2f sync+download %.2f\n", ms(t0, t1),
                 ms(t1, t2), ms(t2, now()));
  }
  return outs;
}

}  // namespace

std::vector<Tensor> eval_fp32(const Graph& g, const FeedMap& feed, const SimBinding* binding) {
  return run_single(g, feed_views(g, feed), binding, false, OverflowMode::kSaturate);
}

std::map<NodeId, Tensor> eval_fp32_values(const Graph& g, const FeedMap& feed,
                                          const SimBinding* binding) {
  engine::Plan plan(g);
  auto bufs = feed_inputs(g, feed);
  engine::RunSpec spec;
  spec.batch = 1;
  for (auto& b : bufs) spec.inputs.push_back(static_cast<const float*>(b.get()));
  spec.binding = binding;
  for (size_t i = 0; i < plan.steps().size(); ++i) spec.keep.push_back(static_cast<int>(i));
  auto vals = engine::run(plan, spec);
  std::map<NodeId, Tensor> out;
  for (size_t i = 0; i < vals.size(); ++i) {
    out[plan.steps()[i].node->id] = engine::download(vals[i], 1);
  }
  return out;
}

std::vector<Tensor> eval_int(const Graph& g, const FeedMap& feed, OverflowMode mode) {
  if (g.contains_op(OpKind::kSimulatedQuantize)) {
    throw EvalError("eval_int expects a realized graph without simulated_quantize nodes");
  }
  return run_single(g, feed_views(g, feed), nullptr, true, mode);
}

namespace engine {

// C-ABI entry points: the single graph input straight from the caller's
// buffer (the FeedMap route copies the input into a Tensor, then into the
// feed: ~20 ms of host copies and page faults for a 38.5 MB batch)
std::vector<Tensor> eval_fp32_host(const Graph& g, const float* x, const std::vector<int64_t>& shape,
                                   const SimBinding* binding) {
  if (g.inputs().size() != 1) throw EvalError("C-ABI eval supports single-input graphs");
  return run_single(g, {HostInput{x, shape}}, binding, false, OverflowMode::kSaturate);
}

std::vector<Tensor> eval_int_host(const Graph& g, const float* x, const std::vector<int64_t>& shape,
                                  OverflowMode mode) {
  if (g.inputs().size() != 1) throw EvalError("C-ABI eval supports single-input graphs");
  if (g.contains_op(OpKind::kSimulatedQuantize)) {
    throw EvalError("eval_int expects a realized graph without simulated_quantize nodes");
  }
  return run_single(g, {HostInput{x, shape}}, nullptr, true, mode);
}

}  // namespace engine

std::vector<Tensor> eval_model(const Graph& g, const FeedMap& feed, OverflowMode mode,
                               const SimBinding* binding) {
  if (g.is_realized()) return eval_int(g, feed, mode);
  return eval_fp32(g, feed, binding);
}

FeedMap feed_for(const Graph& g, const Sample& sample) {
  if (sample.inputs.size() != g.inputs().size()) {
    throw EvalError("sample provides " + std::to_string(sample.inputs.size()) + " tensors for " +
                    std::to_string(g.inputs().size()) + " graph inputs");
  }
  FeedMap feed;
  for (size_t i = 0; i < g.inputs().size(); ++i) {
    feed[g.node(g.inputs()[i]).attr_or<std::string>("name", "")] = sample.inputs[i];
  }
  return feed;
}

int64_t argmax_class(const Tensor& scores) {
  auto s = scores.floats();
  if (s.empty()) throw EvalError("empty score vector");
  int64_t best = 0;
  for (size_t i = 1; i < s.size(); ++i) {
    if (s[i] > s[static_cast<size_t>(best)]) best = static_cast<int64_t>(i);
  }
  return best;
}

std::vector<int64_t> predict_top1(const Graph& g, const Dataset& dataset, int workers,
                                  const SimBinding* binding) {
  (void)workers;  // per-sample parallelism is the GPU batch dimension
  if (dataset.empty()) return {};
  static const bool hprof = std::getenv("QUANTC_HOST_PROF") != nullptr;
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  const engine::PlanLease lease = engine::lease_plan(g);  // weights stay resident across calls
  const engine::Plan& plan = lease.plan();
  const auto t1 = clk::now();
  const bool realized = g.is_realized();
  if (realized && g.contains_op(OpKind::kSimulatedQuantize)) {
    throw EvalError("eval_int expects a realized graph without simulated_quantize nodes");
  }
  std::shared_ptr<void> preds;
  if (realized) {
    gpu::DeviceDataset dd(g, dataset);
    preds = gpu::predict_device(plan, dd, nullptr, true, false);
  } else {
    preds = gpu::predict_streamed(plan, g, dataset, binding);
  }
  const auto t2 = clk::now();
  const auto t3 = t2;
  std::vector<int64_t> h(dataset.size());
  cudaMemcpyAsync(h.data(), preds.get(), h.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, S());
  device::synchronize();
  if (hprof) {
    auto us = [](clk::time_point a, clk::time_point b) {
      return std::chrono::duration<double, std::micro>(b - a).count();
    };
    std::fprintf(stderr, "predict_top1 us: lease %.1f upload+predict(host) %.1f - %.1f sync %.1f total %.1f\n",
                 us(t0, t1), us(t1, t2), us(t2, t3), us(t3, clk::now()), us(t0, clk::now()));
  }
  return h;
}

std::vector<float> predict_scores(const Graph& g, const Dataset& dataset,
                                  const SimBinding* binding, int64_t* per_sample) {
  *per_sample = 0;
  if (dataset.empty()) return {};
  const engine::PlanLease lease = engine::lease_plan(g);
  const engine::Plan& plan = lease.plan();
  gpu::DeviceDataset dd(g, dataset);
  const bool realized = g.is_realized();
  std::shared_ptr<void> scores;
  gpu::predict_device(plan, dd, realized ? nullptr : binding, realized,
                      /*allow_fast=*/binding != nullptr, &scores, per_sample);
  std::vector<float> h(static_cast<size_t>(dataset.size() * *per_sample));
  cudaMemcpyAsync(h.data(), scores.get(), h.size() * 4, cudaMemcpyDeviceToHost, S());
  device::synchronize();
  return h;
}

double top1_agreement(const Graph& g_ref, const Graph& g_test, const Dataset& dataset,
                      int workers) {
  if (dataset.empty()) throw EvalError("empty dataset");
  if (g_ref.inputs().size() != g_test.inputs().size()) {
    throw EvalError("models have different input signatures");
  }
  auto a = predict_top1(g_ref, dataset, workers);
  auto b = predict_top1(g_test, dataset, workers);
  int64_t same = 0;
  for (size_t i = 0; i < a.size(); ++i) same += a[i] == b[i] ? 1 : 0;
  return static_cast<double>(same) / static_cast<double>(a.size());
}

double labeled_accuracy(const Graph& g, const Dataset& dataset, int workers) {
  auto preds = predict_top1(g, dataset, workers);
  int64_t labeled = 0, correct = 0;
  for (size_t i = 0; i < dataset.size(); ++i) {
    if (!dataset[i].label) continue;
    ++labeled;
    correct += preds[i] == *dataset[i].label ? 1 : 0;
  }
  if (labeled == 0) throw EvalError("dataset carries no labels");
  return static_cast<double>(correct) / static_cast<double>(labeled);
}

double mean_abs_output_diff(const Graph& g_a, const Graph& g_b, const Dataset& dataset,
                            int workers) {
  (void)workers;
  if (dataset.empty()) throw EvalError("empty dataset");
  double total = 0.0;
  for (const Sample& s : dataset) {
    Tensor a = eval_model(g_a, feed_for(g_a, s))[0];
    Tensor b = eval_model(g_b, feed_for(g_b, s))[0];
    if (!a.same_shape(b)) throw EvalError("output shape mismatch");
    auto aa = a.floats();
    auto bb = b.floats();
    double acc = 0.0;
    for (size_t k = 0; k < aa.size(); ++k) {
      acc += std::fabs(static_cast<double>(aa[k]) - static_cast<double>(bb[k]));
    }
    total += acc / static_cast<double>(aa.size());
  }
  return total / static_cast<double>(dataset.size());
}

}  // namespace quantc
