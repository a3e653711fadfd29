// engine.hpp — the GPU graph executor behind every quantc evaluation entry
// point (eval_fp32 / eval_int / predict_top1 / collect_stats /
// CandidateEvaluator).  Internal to the B200 build.
//
// A Plan is compiled once per graph (traversal order, port wiring, constants
// resident in HBM).  run() executes the plan over a batch of samples on the
// engine stream: samples are stacked along the leading dimension (every
// per-sample computation of the reference is independent, so batching changes
// no result), constants and values derived only from constants are computed
// once per run (weight simulated-quantize happens once per candidate, not once
// per sample as in the reference, which is bit-identical).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <memory>
#include <unordered_map>
#include <vector>

#include "quantc/graph.hpp"
#include "quantc/interpreter.hpp"
#include "../kernels/kernels.h"

namespace quantc::fast {
class FastPlan;
}

namespace quantc::engine {

struct DevTensor {
  std::shared_ptr<void> buf;  // device memory (shared by aliases, e.g. flatten)
  DType dtype = f32;          // float32 or integer (int32 storage)
  std::vector<int64_t> shape; // batched: per-sample shape; else full shape
  bool batched = false;
  // integer values of <= 8 bits may also carry their NHWC code bytes
  // [pixels][codes_ld] (written by the producing conv's epilogue): an integer
  // conv consuming them without a zero-point border skips its pack pass
  std::shared_ptr<void> codes;
  int codes_ld = 0;

  int64_t per_numel() const { return shape_numel(shape); }
  int64_t numel(int batch) const { return batched ? per_numel() * batch : per_numel(); }
  float* f() const { return static_cast<float*>(buf.get()); }
  int32_t* i() const { return static_cast<int32_t*>(buf.get()); }
};

// stream-ordered device allocation
std::shared_ptr<void> device_alloc(size_t bytes);
// stream-ordered allocation (and free) on `stream` (a cudaStream_t)
std::shared_ptr<void> device_alloc_on(void* stream, size_t bytes);

kern::SqParams resolve_sq(const QParams& p);  // validates like simulate.cpp:47-60
QParams qparams_of(const Node& n, const SimBinding* binding);

class Plan {
 public:
  explicit Plan(const Graph& g);
  Plan(const Plan&) = delete;

  struct Step {
    const Node* node = nullptr;
    std::vector<int> in;  // producer step index per port (-1 unfed)
    int uses = 0;         // consumers + graph-output references
  };

  const Graph& graph() const { return g_; }
  const std::vector<Step>& steps() const { return steps_; }
  int step_of(NodeId id) const { return index_.at(id); }
  const DevTensor& constant(int step) const { return constants_.at(step); }
  // per-sample output shape of every step (batched values) / full shape
  const std::vector<int64_t>& shape(int step) const { return shapes_[static_cast<size_t>(step)]; }
  bool batched(int step) const { return batched_[static_cast<size_t>(step)] != 0; }
  int64_t per_sample_bytes_peak() const { return peak_bytes_; }
  int batch_for(int64_t n_samples) const;

 private:
  const Graph& g_;
  std::vector<Step> steps_;
  std::unordered_map<NodeId, int> index_;
  std::unordered_map<int, DevTensor> constants_;
  std::vector<std::vector<int64_t>> shapes_;
  std::vector<char> batched_;
  int64_t peak_bytes_ = 0;

 public:
  // lazily compiled fused int8 dataflow (engine v2) for this graph
  mutable std::shared_ptr<fast::FastPlan> fused;
  mutable bool fused_tried = false;
  // extra instances of the fused plan, one per auxiliary stream: a batch is
  // split across the streams so one forward's per-layer fill/drain latency
  // overlaps another's work (dataset.cpp fused_predict)
  mutable std::vector<std::shared_ptr<fast::FastPlan>> fused_aux;
  // realized-graph integer convs: packed weights (w - zp1) and row sums per
  // (step, backend), built once per plan; ok = false when w - zp1 leaves
  // the backend's range (the layer then runs on the int64 kernel)
  struct IntWeights {
    std::shared_ptr<void> codes, wsum;
    bool ok = false;
  };
  mutable std::map<std::pair<int, int>, IntWeights> int_weights;
};

// Process-wide cache of compiled plans (device-resident constants, the fused
// plan with its activation arena and weight codes), keyed by Graph::uid() so a
// serving loop calling predict_top1 on the same graph uploads its weights
// once.  A lease holds the entry's lock: concurrent callers on one graph
// serialise, different graphs run independently.  Capacity: QUANTC_PLAN_CACHE
// entries (default 2; 0 = no caching, a private plan per call).
class PlanLease {
 public:
  const Plan& plan() const { return *plan_; }
  struct Entry;

 private:
  friend PlanLease lease_plan(const Graph& g);
  std::shared_ptr<Entry> entry_;
  std::unique_ptr<Plan> own_;
  std::shared_ptr<void> lock_;
  const Plan* plan_ = nullptr;
};
PlanLease lease_plan(const Graph& g);

struct RunSpec {
  int batch = 1;
  std::vector<const float*> inputs;  // device, one per graph input, [batch x per-sample]
  const SimBinding* binding = nullptr;
  bool integer_regime = false;
  OverflowMode mode = OverflowMode::kSaturate;
  bool allow_fast = false;  // tcgen05 int8 path permitted (sim-quant evaluation)
  // called right after a step's value is produced
  std::function<void(int step, const DevTensor&)> on_value;
  std::vector<int> keep;  // steps whose values are returned
};

// Runs a plan; returns kept values indexed like spec.keep.
std::vector<DevTensor> run(const Plan& plan, const RunSpec& spec);

// Host <-> device helpers
DevTensor upload(const Tensor& t);
// eval_fp32 / eval_int of a single-input graph on a caller-owned host buffer
// (interpreter.cpp; the C-ABI's qc_eval_fp32 / qc_eval_int)
std::vector<Tensor> eval_fp32_host(const Graph& g, const float* x, const std::vector<int64_t>& shape,
                                   const SimBinding* binding);
std::vector<Tensor> eval_int_host(const Graph& g, const float* x, const std::vector<int64_t>& shape,
                                  OverflowMode mode);
Tensor download(const DevTensor& d, int batch);

}  // namespace quantc::engine
