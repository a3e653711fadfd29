// fastplan.hpp — engine v2: the fused int8 dataflow for simulated-quantize
// evaluation (internal to the B200 build).
//
// Compiles a simulated graph into stages, each = one producing operator
// (graph input, tcgen05 conv/dense GEMM, max-pool on codes, GAP) + the
// per-element program of everything elementwise hanging off it (consumer
// simulated_quantize, relu, clip, residual add, flatten).  Values cross stage
// boundaries as NHWC int8 codes (sq outputs) or fp32 rows (boundary values,
// graph outputs).  See kernels/fused.h for the program ops and the exactness
// argument (power-of-two scales).
#pragma once

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "engine.hpp"

namespace quantc::fast {

class FastPlan {
 public:
  explicit FastPlan(const engine::Plan& plan);
  ~FastPlan();
  FastPlan(const FastPlan&) = delete;

  bool ok() const { return ok_; }
  const std::string& why_not() const { return why_; }

  // Binding eligibility: every simulated_quantize resolvable to the fp32
  // program form, every materialised code int8; `exact` additionally
  // requires power-of-two scales (bit-identical to the reference).
  bool eligible(const SimBinding* binding, bool exact, std::string* why = nullptr) const;

  // Runs one batch; writes per-sample argmax of graph output 0 to preds.
  // d_scores (optional): the output rows themselves, [batch x out_per_sample()]
  void predict(int batch, const std::vector<const float*>& inputs, const SimBinding* binding,
               int64_t* d_preds, float* d_scores = nullptr);
  // several bindings (<= 4) over the same samples; compatible GEMM stages
  // run as one grouped tcgen05 launch (fastplan.cpp)
  void predict_group(int batch, const std::vector<const float*>& inputs,
                     const std::vector<const SimBinding*>& bindings,
                     const std::vector<int64_t*>& preds,
                     const std::vector<float*>* scores = nullptr);
  int64_t out_per_sample() const { return out_per_sample_; }
  // stream this instance enqueues on (nullptr: the engine stream); every
  // buffer, table upload and launch of the instance is ordered on it
  void set_stream(void* s) { stream_ = s; }

  struct Val;
  struct Stage;

 private:
  const engine::Plan& plan_;
  void* stream_ = nullptr;
  bool ok_ = false;
  std::string why_;
  std::vector<std::unique_ptr<Val>> vals_;
  std::vector<std::unique_ptr<Stage>> stages_;
  std::map<int, int> sq_index_;  // sq step -> FSq table slot
  std::vector<int> sq_steps_;
  std::vector<float> clip_lo_, clip_hi_;
  int out_val_ = -1;
  int64_t out_per_sample_ = 0;
  std::shared_ptr<void> d_code_;  // all programs, uploaded once
  // per-batch arenas (one per concurrently prepared binding): a buffer per
  // materialised value and the stage-table block
  struct Arena {
    int batch = -1;
    std::vector<std::shared_ptr<void>> bufs;
    std::shared_ptr<void> tables;
  };
  Arena arenas_[kern::kMaxGroups];
  // weight code cache: (stage, FSq bytes) -> codes
  std::map<std::pair<int, std::string>, std::shared_ptr<void>> wcache_;
  size_t wcache_bytes_ = 0;
  void trim_weight_cache();
  // integer-epilogue folds (fold_integer): per (stage, sq0 grid) the device
  // table of folded biases, or null when some channel's breakpoints are
  // irregular (the float shape then runs)
  std::map<std::pair<int, std::string>, std::pair<std::shared_ptr<void>, int64_t>> ctab_cache_;
  bool fold_integer(size_t si, int shape, double sxw, double acc_bound, kern::EpiConsts& e,
                    std::vector<std::shared_ptr<void>>& keep);

  struct Run;
  void compile();
  void fail(const std::string& why);
  void ensure_arena(int batch, int group);
  void prepare(Run& r);
  void* buf(const Run& r, int vid) const;
  // a value's device pointer in arena `group`, through concat column slices
  void* arena_ptr(int group, int vid) const;
  void gemm_spec(Run& r, size_t si, kern::TcConvSpec& sp);
  void launch_gemm(size_t si, const kern::TcConvSpec& sp);
  void run_stage(Run& r, size_t si);
  void finish(Run& r);
};

}  // namespace quantc::fast
