// dataset.hpp — calibration/evaluation samples resident in HBM and the
// batched top-1 prediction loop shared by predict_top1, collect_stats and
// CandidateEvaluator (internal to the B200 build).
#pragma once

#include <memory>
#include <vector>

#include "engine.hpp"
#include "quantc/interpreter.hpp"

namespace quantc::gpu {

// host -> device copy through the reusable pinned staging chunks (packed by
// host threads while the previous chunk's DMA runs): a pageable source of
// tens of MB arrives at the staging rate instead of the pageable DMA rate
void staged_h2d(void* dst_dev, const void* src, size_t bytes, void* stream = nullptr);

class DeviceDataset {
 public:
  // Validates every sample against the graph inputs (reference
  // interpreter.cpp:115-125, :519-531) and uploads [first, first+count).
  // upload: the stream the copies are issued on (default: the engine
  // stream).  On another stream, ready() is an event the engine waits on.
  DeviceDataset(const Graph& g, const Dataset& ds, int64_t first = 0, int64_t count = -1,
                void* upload = nullptr);
  ~DeviceDataset();
  DeviceDataset(const DeviceDataset&) = delete;
  // make the engine stream wait for this dataset's upload
  void wait_ready() const;
  int64_t size() const { return n_; }
  const float* input(size_t k, int64_t sample) const {
    return static_cast<const float*>(bufs_[k].get()) + sample * per_[k];
  }
  size_t num_inputs() const { return bufs_.size(); }

 private:
  int64_t n_ = 0;
  void* ready_ = nullptr;  // cudaEvent_t recorded after the upload (other-stream uploads)
  std::vector<std::shared_ptr<void>> bufs_;
  std::vector<int64_t> per_;
};

// Per-sample argmax of the first graph output over every sample, on device
// (int64 [size]).
// predict_top1's device part over a HOST dataset: uploads overlap the fused
// forward (chunked on the copy stream); other engines upload, then run.
std::shared_ptr<void> predict_streamed(const engine::Plan& plan, const Graph& g,
                                       const Dataset& ds, const SimBinding* binding);

// scores (optional): also returns the output rows, [size x *per_sample] fp32.
std::shared_ptr<void> predict_device(const engine::Plan& plan, const DeviceDataset& dd,
                                     const SimBinding* binding, bool integer_regime,
                                     bool allow_fast, std::shared_ptr<void>* scores = nullptr,
                                     int64_t* per_sample = nullptr);

// Several bindings (2..4) over the same device samples (the candidate-batch
// path of the search): when the fused int8 engine applies to all of them,
// every compatible GEMM stage runs as one grouped tcgen05 launch.  Returns
// [G x N] predictions (binding g's rows at g*N), or nullptr when the grouped
// path does not apply.
// scores (optional): also returns the output rows, [G x N x per_sample] fp32.
std::shared_ptr<void> predict_device_group(const engine::Plan& plan, const DeviceDataset& dd,
                                           const std::vector<const SimBinding*>& bindings,
                                           std::shared_ptr<void>* scores = nullptr,
                                           int64_t* per_sample = nullptr);

}  // namespace quantc::gpu
