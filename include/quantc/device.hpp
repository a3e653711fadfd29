// quantc/device.hpp — B200 extension: device context and errors.
//
// Not part of the reference API.  One process drives one GPU (the device is
// picked from QUANTC_DEVICE, else LOCAL_RANK, else 0); all engine work is
// issued on one stream of that device with stream-ordered allocation.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "quantc/interpreter.hpp"

namespace quantc {

class DeviceError : public std::runtime_error {
 public:
  explicit DeviceError(const std::string& what) : std::runtime_error(what) {}
};

namespace device {

// Engine selection for sim-quant evaluation (CandidateEvaluator, predict_top1
// with a binding).  kExact: FP64 exact-order conv/dense everywhere
// (bit-identical to the reference).  kFast: int8 tcgen05 GEMMs wherever both
// MAC operands are int8-grid simulated-quantize outputs (bit-identical when
// thresholds are powers of two; documented tolerance otherwise).  kAuto: kFast
// only where it is provably bit-identical, kExact elsewhere.
enum class EngineMode { kExact = 0, kFast = 1, kAuto = 2 };

void set_engine_mode(EngineMode m);
EngineMode engine_mode();

int current_device();
void* stream();       // cudaStream_t of the engine
void* copy_stream();  // cudaStream_t for uploads that overlap engine work
void* aux_stream(int i);  // i-th auxiliary compute stream (created on first use)

// Page-locked host ranges.  Datasets created through the C-ABI pin their
// sample storage once (cudaHostRegister) so DeviceDataset DMAs straight from
// it instead of packing into staging.  pin_host is best effort (false: not
// pinned, e.g. no device or over QUANTC_PIN_MAX_MB); unpin_host before the
// memory is freed.
bool pin_host(const void* p, size_t bytes);
void unpin_host(const void* p);
bool host_pinned(const void* p, size_t bytes);

// A contiguous page-locked copy of a C-ABI dataset's input samples (sample s
// at [s * bytes_per, (s + 1) * bytes_per)): one DMA per upload instead of one
// per sample.  alloc_pinned returns nullptr when it cannot (no device, cap).
void* alloc_pinned(size_t bytes);
void free_pinned(void* p);
void set_dataset_mirror(const void* dataset, const void* pinned, size_t bytes_per, int64_t n);
void clear_dataset_mirror(const void* dataset);
bool dataset_mirror(const void* dataset, const void** pinned, size_t* bytes_per, int64_t* n);
void synchronize();
size_t memory_budget_bytes();  // per-batch activation budget
// make sure the engine stream's allocator pool holds at least `bytes` (one
// allocate/free pair; the pool keeps released memory)
void pool_reserve(size_t bytes);

// Counters (for bench / profiling evidence).
struct Counters {
  int64_t kernel_launches = 0;  // every sm_100a kernel this library launched
  int64_t tcgen05_gemms = 0;
  int64_t f64_convs = 0;
  int64_t fused_batches = 0;  // batches evaluated by the fused int8 dataflow (engine v2)
  int64_t simt_int_convs = 0;  // realized int conv/dense on the CUDA-core backend
};
Counters& counters();

// Optional per-GEMM timing with CUDA events on the engine stream: when
// enabled, every tcgen05 GEMM launch is bracketed by events and its
// algorithmic int8 op count (2*M*N*K_true) recorded.
void profile_enable(bool on);
bool profile_enabled();
void profile_gemm_begin();
// ops: algorithmic int8 ops (2*M*N*K_true); bytes: algorithmic HBM bytes of
// the launch (each operand / result touched once)
void profile_gemm_end(double ops, double bytes = 0.0);
// drains recorded events: total GEMM ms, launches, algorithmic ops
void profile_read(double* gemm_ms, int64_t* gemm_launches, double* gemm_ops,
                  double* gemm_bytes = nullptr);

}  // namespace device


// Two-pass calibration pieces for sharded (multi-GPU) statistics: pass 1
// exact extrema of the listed canonical edges over this shard; pass 2
// histograms against the GLOBAL absmax (after the extrema all-reduce).
// collect_stats == pass1 + absmax + pass2 on one shard.
// shard_key != 0 (e.g. the C-ABI dataset handle's uid) lets pass 2 on the
// same graph, key and edges reuse the activations pass 1 kept resident; 0
// recomputes the forward in pass 2.  (quantc/distributed.hpp's collect_stats
// runs both passes and the merges in one call.)
void collect_extrema(const Graph& g, const std::vector<Sample>& shard, const std::vector<int>& edges,
                     std::vector<double>* mins, std::vector<double>* maxs, uint64_t shard_key = 0);
void collect_histograms(const Graph& g, const std::vector<Sample>& shard,
                        const std::vector<int>& edges, const std::vector<double>& absmax, int bins,
                        std::vector<int64_t>* counts /* edges x bins */, uint64_t shard_key = 0);

// predict_top1's fp32 score rows (first graph output, samples x per-sample
// numel) under the active engine mode: the fused int8 engine in auto/fast
// mode when eligible, the FP64 exact engine otherwise.  Lets tests compare
// engines bit for bit below the argmax.
// Why the fused int8 engine does or does not run this graph under this
// binding in the active engine mode: "" when it runs, else the reason
// (the plan compiler's or the binding's).  Diagnostics for tests / users.
std::string fused_status(const Graph& g, const SimBinding* binding);

std::vector<float> predict_scores(const Graph& g, const std::vector<Sample>& dataset,
                                  const SimBinding* binding, int64_t* per_sample);

}  // namespace quantc
