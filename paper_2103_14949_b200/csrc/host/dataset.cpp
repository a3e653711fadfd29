// dataset.cpp — device-resident samples and the batched prediction loop.
#include "dataset.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <vector>

#include "quantc/parallel.hpp"

#include "fastplan.hpp"
#include "quantc/device.hpp"

namespace quantc::gpu {

namespace {
cudaStream_t S() { return static_cast<cudaStream_t>(device::stream()); }

// Reusable pinned staging for sample uploads: two chunk buffers, packed by
// host threads while the other chunk's DMA runs.  Pinned and reused, so an
// upload touches no fresh pages and copies at full PCIe/C2C rate.
class Staging {
 public:
  static constexpr size_t kChunk = size_t{8} << 20;

  static Staging& get() {
    static Staging s;
    return s;
  }
  std::mutex& mu() { return mu_; }

  // pack `count` samples of `bytes_per` each via pack(sample, dst) and copy
  // them to dst_dev, chunk by chunk
  void upload(uint8_t* dst_dev, int64_t count, size_t bytes_per,
              const std::function<void(int64_t, uint8_t*)>& pack, cudaStream_t us) {
    ensure();
    const int64_t per_chunk = std::max<int64_t>(1, static_cast<int64_t>(kChunk / bytes_per));
    int ci = 0;
    for (int64_t s0 = 0; s0 < count; s0 += per_chunk, ++ci) {
      const int64_t n = std::min(per_chunk, count - s0);
      const int slot = ci & 1;
      uint8_t* buf = static_cast<uint8_t*>(buf_[slot]);
      const size_t bytes = static_cast<size_t>(n) * bytes_per;
      if (bytes > kChunk) {
        // one sample larger than a chunk: pageable path
        std::vector<uint8_t> tmp(bytes);
        for (int64_t s = 0; s < n; ++s) pack(s0 + s, tmp.data() + s * bytes_per);
        check(cudaMemcpyAsync(dst_dev + s0 * bytes_per, tmp.data(), bytes, cudaMemcpyHostToDevice, us));
        check(cudaStreamSynchronize(us));
        continue;
      }
      check(cudaEventSynchronize(ev_[slot]));  // DMA out of this buffer finished
      static const int workers = [] {
        const char* e = std::getenv("QUANTC_PACK_WORKERS");
        return e ? std::max(1, std::atoi(e)) : 3;  // memcpy-bound; more threads only contend (B200 box, 16 cores)
      }();
      parallel_for(static_cast<size_t>(n), n >= 4 ? workers : 1,
                   [&](size_t s) { pack(s0 + static_cast<int64_t>(s), buf + s * bytes_per); });
      check(cudaMemcpyAsync(dst_dev + s0 * bytes_per, buf, bytes, cudaMemcpyHostToDevice, us));
      check(cudaEventRecord(ev_[slot], us));
    }
  }

 private:
  void ensure() {
    if (buf_[0]) return;
    for (int i = 0; i < 2; ++i) {
      check(cudaHostAlloc(&buf_[i], kChunk, cudaHostAllocDefault));
      check(cudaEventCreateWithFlags(&ev_[i], cudaEventDisableTiming));
      check(cudaEventRecord(ev_[i], S()));
    }
  }
  static void check(cudaError_t e) {
    if (e != cudaSuccess) throw DeviceError(std::string("staging: ") + cudaGetErrorString(e));
  }
  std::mutex mu_;
  void* buf_[2] = {nullptr, nullptr};
  cudaEvent_t ev_[2] = {nullptr, nullptr};
};
}  // namespace

void staged_h2d(void* dst_dev, const void* src, size_t bytes, void* stream) {
  const cudaStream_t us = stream ? static_cast<cudaStream_t>(stream) : S();
  constexpr size_t kUnit = size_t{1} << 20;
  const size_t units = bytes / kUnit, tail = bytes - units * kUnit;
  const uint8_t* s8 = static_cast<const uint8_t*>(src);
  uint8_t* d8 = static_cast<uint8_t*>(dst_dev);
  if (units > 0) {
    Staging& st = Staging::get();
    std::lock_guard<std::mutex> lk(st.mu());
    st.upload(d8, static_cast<int64_t>(units), kUnit,
              [&](int64_t u, uint8_t* dst) { std::memcpy(dst, s8 + static_cast<size_t>(u) * kUnit, kUnit); },
              us);
  }
  if (tail > 0 && cudaMemcpyAsync(d8 + units * kUnit, s8 + units * kUnit, tail, cudaMemcpyHostToDevice, us) !=
                      cudaSuccess) {
    throw DeviceError("staged upload failed");
  }
}

DeviceDataset::DeviceDataset(const Graph& g, const Dataset& ds, int64_t first, int64_t count,
                             void* upload) {
  const cudaStream_t us = upload ? static_cast<cudaStream_t>(upload) : S();
  if (count < 0) count = static_cast<int64_t>(ds.size()) - first;
  n_ = count;
  const size_t n_in = g.inputs().size();
  for (size_t k = 0; k < n_in; ++k) {
    const Node& node = g.node(g.inputs()[k]);
    const std::string name = node.attr_or<std::string>("name", "");
    const auto shape = node.attr<std::vector<int64_t>>("shape");
    const int64_t per = shape_numel(shape);
    for (int64_t s = 0; s < count; ++s) {
      const Sample& smp = ds[static_cast<size_t>(first + s)];
      if (smp.inputs.size() != n_in) {
        throw EvalError("sample provides " + std::to_string(smp.inputs.size()) + " tensors for " +
                        std::to_string(n_in) + " graph inputs");
      }
      const Tensor& t = smp.inputs[k];
      if (t.shape() != shape) {
        throw EvalError("input " + name + " has shape " + shape_to_string(t.shape()) +
                        ", expected " + shape_to_string(shape));
      }
      if (!t.dtype().is_float()) {
        throw EvalError("B200 engine: graph inputs must be float32 (input " + name + ")");
      }
    }
    auto buf = engine::device_alloc(static_cast<size_t>(per * count) * 4);
    if (us != S()) {
      // the buffer comes from the engine stream's pool: order the copies after it
      cudaEvent_t alloc_done;
      cudaEventCreateWithFlags(&alloc_done, cudaEventDisableTiming);
      cudaEventRecord(alloc_done, S());
      cudaStreamWaitEvent(us, alloc_done, 0);
      cudaEventDestroy(alloc_done);
    }
    const void* mirror = nullptr;
    size_t mirror_bytes = 0;
    int64_t mirror_n = 0;
    if (n_in == 1 && per * count > 0 && device::dataset_mirror(&ds, &mirror, &mirror_bytes, &mirror_n) &&
        mirror_bytes == static_cast<size_t>(per) * 4 && first + count <= mirror_n) {
      // the dataset's contiguous page-locked mirror: one DMA
      const cudaError_t e = cudaMemcpyAsync(
          buf.get(), static_cast<const uint8_t*>(mirror) + static_cast<size_t>(first) * mirror_bytes,
          static_cast<size_t>(count) * mirror_bytes, cudaMemcpyHostToDevice, us);
      if (e != cudaSuccess) throw DeviceError(std::string("dataset upload: ") + cudaGetErrorString(e));
      bufs_.push_back(buf);
      per_.push_back(per);
      continue;
    }
    bool pinned = per * count > 0;
    for (int64_t s = 0; s < count && pinned; ++s) {
      pinned = device::host_pinned(ds[static_cast<size_t>(first + s)].inputs[k].floats().data(),
                                   static_cast<size_t>(per) * 4);
    }
    if (pinned) {
      // page-locked samples (C-ABI datasets): DMA straight from them, merging
      // samples that happen to be contiguous
      const size_t bytes_per = static_cast<size_t>(per) * 4;
      int64_t s = 0;
      while (s < count) {
        const auto* src = reinterpret_cast<const uint8_t*>(ds[static_cast<size_t>(first + s)].inputs[k].floats().data());
        int64_t run = 1;
        while (s + run < count &&
               reinterpret_cast<const uint8_t*>(ds[static_cast<size_t>(first + s + run)].inputs[k].floats().data()) ==
                   src + run * bytes_per) {
          ++run;
        }
        const cudaError_t e = cudaMemcpyAsync(static_cast<uint8_t*>(buf.get()) + s * bytes_per, src,
                                              static_cast<size_t>(run) * bytes_per,
                                              cudaMemcpyHostToDevice, us);
        if (e != cudaSuccess) throw DeviceError(std::string("dataset upload: ") + cudaGetErrorString(e));
        s += run;
      }
    } else if (per * count > 0) {
      Staging& st = Staging::get();
      std::lock_guard<std::mutex> lk(st.mu());
      st.upload(static_cast<uint8_t*>(buf.get()), count, static_cast<size_t>(per) * 4,
                [&](int64_t s, uint8_t* dst) {
                  const Tensor& t = ds[static_cast<size_t>(first + s)].inputs[k];
                  std::memcpy(dst, t.floats().data(), static_cast<size_t>(per) * 4);
                },
                us);
    }
    bufs_.push_back(buf);
    per_.push_back(per);
  }
  if (us != S()) {
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaEventRecord(e, us);
    ready_ = e;
  }
}

DeviceDataset::~DeviceDataset() {
  if (ready_) {
    // the buffers are freed on the engine stream; the copies must be done
    cudaStreamWaitEvent(S(), static_cast<cudaEvent_t>(ready_), 0);
    cudaEventDestroy(static_cast<cudaEvent_t>(ready_));
  }
}

void DeviceDataset::wait_ready() const {
  if (ready_) cudaStreamWaitEvent(S(), static_cast<cudaEvent_t>(ready_), 0);
}

namespace {
// the fused int8 engine applies: the plan compiles and the binding is
// eligible (power-of-two scales in auto mode => bit-identical)
bool fused_ready(const engine::Plan& plan, const SimBinding* binding, bool integer_regime,
                 bool allow_fast) {
  const auto mode = device::engine_mode();
  const char* fused_env = std::getenv("QUANTC_FUSED");
  const bool fused_on = !(fused_env && std::string(fused_env) == "0");
  if (!(allow_fast && !integer_regime && fused_on && mode != device::EngineMode::kExact &&
        kern::gemm_s8_tcgen05_available())) {
    return false;
  }
  if (!plan.fused_tried) {
    plan.fused_tried = true;
    plan.fused = std::make_shared<fast::FastPlan>(plan);
  }
  return plan.fused->ok() && plan.fused->eligible(binding, mode == device::EngineMode::kAuto);
}
}  // namespace

namespace {
// One fused forward of `b` samples starting at sample `first` of dd,
// optionally split across QUANTC_STREAMS streams: group g runs on its own
// FastPlan instance (own arena, tables, weight-code cache) and stream.
// Results are per sample, hence identical.  Default 1: measured on B200 at
// batch 64, 2 streams 1.58 ms and 3 streams 1.92 ms per step vs 1.33 ms —
// the persistent one-CTA-per-SM kernels of two streams do not co-run, they
// only serialise with extra per-group fixed costs.
void fused_predict(const engine::Plan& plan, const DeviceDataset& dd, int64_t first, int b,
                   const SimBinding* binding, int64_t* preds, float* scores) {
  static const int streams_env = [] {
    const char* e = std::getenv("QUANTC_STREAMS");
    return e ? std::max(1, std::atoi(e)) : 1;
  }();
  const int64_t per = plan.fused->out_per_sample();
  auto run = [&](fast::FastPlan& fp, int64_t f0, int n) {
    std::vector<const float*> ins;
    for (size_t k = 0; k < dd.num_inputs(); ++k) ins.push_back(dd.input(k, f0));
    fp.predict(n, ins, binding, preds + (f0 - first), scores ? scores + (f0 - first) * per : nullptr);
  };
  const int G = std::min(streams_env, std::max(1, b / 16));
  if (G <= 1 || device::profile_enabled()) {
    run(*plan.fused, first, b);
    return;
  }
  while (static_cast<int>(plan.fused_aux.size()) < G - 1) {
    auto fp = std::make_shared<fast::FastPlan>(plan);
    fp->set_stream(device::aux_stream(static_cast<int>(plan.fused_aux.size())));
    plan.fused_aux.push_back(fp);
  }
  const cudaStream_t s0 = S();
  cudaEvent_t start;
  cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
  cudaEventRecord(start, s0);
  for (int g = 1; g < G; ++g) {
    cudaStreamWaitEvent(static_cast<cudaStream_t>(device::aux_stream(g - 1)), start, 0);
  }
  cudaEventDestroy(start);
  // contiguous sample groups, sizes differing by at most one
  int64_t f0 = first;
  for (int g = 0; g < G; ++g) {
    const int n = b / G + (g < b % G ? 1 : 0);
    run(g == 0 ? *plan.fused : *plan.fused_aux[static_cast<size_t>(g - 1)], f0, n);
    f0 += n;
  }
  for (int g = 1; g < G; ++g) {
    cudaEvent_t done;
    cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
    cudaEventRecord(done, static_cast<cudaStream_t>(device::aux_stream(g - 1)));
    cudaStreamWaitEvent(s0, done, 0);
    cudaEventDestroy(done);
  }
}
}  // namespace

std::shared_ptr<void> predict_streamed(const engine::Plan& plan, const Graph& g,
                                       const Dataset& ds, const SimBinding* binding) {
  static const int parts_env = [] {
    const char* e = std::getenv("QUANTC_E2E_PARTS");
    return e ? std::max(1, std::atoi(e)) : 0;
  }();
  const int64_t n = static_cast<int64_t>(ds.size());
  if (!fused_ready(plan, binding, false, binding != nullptr)) {
    DeviceDataset dd(g, ds);
    return predict_device(plan, dd, binding, false, binding != nullptr);
  }
  // QUANTC_E2E_PARTS > 1 splits the call so part k+1's packing and DMA overlap
  // the forward of part k.  Default 1: host packing into pinned staging is the
  // bottleneck of this path, and each extra part repeats the per-launch host
  // work (measured on B200: 2 parts -28%, 4 parts -55% at 64 images)
  const int parts = parts_env ? parts_env : 1;
  auto preds = engine::device_alloc(static_cast<size_t>(std::max<int64_t>(1, n)) * 8);
  std::vector<std::unique_ptr<DeviceDataset>> dds;
  const int64_t per = (n + parts - 1) / parts;
  // every part's buffers are allocated (engine-stream pool) and its upload
  // queued on the copy stream BEFORE any forward is queued, so part k+1's DMA
  // runs under part k's forward instead of waiting behind it
  std::vector<int64_t> firsts;
  for (int64_t first = 0; first < n; first += per) {
    firsts.push_back(first);
    dds.push_back(std::make_unique<DeviceDataset>(g, ds, first, std::min(per, n - first),
                                                  device::copy_stream()));
  }
  for (size_t p = 0; p < dds.size(); ++p) {
    const int64_t first = firsts[p];
    const int64_t cnt = dds[p]->size();
    const DeviceDataset& dd = *dds[p];
    dd.wait_ready();
    const int fb = static_cast<int>(std::min<int64_t>(cnt, 256));
    for (int64_t f = 0; f < cnt; f += fb) {
      const int b = static_cast<int>(std::min<int64_t>(fb, cnt - f));
      fused_predict(plan, dd, f, b, binding, static_cast<int64_t*>(preds.get()) + first + f,
                    nullptr);
    }
  }
  return preds;
}

std::shared_ptr<void> predict_device_group(const engine::Plan& plan, const DeviceDataset& dd,
                                           const std::vector<const SimBinding*>& bindings,
                                           std::shared_ptr<void>* scores, int64_t* per_sample) {
  const int G = static_cast<int>(bindings.size());
  if (G < 2) return nullptr;
  for (const SimBinding* b : bindings) {
    if (!fused_ready(plan, b, false, true)) return nullptr;
  }
  const int64_t n = dd.size();
  auto preds = engine::device_alloc(static_cast<size_t>(std::max<int64_t>(1, G * n)) * 8);
  auto* p = static_cast<int64_t*>(preds.get());
  const int64_t per = plan.fused->out_per_sample();
  if (scores) {
    *scores = engine::device_alloc(static_cast<size_t>(std::max<int64_t>(1, G * n * per)) * 4);
    *per_sample = per;
  }
  const int fb = static_cast<int>(std::min<int64_t>(std::max<int64_t>(1, n), 256));
  for (int64_t first = 0; first < n; first += fb) {
    const int b = static_cast<int>(std::min<int64_t>(fb, n - first));
    std::vector<const float*> ins;
    for (size_t k = 0; k < dd.num_inputs(); ++k) ins.push_back(dd.input(k, first));
    std::vector<int64_t*> outs;
    for (int g = 0; g < G; ++g) outs.push_back(p + g * n + first);
    std::vector<float*> souts;
    if (scores) {
      for (int g = 0; g < G; ++g) {
        souts.push_back(static_cast<float*>(scores->get()) + (g * n + first) * per);
      }
    }
    plan.fused->predict_group(b, ins, bindings, outs, scores ? &souts : nullptr);
  }
  return preds;
}

std::shared_ptr<void> predict_device(const engine::Plan& plan, const DeviceDataset& dd,
                                     const SimBinding* binding, bool integer_regime,
                                     bool allow_fast, std::shared_ptr<void>* scores,
                                     int64_t* per_sample) {
  const Graph& g = plan.graph();
  if (g.outputs().empty()) throw EvalError("model has no outputs");
  const int out_step = plan.step_of(g.outputs()[0].node);
  auto preds = engine::device_alloc(static_cast<size_t>(std::max<int64_t>(1, dd.size())) * 8);
  // engine v2: fused int8 dataflow, when the graph compiles and the binding is
  // eligible (power-of-two scales in auto mode => bit-identical)
  {
    if (fused_ready(plan, binding, integer_regime, allow_fast)) {
      const int fb = std::min<int64_t>(std::max<int64_t>(1, dd.size()), 256);
      const int64_t per = plan.fused->out_per_sample();
      if (scores) {
        *scores = engine::device_alloc(static_cast<size_t>(dd.size() * per) * 4);
        *per_sample = per;
      }
      for (int64_t first = 0; first < dd.size(); first += fb) {
        const int b = static_cast<int>(std::min<int64_t>(fb, dd.size() - first));
        fused_predict(plan, dd, first, b, binding, static_cast<int64_t*>(preds.get()) + first,
                      scores ? static_cast<float*>(scores->get()) + first * per : nullptr);
      }
      return preds;
    }
  }
  const int batch = plan.batch_for(dd.size());
  for (int64_t first = 0; first < dd.size(); first += batch) {
    const int b = static_cast<int>(std::min<int64_t>(batch, dd.size() - first));
    engine::RunSpec spec;
    spec.batch = b;
    for (size_t k = 0; k < dd.num_inputs(); ++k) spec.inputs.push_back(dd.input(k, first));
    spec.binding = binding;
    spec.integer_regime = integer_regime;
    spec.allow_fast = allow_fast;
    spec.keep = {out_step};
    auto vals = engine::run(plan, spec);
    const engine::DevTensor& out = vals[0];
    if (!out.dtype.is_float()) {
      throw EvalError("model output is not dequantized to a float score vector");
    }
    int64_t* dst = static_cast<int64_t*>(preds.get()) + first;
    if (out.per_numel() == 0) throw EvalError("empty score vector");
    if (scores) {
      const int64_t per = out.per_numel();
      if (!*scores) {
        *scores = engine::device_alloc(static_cast<size_t>(dd.size() * per) * 4);
        *per_sample = per;
      }
      float* sdst = static_cast<float*>(scores->get()) + first * per;
      for (int s = 0; s < b; ++s) {
        cudaMemcpyAsync(sdst + s * per, out.f() + (out.batched ? s * per : 0), per * 4,
                        cudaMemcpyDeviceToDevice, S());
      }
    }
    if (out.batched) {
      kern::argmax_rows(out.f(), b, out.per_numel(), dst, S());
    } else {
      kern::argmax_rows(out.f(), 1, out.per_numel(), dst, S());
      for (int s = 1; s < b; ++s) {
        cudaMemcpyAsync(dst + s, dst, 8, cudaMemcpyDeviceToDevice, S());
      }
    }
  }
  return preds;
}

}  // namespace quantc::gpu

namespace quantc {
std::string fused_status(const Graph& g, const SimBinding* binding) {
  const engine::PlanLease lease = engine::lease_plan(g);
  const engine::Plan& plan = lease.plan();
  const auto mode = device::engine_mode();
  if (mode == device::EngineMode::kExact) return "engine mode is exact";
  if (!kern::gemm_s8_tcgen05_available()) return "tcgen05 unavailable on this device";
  if (!plan.fused_tried) {
    plan.fused_tried = true;
    plan.fused = std::make_shared<fast::FastPlan>(plan);
  }
  if (!plan.fused->ok()) return "plan: " + plan.fused->why_not();
  std::string why;
  if (!plan.fused->eligible(binding, mode == device::EngineMode::kAuto, &why)) {
    return "binding: " + why;
  }
  return "";
}
}  // namespace quantc
