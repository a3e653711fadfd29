// dataset.cpp — device-resident samples and the batched prediction loop.
#include "dataset.hpp"

#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <string>

#include "fastplan.hpp"
#include "quantc/device.hpp"

namespace quantc::gpu {

namespace {
cudaStream_t S() { return static_cast<cudaStream_t>(device::stream()); }
}  // namespace

DeviceDataset::DeviceDataset(const Graph& g, const Dataset& ds, int64_t first, int64_t count) {
  if (count < 0) count = static_cast<int64_t>(ds.size()) - first;
  n_ = count;
  const size_t n_in = g.inputs().size();
  for (size_t k = 0; k < n_in; ++k) {
    const Node& node = g.node(g.inputs()[k]);
    const std::string name = node.attr_or<std::string>("name", "");
    const auto shape = node.attr<std::vector<int64_t>>("shape");
    const int64_t per = shape_numel(shape);
    std::vector<float> host(static_cast<size_t>(per * count));
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
      std::memcpy(host.data() + s * per, t.floats().data(), static_cast<size_t>(per) * 4);
    }
    auto buf = engine::device_alloc(host.size() * 4);
    if (!host.empty()) {
      cudaError_t e = cudaMemcpyAsync(buf.get(), host.data(), host.size() * 4,
                                      cudaMemcpyHostToDevice, S());
      if (e != cudaSuccess) throw DeviceError(cudaGetErrorString(e));
    }
    bufs_.push_back(buf);
    per_.push_back(per);
    device::synchronize();  // host staging goes out of scope
  }
}

std::shared_ptr<void> predict_device(const engine::Plan& plan, const DeviceDataset& dd,
                                     const SimBinding* binding, bool integer_regime,
                                     bool allow_fast) {
  const Graph& g = plan.graph();
  if (g.outputs().empty()) throw EvalError("model has no outputs");
  const int out_step = plan.step_of(g.outputs()[0].node);
  auto preds = engine::device_alloc(static_cast<size_t>(std::max<int64_t>(1, dd.size())) * 8);
  // engine v2: fused int8 dataflow, when the graph compiles and the binding is
  // eligible (power-of-two scales in auto mode => bit-identical)
  const auto mode = device::engine_mode();
  const char* fused_env = std::getenv("QUANTC_FUSED");
  const bool fused_on = !(fused_env && std::string(fused_env) == "0");
  if (allow_fast && !integer_regime && fused_on && mode != device::EngineMode::kExact &&
      kern::gemm_s8_tcgen05_available()) {
    if (!plan.fused_tried) {
      plan.fused_tried = true;
      plan.fused = std::make_shared<fast::FastPlan>(plan);
    }
    if (plan.fused->ok() &&
        plan.fused->eligible(binding, mode == device::EngineMode::kAuto)) {
      const int fb = std::min<int64_t>(std::max<int64_t>(1, dd.size()), 256);
      for (int64_t first = 0; first < dd.size(); first += fb) {
        const int b = static_cast<int>(std::min<int64_t>(fb, dd.size() - first));
        std::vector<const float*> ins;
        for (size_t k = 0; k < dd.num_inputs(); ++k) ins.push_back(dd.input(k, first));
        plan.fused->predict(b, ins, binding, static_cast<int64_t*>(preds.get()) + first);
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
