// simulate.cpp — Eq. 1-3 scalars on the host, the simulated_quantize tensor
// operator on the device (reference simulate.cpp:12-93).
#include "quantc/simulate.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <stdexcept>

#include "engine.hpp"
#include "quantc/device.hpp"

namespace quantc {

double compute_scale(double threshold, int bit, int sign) {
  if (!(threshold > 0.0)) throw std::invalid_argument("threshold must be positive");
  if (bit < 2) throw std::invalid_argument("bit must be >= 2");
  if (sign != 0 && sign != 1) throw std::invalid_argument("sign must be 0 or 1");
  return threshold / std::exp2(static_cast<double>(bit - sign));
}

QuantBounds quant_bounds(int bit, int sign) {
  if (bit < 2) throw std::invalid_argument("bit must be >= 2");
  if (sign == 1) return {-(int64_t{1} << (bit - 1)), (int64_t{1} << (bit - 1)) - 1};
  return {0, (int64_t{1} << bit) - 1};
}

QParams QParams::symmetric(double threshold, int bit, DType storage) {
  QParams p;
  p.threshold = threshold;
  p.bit = bit;
  p.sign = 1;
  p.in_dtype = storage;
  p.out_dtype = storage;
  return p;
}

QParams noop_params() {
  QParams p;
  p.passthrough = true;
  p.in_dtype = f32;
  p.out_dtype = f32;
  return p;
}

Tensor simulated_quantize(const Tensor& x, const QParams& p) {
  if (x.dtype() != f32) throw std::invalid_argument("simulated_quantize needs a float32 tensor");
  kern::SqParams k = engine::resolve_sq(p);  // check_params semantics
  if (p.passthrough && !p.acc_dtype.has_value()) return x;
  engine::DevTensor d = engine::upload(x);
  kern::sim_quant(d.f(), d.f(), x.numel(), k, static_cast<cudaStream_t>(device::stream()));
  return engine::download(d, 1);
}

float simulated_quantize_value(float x, const QParams& p) {
  // The scalar form is the same device function over a one-element tensor;
  // unlike the tensor API it applies no parameter validation (as in the
  // reference, where only simulated_quantize() calls check_params).
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
  engine::DevTensor d = engine::upload(Tensor::scalar(x));
  kern::sim_quant(d.f(), d.f(), 1, k, static_cast<cudaStream_t>(device::stream()));
  return engine::download(d, 1).floats()[0];
}

int64_t asymmetric_zero_point(double min_value, double range_threshold, int bit) {
  const double s = compute_scale(range_threshold, bit, 0);
  const int64_t zp = static_cast<int64_t>(std::llround(-min_value / s));
  return std::clamp<int64_t>(zp, 0, (int64_t{1} << bit) - 1);
}

}  // namespace quantc
