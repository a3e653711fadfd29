// quantc/simulate.hpp — simulated_quantize operator and Eq. 1-3 (B200 build).
//
// Drop-in for /root/reference/proj/include/quantc/simulate.hpp.  The tensor
// operator runs as the sm_100a streaming kernel (csrc/kernels/simquant.cu);
// the scalar form is the same device function applied to one element.
#pragma once

#include <cstdint>
#include <optional>

#include "quantc/tensor.hpp"

namespace quantc {

double compute_scale(double threshold, int bit, int sign);  // reference simulate.hpp:14

struct QuantBounds {
  int64_t qmin;
  int64_t qmax;
};

QuantBounds quant_bounds(int bit, int sign);  // reference simulate.hpp:24

// reference simulate.hpp:33-45
struct QParams {
  double threshold = 0.0;
  int bit = 8;
  int sign = 1;
  DType in_dtype = i8;
  DType out_dtype = i8;
  int64_t zero_point = 0;
  bool passthrough = false;
  std::optional<DType> acc_dtype;
  double acc_scale = 0.0;

  static QParams symmetric(double threshold, int bit, DType storage);
};

QParams noop_params();

// reference simulate.hpp:54 — fp32 tensor in, fp32 tensor out (device kernel)
Tensor simulated_quantize(const Tensor& x, const QParams& p);

// reference simulate.hpp:57
float simulated_quantize_value(float x, const QParams& p);

int64_t asymmetric_zero_point(double min_value, double range_threshold, int bit);

}  // namespace quantc
