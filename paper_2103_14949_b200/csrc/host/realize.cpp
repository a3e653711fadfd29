// realize.cpp — realization helpers declared by reference realize.hpp:17-62.
// The reference ships no implementation; these follow SPEC.md's realize
// module (:593-672).  Full graph lowering (realize()) is SURVEY §8(f) rank 1.
#include "quantc/realize.hpp"

#include <algorithm>
#include <cmath>

#include "quantc/simulate.hpp"

namespace quantc {

double RequantParams::value() const { return std::ldexp(static_cast<double>(multiplier), -shift); }

double EdgeDecision::scale() const { return compute_scale(threshold, bit, sign); }

RequantParams requantize_params(double s_in, double s_out) {
  if (!(s_in > 0.0) || !(s_out > 0.0)) throw RealizeError("requantize_params needs positive scales");
  int e = 0;
  const double m = std::frexp(s_in / s_out, &e);  // ratio = m * 2^e, m in [0.5, 1)
  int64_t mult = std::llround(std::ldexp(m, 31));
  int shift = 31 - e;
  if (mult == (int64_t{1} << 31)) {
    mult >>= 1;
    --shift;
  }
  RequantParams r;
  r.multiplier = static_cast<int32_t>(mult);
  r.shift = shift;
  return r;
}

DType choose_storage_dtype(int bit, const std::vector<DType>& candidates, int sign) {
  const DType* best = nullptr;
  for (const DType& d : candidates) {
    if (d.is_float() || max_bits(d) < bit) continue;
    if (sign == 1 && !d.is_signed()) continue;
    if (sign == 0 && d.is_signed()) continue;
    if (!best || d.width() < best->width()) best = &d;
  }
  if (!best) {
    throw RealizeError("no candidate dtype can hold " + std::to_string(bit) + " effective bits");
  }
  return *best;
}

std::pair<int64_t, int64_t> rewrite_clip(double min_f, double max_f, double s_out,
                                         int64_t zero_point, DType storage) {
  int64_t lo = std::llround(min_f / s_out) + zero_point;
  int64_t hi = std::llround(max_f / s_out) + zero_point;
  lo = std::clamp(lo, storage.min_value(), storage.max_value());
  hi = std::clamp(hi, storage.min_value(), storage.max_value());
  return {lo, hi};
}

Graph realize(const Graph& sim_g, const Strategy& strategy, const HardwareSpec& spec) {
  (void)sim_g;
  (void)strategy;
  (void)spec;
  throw RealizeError("realize(): integer lowering is not part of this build (SURVEY.md §8f)");
}

}  // namespace quantc
