// quantc/realize.hpp — strategy types and integer lowering (B200 build).
//
// Drop-in for /root/reference/proj/include/quantc/realize.hpp.  The
// reference declares these but ships no implementation;
// EdgeDecision/Strategy are the search output.  requantize_params,
// choose_storage_dtype and rewrite_clip are implemented from SPEC.md
// realize module (:593-672); realize() is implemented from that restatement
// (host/realize.cpp), the reference only declares it.
#pragma once

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "quantc/graph.hpp"
#include "quantc/hwspec.hpp"

namespace quantc {

struct RequantParams {
  int32_t multiplier = 1 << 30;
  int shift = 30;
  double value() const;
};

class RealizeError : public std::runtime_error {
 public:
  explicit RealizeError(const std::string& what) : std::runtime_error(what) {}
};

RequantParams requantize_params(double s_in, double s_out);

struct EdgeDecision {
  int bit = 8;
  double threshold = 1.0;
  int sign = 1;
  int64_t zero_point = 0;
  DType storage_dtype = i8;
  double scale() const;
};

struct Strategy {
  std::map<int, EdgeDecision> edges;
};

DType choose_storage_dtype(int bit, const std::vector<DType>& candidates, int sign = 1);
std::pair<int64_t, int64_t> rewrite_clip(double min_f, double max_f, double s_out,
                                         int64_t zero_point, DType storage);
Graph realize(const Graph& sim_g, const Strategy& strategy, const HardwareSpec& spec);

}  // namespace quantc
