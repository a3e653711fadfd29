// common.cuh — device helpers shared by the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>

#include "kernels.h"

namespace quantc::kern {

#define QC_CUDA_CHECK_LAUNCH() ::quantc::kern::check_launch(__FILE__, __LINE__)
void check_launch(const char* file, int line);

// ---- programmatic dependent launch (PDL) -----------------------------------
// Engine kernels are launched with programmatic stream serialisation: a
// kernel may start (prologue: barriers, TMEM, tables) while its predecessor's
// last CTAs drain.  Every PDL kernel calls pdl_wait() before touching data a
// predecessor produced and before it can complete, so completion stays
// transitive along the stream.  QUANTC_NO_PDL=1 launches them plainly.
bool pdl_enabled();

__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

inline int grid_for(int64_t n, int block, int max_blocks = 148 * 16) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  return static_cast<int>(g > max_blocks ? max_blocks : g);
}

// std::clamp(v, lo, hi) for doubles, NaN passes through (reference semantics)
__device__ __forceinline__ double clampd(double v, double lo, double hi) {
  return (v < lo) ? lo : ((hi < v) ? hi : v);
}

// q = clamp(round(v/s) + zp, qmin, qmax) of reference simulate.cpp:75-76,
// with v/s evaluated as the IEEE quotient.  Fast path: v * RN(1/s) is within
// ~2 ulp of v/s; round() can only differ when that lies within a few ulp of a
// half-integer, in which case the true quotient is computed.
__device__ __forceinline__ double sq_code(double v, const SqParams& p) {
  double y = __dmul_rn(v, p.inv_s);
  const double frac = fabs(y - trunc(y));
  if (p.exact_div || fabs(frac - 0.5) <= fabs(y) * 0x1p-48 + 0x1p-1000) {
    y = __ddiv_rn(v, p.s);
  }
  const double q = __dadd_rn(round(y), p.zp);
  return clampd(q, p.qmin, p.qmax);
}

// simulated_quantize_value (reference simulate.cpp:64-78), bit-exact.
__device__ __forceinline__ float sq_value(float x, const SqParams& p) {
  double v = static_cast<double>(x);
  if (p.has_acc) v = clampd(v, p.lo, p.hi);
  if (p.passthrough) return __double2float_rn(v);
  const double q = sq_code(v, p);
  return __double2float_rn(__dmul_rn(__dsub_rn(q, p.zp), p.s));
}

// Monotone uint64 key of a double (total order matching < on non-NaN values,
// with -0.0 ordered just below +0.0).
__device__ __forceinline__ unsigned long long order_key(double d) {
  unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(d));
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_to_double(unsigned long long k) {
  unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double(static_cast<long long>(b));
}

}  // namespace quantc::kern
