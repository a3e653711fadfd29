// stats.cu — calibration statistics (reference calibration.cpp:62-113).
//
// minmax: exact double min/max of fp32 values.  Per-thread partials over a
//   grid-stride float4 stream, warp shuffles, one atomicMin/atomicMax per
//   block on monotone uint64 keys (order-independent, hence identical to the
//   reference's sequential merge for non-NaN data).  4 B/element.
// histogram: |v| binned against the final absmax into B bins, bin i covering
//   (i*w, (i+1)*w], zeros in bin 0 (calibration.cpp:28-33).  Block-private
//   shared-memory u32 histogram (B <= 8192 bins => <= 32 KB), flushed with one
//   64-bit global atomic per non-empty bin.  4 B/element.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace quantc::kern {

namespace {

__global__ void minmax_init_kernel(unsigned long long* keys, int n_slots) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_slots) {
    keys[2 * i] = ~0ull;     // min key starts at +max
    keys[2 * i + 1] = 0ull;  // max key starts at -max
  }
}

__global__ void __launch_bounds__(256) minmax_kernel(const float* __restrict__ x, int64_t n,
                                                     unsigned long long* keys) {
  float lo = __int_as_float(0x7f800000), hi = __int_as_float(0xff800000);  // +inf, -inf
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  if ((reinterpret_cast<uintptr_t>(x) & 15) == 0) {
    const int64_t n4 = n >> 2;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    for (int64_t i = tid; i < n4; i += stride) {
      float4 v = __ldg(x4 + i);
      lo = fminf(lo, fminf(fminf(v.x, v.y), fminf(v.z, v.w)));
      hi = fmaxf(hi, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
    }
    for (int64_t i = (n4 << 2) + tid; i < n; i += stride) {
      lo = fminf(lo, x[i]);
      hi = fmaxf(hi, x[i]);
    }
  } else {
    for (int64_t i = tid; i < n; i += stride) {
      lo = fminf(lo, x[i]);
      hi = fmaxf(hi, x[i]);
    }
  }
  // float -> double conversion is exact and monotone; reduce keys.
  unsigned long long kmin = order_key(static_cast<double>(lo));
  unsigned long long kmax = order_key(static_cast<double>(hi));
  for (int o = 16; o > 0; o >>= 1) {
    kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
    kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
  }
  __shared__ unsigned long long smin[8], smax[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    smin[warp] = kmin;
    smax[warp] = kmax;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (blockDim.x >> 5); ++w) {
      kmin = min(kmin, smin[w]);
      kmax = max(kmax, smax[w]);
    }
    atomicMin(keys, kmin);
    atomicMax(keys + 1, kmax);
  }
}

__global__ void minmax_decode_kernel(const unsigned long long* keys, double* out, int n_slots) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_slots) {
    out[2 * i] = keys[2 * i] == ~0ull ? __longlong_as_double(0x7ff0000000000000ll)
                                      : key_to_double(keys[2 * i]);
    out[2 * i + 1] = keys[2 * i + 1] == 0ull ? __longlong_as_double(0xfff0000000000000ll)
                                             : key_to_double(keys[2 * i + 1]);
  }
}

// bin_index of reference calibration.cpp:28-33 for absmax > 0
__device__ __forceinline__ int bin_of(float v, double absmax, double bins_over_absmax, int bins) {
  const double a = fabs(static_cast<double>(v));
  if (!(a > 0.0)) return 0;  // a <= 0 (NaN falls through the reference clamp to 0 as well)
  double t = __dmul_rn(a, bins_over_absmax);
  const double fr = t - floor(t);
  const double tol = t * 0x1p-48 + 0x1p-1000;
  if (fr <= tol || fr >= 1.0 - tol) {
    t = __dmul_rn(__ddiv_rn(a, absmax), static_cast<double>(bins));
  }
  int idx = static_cast<int>(ceil(t)) - 1;
  return idx < 0 ? 0 : (idx > bins - 1 ? bins - 1 : idx);
}

// Same bin with an fp32 fast path: t_f = |v| * RN32(B/absmax) is within a few
// ulp (relative 2^-21) of the reference's double t; when t_f is farther than
// that from every integer, floor(t_f) = floor(t) and t is not an integer, so
// the bin ceil(t) - 1 = floor(t_f).  floor(t_f) (t_f < 2^22) is the integer
// bits of RZ(t_f + 1.5*2^23).  Near an integer (or for zeros / huge t) the
// exact double bin_of decides.
__device__ __forceinline__ int bin_of_fast(float v, float r_f, double absmax,
                                           double bins_over_absmax, int bins) {
  const float a = fabsf(v);
  const float t = __fmul_rn(a, r_f);
  const float T = __fadd_rz(t, 12582912.0f);
  const float fl = __fsub_rn(T, 12582912.0f);
  const float fr = __fsub_rn(t, fl);
  const float margin = t * 0x1p-19f;
  if (a > 0.0f && t < 4194304.0f && fr > margin && fr < 1.0f - margin) {
    const int idx = __float_as_int(T) - 0x4B400000;
    return idx > bins - 1 ? bins - 1 : idx;
  }
  return bin_of(v, absmax, bins_over_absmax, bins);
}

// Shared-memory privatised histogram.  Two contention relief measures for
// activation edges (a relu edge puts ~half its elements into bin 0):
//   * bin-0 hits (zeros and |v| < absmax/bins) are counted in a register and
//     reduced per warp (one shared atomic per warp at the end);
//   * `reps` replicated sub-histograms, warp w updating copy w % reps, merged
//     once per CTA before the global atomics.
template <bool ZREG>
__global__ void __launch_bounds__(512) hist_kernel(const float* __restrict__ x, int64_t n,
                                                   double absmax, double bins_over_absmax,
                                                   int bins, int reps, unsigned long long* counts,
                                                   unsigned long long mult) {
  extern __shared__ unsigned int sh[];
  for (int b = threadIdx.x; b < bins * reps; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  unsigned int* hs = sh + ((threadIdx.x >> 5) % reps) * bins;
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  unsigned int zeros = 0;
  auto put = [&](int b) {
    if (ZREG && b == 0) {
      ++zeros;
    } else {
      atomicAdd(&hs[b], 1u);
    }
  };
  if (absmax > 0.0) {
    const float r_f = static_cast<float>(bins_over_absmax);
    if ((reinterpret_cast<uintptr_t>(x) & 15) == 0) {
      const int64_t n4 = n >> 2;
      const float4* x4 = reinterpret_cast<const float4*>(x);
      for (int64_t i = tid; i < n4; i += stride) {
        float4 v = __ldg(x4 + i);
        put(bin_of_fast(v.x, r_f, absmax, bins_over_absmax, bins));
        put(bin_of_fast(v.y, r_f, absmax, bins_over_absmax, bins));
        put(bin_of_fast(v.z, r_f, absmax, bins_over_absmax, bins));
        put(bin_of_fast(v.w, r_f, absmax, bins_over_absmax, bins));
      }
      for (int64_t i = (n4 << 2) + tid; i < n; i += stride) {
        put(bin_of(x[i], absmax, bins_over_absmax, bins));
      }
    } else {
      for (int64_t i = tid; i < n; i += stride) put(bin_of(x[i], absmax, bins_over_absmax, bins));
    }
  } else {
    // absmax <= 0: every element lands in bin 0 (calibration.cpp:103)
    for (int64_t i = tid; i < n; i += stride) ++zeros;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) zeros += __shfl_xor_sync(0xffffffffu, zeros, o);
  if ((threadIdx.x & 31) == 0 && zeros) atomicAdd(&sh[0], zeros);
  __syncthreads();
  for (int b = threadIdx.x; b < bins; b += blockDim.x) {
    unsigned long long c = 0;
    for (int r = 0; r < reps; ++r) c += sh[r * bins + b];
    if (c) atomicAdd(counts + b, c * mult);
  }
}

}  // namespace

void minmax_init(unsigned long long* keys, int n_slots, cudaStream_t s) {
  if (n_slots <= 0) return;
  minmax_init_kernel<<<(n_slots + 255) / 256, 256, 0, s>>>(keys, n_slots);
  QC_CUDA_CHECK_LAUNCH();
}

void minmax_accumulate(const float* x, int64_t n, unsigned long long* keys2, cudaStream_t s) {
  if (n <= 0) return;
  minmax_kernel<<<grid_for((n + 3) / 4, 256, 148 * 8), 256, 0, s>>>(x, n, keys2);
  QC_CUDA_CHECK_LAUNCH();
}

void minmax_decode(const unsigned long long* keys, double* out, int n_slots, cudaStream_t s) {
  if (n_slots <= 0) return;
  minmax_decode_kernel<<<(n_slots + 255) / 256, 256, 0, s>>>(keys, out, n_slots);
  QC_CUDA_CHECK_LAUNCH();
}

void histogram_accumulate(const float* x, int64_t n, double absmax, int bins,
                          unsigned long long* counts, unsigned long long multiplier,
                          cudaStream_t s) {
  if (n <= 0) return;
  const size_t one = static_cast<size_t>(bins) * sizeof(unsigned int);
  if (one > 200 * 1024) throw std::runtime_error("histogram: too many bins for shared memory");
  static const int reps0 = [] {
    const char* e = std::getenv("QUANTC_HIST_REPS");
    return e ? std::max(1, std::atoi(e)) : 4;
  }();
  int reps = reps0;
  while (reps > 1 && one * reps > 64 * 1024) reps >>= 1;
  const size_t smem = one * reps;
  static const bool zreg = [] {
    const char* e = std::getenv("QUANTC_HIST_ZREG");
    return e ? std::atoi(e) != 0 : false;  // measured: the branch costs more than it saves
  }();
  auto kfn = zreg ? hist_kernel<true> : hist_kernel<false>;
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  }
  // bins/absmax: with a power-of-two bin count this equals bins * RN(1/absmax)
  const double boa = absmax > 0.0 ? static_cast<double>(bins) / absmax : 0.0;
  const int grid = grid_for((n + 3) / 4, 512, 148 * 4);
  kfn<<<grid, 512, smem, s>>>(x, n, absmax, boa, bins, reps, counts, multiplier);
  QC_CUDA_CHECK_LAUNCH();
}

}  // namespace quantc::kern
