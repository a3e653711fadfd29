// kl.cu — KL-divergence threshold sweep (reference calibration.cpp:138-206).
//
// Grid = (edges, splits); each CTA stages one edge's histogram in shared
// memory (counts as doubles + int64 prefix sums, so group sums and the folded
// tail are O(1) and exact), and each thread evaluates candidate clip points
// i = 2^b .. B round-robin.  Per candidate the thread reproduces the
// reference's arithmetic sequence exactly (sequential p_sum/q_sum/kl sums,
// explicit _rn intrinsics so nothing is contracted into FMAs); only log()
// may differ from glibc by <= 1 ulp.  Per-CTA winners (first minimum: lowest
// KL, ties to the smallest i) are merged by a second tiny kernel.
#include <cfloat>

#include "common.cuh"

namespace quantc::kern {

namespace {

constexpr double kSmooth = 1e-9;
constexpr int kThreads = 256;
constexpr int kSplits = 4;

struct Best {
  double kl;
  int i;
};

__device__ __forceinline__ bool better(double kl, int i, double bkl, int bi) {
  // NaN never wins (reference: `kl < best_kl` is false for NaN)
  if (kl != kl) return false;
  if (bkl != bkl) return true;
  return kl < bkl || (kl == bkl && i < bi);
}

// KL of clip point i (reference calibration.cpp:173-203)
__device__ double kl_at(int i, int levels, const double* cnt, const long long* prefix,
                        long long total) {
  // p[b] = counts[b] for b < i-1; p[i-1] = sum_{b >= i-1} counts[b]
  const double tail = static_cast<double>(total - prefix[i - 1]);
  auto pval = [&](int b) { return b == i - 1 ? tail : cnt[b]; };
  const int merged = i / levels;

  // pass 1: p_sum over smoothed p
  double p_sum = 0.0;
  for (int b = 0; b < i; ++b) {
    double v = pval(b);
    p_sum = __dadd_rn(p_sum, v == 0.0 ? kSmooth : v);
  }
  // pass 2: q_sum over smoothed q; group value = group sum / nonzero bins
  double q_sum = 0.0;
  for (int j = 0; j < levels; ++j) {
    const int start = j * merged;
    const int end = (j == levels - 1) ? i : (j + 1) * merged;
    int nonzero = 0;
    for (int b = start; b < end; ++b) nonzero += pval(b) != 0.0;
    const long long gsum = (end == i ? total : prefix[end]) - prefix[start];
    const double value =
        nonzero ? __ddiv_rn(static_cast<double>(gsum), static_cast<double>(nonzero)) : 0.0;
    for (int b = start; b < end; ++b) {
      double q = pval(b) != 0.0 ? value : 0.0;
      q_sum = __dadd_rn(q_sum, q == 0.0 ? kSmooth : q);
    }
  }
  // pass 3: kl = sum pi * log(pi / qi)
  double kl = 0.0;
  for (int j = 0; j < levels; ++j) {
    const int start = j * merged;
    const int end = (j == levels - 1) ? i : (j + 1) * merged;
    int nonzero = 0;
    for (int b = start; b < end; ++b) nonzero += pval(b) != 0.0;
    const long long gsum = (end == i ? total : prefix[end]) - prefix[start];
    const double value =
        nonzero ? __ddiv_rn(static_cast<double>(gsum), static_cast<double>(nonzero)) : 0.0;
    for (int b = start; b < end; ++b) {
      double p = pval(b);
      double q = p != 0.0 ? value : 0.0;
      if (p == 0.0) p = kSmooth;
      if (q == 0.0) q = kSmooth;
      const double pi = __ddiv_rn(p, p_sum);
      const double qi = __ddiv_rn(q, q_sum);
      kl = __dadd_rn(kl, __dmul_rn(pi, log(__ddiv_rn(pi, qi))));
    }
  }
  return kl;
}

__global__ void __launch_bounds__(kThreads) kl_partial_kernel(const int64_t* __restrict__ counts,
                                                              int bins, int levels,
                                                              Best* __restrict__ partial) {
  extern __shared__ unsigned char smem_raw[];
  double* cnt = reinterpret_cast<double*>(smem_raw);
  long long* prefix = reinterpret_cast<long long*>(cnt + bins);  // bins + 1 entries
  const int edge = blockIdx.x;
  const int64_t* c = counts + static_cast<int64_t>(edge) * bins;
  for (int b = threadIdx.x; b < bins; b += blockDim.x) cnt[b] = static_cast<double>(c[b]);
  __syncthreads();
  if (threadIdx.x == 0) {
    long long acc = 0;
    for (int b = 0; b < bins; ++b) {
      prefix[b] = acc;
      acc += c[b];
    }
    prefix[bins] = acc;
  }
  __syncthreads();
  const long long total = prefix[bins];

  double bkl = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  int bi = levels;
  const int n_cand = bins - levels + 1;
  const int first = blockIdx.y * blockDim.x + threadIdx.x;
  const int step = gridDim.y * blockDim.x;
  // interleave large and small i across threads for balance
  for (int t = first; t < n_cand; t += step) {
    const int i = levels + t;
    const double kl = kl_at(i, levels, cnt, prefix, total);
    if (better(kl, i, bkl, bi)) {
      bkl = kl;
      bi = i;
    }
  }
  // block argmin
  for (int o = 16; o > 0; o >>= 1) {
    double okl = __shfl_xor_sync(0xffffffffu, bkl, o);
    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (better(okl, oi, bkl, bi)) {
      bkl = okl;
      bi = oi;
    }
  }
  __shared__ Best wbest[kThreads / 32];
  if ((threadIdx.x & 31) == 0) wbest[threadIdx.x >> 5] = {bkl, bi};
  __syncthreads();
  if (threadIdx.x == 0) {
    Best b = wbest[0];
    for (int w = 1; w < kThreads / 32; ++w) {
      if (better(wbest[w].kl, wbest[w].i, b.kl, b.i)) b = wbest[w];
    }
    partial[edge * gridDim.y + blockIdx.y] = b;
  }
}

__global__ void kl_merge_kernel(const Best* partial, int splits, int n_edges, int levels,
                                int* best_i, double* best_kl) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_edges) return;
  Best b = {__longlong_as_double(0x7ff0000000000000ll), levels};
  for (int s = 0; s < splits; ++s) {
    const Best& p = partial[e * splits + s];
    if (better(p.kl, p.i, b.kl, b.i)) b = p;
  }
  best_i[e] = b.i;
  best_kl[e] = b.kl;
}

}  // namespace

void kl_sweep(const int64_t* counts, int n_edges, int bins, int target_bit, int* best_i,
              double* best_kl, cudaStream_t s) {
  if (n_edges <= 0) return;
  const int levels = 1 << target_bit;
  Best* partial = nullptr;
  if (cudaMallocAsync(&partial, sizeof(Best) * n_edges * kSplits, s) != cudaSuccess) {
    throw std::runtime_error("kl_sweep: allocation failed");
  }
  const size_t smem = static_cast<size_t>(bins) * sizeof(double) +
                      static_cast<size_t>(bins + 1) * sizeof(long long);
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(kl_partial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
  }
  kl_partial_kernel<<<dim3(n_edges, kSplits), kThreads, smem, s>>>(counts, bins, levels, partial);
  QC_CUDA_CHECK_LAUNCH();
  kl_merge_kernel<<<(n_edges + 127) / 128, 128, 0, s>>>(partial, kSplits, n_edges, levels, best_i,
                                                        best_kl);
  QC_CUDA_CHECK_LAUNCH();
  cudaFreeAsync(partial, s);
}

}  // namespace quantc::kern
