// eltwise.cu — fp32 elementwise, pooling and per-sample reductions
// (reference interpreter.cpp:312-430, :533-541).  Semantics:
//   add    float + float (per element, broadcast of an unbatched operand)
//   relu   std::max(v, 0.f)          -> (v < 0) ? 0 : v   (NaN, -0.0 pass)
//   clip   std::clamp(v, lo, hi)     -> (v < lo) ? lo : (hi < v) ? hi : v
//   maxpool  best = lowest; best = (best < v) ? v : best over in-bounds taps
//   gap    sequential double sum / (double)(H*W), rounded to float
//   argmax strict '>' scan == first index of the maximum (non-NaN data)
// Op-set extension (the reference op set has neither):
//   avg_pool2d  sequential double sum over the in-bounds taps (kh, kw) of
//               (double)x * (double)(float)(1/(KH*KW)), rounded to float once
//               — bit-identical to the reference conv2d on the constant
//               depthwise rewrite (fixtures.py _avg_pool, test_rewrites.py);
//               the divisor counts padded taps (count_include_pad)
//   concat      channel concatenation of NCHW tensors (32-bit words: fp32 or
//               the int32 storage of integer tensors)
#include <cfloat>

#include "common.cuh"

namespace quantc::kern {

namespace {

__global__ void add_kernel(const float* __restrict__ a, int64_t na, const float* __restrict__ b,
                           int64_t nb, float* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    y[i] = __fadd_rn(a[na == n ? i : i % na], b[nb == n ? i : i % nb]);
  }
}

__global__ void relu_kernel(const float* __restrict__ x, float* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float v = x[i];
    y[i] = (v < 0.0f) ? 0.0f : v;
  }
}

__global__ void clip_kernel(const float* __restrict__ x, float* __restrict__ y, int64_t n,
                            float lo, float hi) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float v = x[i];
    y[i] = (v < lo) ? lo : ((hi < v) ? hi : v);
  }
}

__global__ void maxpool_kernel(const float* __restrict__ x, float* __restrict__ y, int N, int C,
                               int H, int W, int OH, int OW, int kh, int kw, int sh, int sw,
                               int ph, int pw) {
  const int64_t total = static_cast<int64_t>(N) * C * OH * OW;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int ow = static_cast<int>(i % OW);
    const int oh = static_cast<int>((i / OW) % OH);
    const int64_t nc = i / (static_cast<int64_t>(OW) * OH);
    const float* src = x + nc * H * W;
    float best = -FLT_MAX;
    for (int a = 0; a < kh; ++a) {
      const int ih = oh * sh - ph + a;
      if (ih < 0 || ih >= H) continue;
      for (int b = 0; b < kw; ++b) {
        const int iw = ow * sw - pw + b;
        if (iw < 0 || iw >= W) continue;
        const float v = src[ih * W + iw];
        best = (best < v) ? v : best;
      }
    }
    y[i] = best;
  }
}

// one warp per (n, c): lanes stage the plane through registers, lane 0 sums
// in the reference order
__global__ void avgpool_kernel(const float* __restrict__ x, float* __restrict__ y, int N, int C,
                               int H, int W, int OH, int OW, int kh, int kw, int sh, int sw,
                               int ph, int pw, double wk) {
  const int64_t total = static_cast<int64_t>(N) * C * OH * OW;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int ow = static_cast<int>(i % OW);
    const int oh = static_cast<int>((i / OW) % OH);
    const int64_t nc = i / (static_cast<int64_t>(OW) * OH);
    const float* xp = x + nc * H * W;
    double acc = 0.0;
    for (int a = 0; a < kh; ++a) {
      const int ih = oh * sh - ph + a;
      if (ih < 0 || ih >= H) continue;
      for (int b = 0; b < kw; ++b) {
        const int iw = ow * sw - pw + b;
        if (iw < 0 || iw >= W) continue;
        acc = __fma_rn(static_cast<double>(__ldg(xp + static_cast<int64_t>(ih) * W + iw)), wk, acc);
      }
    }
    y[i] = __double2float_rn(acc);
  }
}

// one input of a channel concat: rows = N, each `inner` words of x landing at
// word offset `off` of a `outer`-word output row
__global__ void concat_kernel(const uint32_t* __restrict__ x, uint32_t* __restrict__ y, int N,
                              int64_t inner, int64_t outer, int64_t off) {
  const int64_t total = static_cast<int64_t>(N) * inner;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t n = i / inner, r = i - n * inner;
    y[n * outer + off + r] = __ldg(x + i);
  }
}

__global__ void concat_v4_kernel(const uint4* __restrict__ x, uint4* __restrict__ y, int N,
                                 int64_t inner, int64_t outer, int64_t off) {
  const int64_t total = static_cast<int64_t>(N) * inner;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t n = i / inner, r = i - n * inner;
    y[n * outer + off + r] = __ldg(x + i);
  }
}

__global__ void gap_kernel(const float* __restrict__ x, float* __restrict__ y, int NC, int HW) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= NC) return;
  const float* src = x + static_cast<int64_t>(warp) * HW;
  double acc = 0.0;
  for (int base = 0; base < HW; base += 32) {
    const int idx = base + lane;
    const float v = idx < HW ? src[idx] : 0.0f;
    const int cnt = min(32, HW - base);
    for (int l = 0; l < cnt; ++l) {
      const float vl = __shfl_sync(0xffffffffu, v, l);
      acc = __dadd_rn(acc, static_cast<double>(vl));
    }
  }
  if (lane == 0) y[warp] = __double2float_rn(__ddiv_rn(acc, static_cast<double>(HW)));
}

__global__ void __launch_bounds__(256) argmax_kernel(const float* __restrict__ x, int64_t cols,
                                                     int64_t* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const float* row = x + static_cast<int64_t>(blockIdx.x) * cols;
  // reference argmax_class (interpreter.cpp:533-541): best = 0, then strict
  // '>' in index order — the first maximum over the non-NaN scores, except
  // that a NaN at index 0 is never replaced (result 0).  NaNs are skipped
  // here and index 0's NaN is applied at the end.
  float bv = -FLT_MAX;
  int64_t bi = -1;
  for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
    const float v = row[c];
    if (v == v && (bi < 0 || v > bv)) {
      bv = v;
      bi = c;
    }
  }
  auto take = [](float v, int64_t i, float& bv2, int64_t& bi2) {
    if (i < 0) return;
    if (bi2 < 0 || v > bv2 || (v == bv2 && i < bi2)) {
      bv2 = v;
      bi2 = i;
    }
  };
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    take(ov, oi, bv, bi);
  }
  __shared__ float sv[8];
  __shared__ int64_t si[8];
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = bv;
    si[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w2 = 1; w2 < static_cast<int>(blockDim.x >> 5); ++w2) take(sv[w2], si[w2], bv, bi);
    const float r0 = row[0];
    out[blockIdx.x] = (bi < 0 || r0 != r0) ? 0 : bi;
  }
}

// argmax of group blockIdx.y's rows (grouped candidate evaluation)
struct RowsPack {
  const float* x[4];
  int64_t* out[4];
};
__global__ void __launch_bounds__(256) argmax_multi_kernel(RowsPack p, int64_t cols) {
  pdl_trigger();
  pdl_wait();
  const float* row = p.x[blockIdx.y] + static_cast<int64_t>(blockIdx.x) * cols;
  float bv = -FLT_MAX;
  int64_t bi = -1;
  for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
    const float v = row[c];
    if (v == v && (bi < 0 || v > bv)) {  // NaN semantics: argmax_kernel
      bv = v;
      bi = c;
    }
  }
  __shared__ float sv[256];
  __shared__ int64_t si[256];
  sv[threadIdx.x] = bv;
  si[threadIdx.x] = bi;
  __syncthreads();
  // first maximum in column order (strict >, lowest index on ties), like argmax_kernel
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const float v2 = sv[threadIdx.x + w];
      const int64_t i2 = si[threadIdx.x + w];
      if (i2 >= 0 && (si[threadIdx.x] < 0 || v2 > sv[threadIdx.x] ||
                      (v2 == sv[threadIdx.x] && i2 < si[threadIdx.x]))) {
        sv[threadIdx.x] = v2;
        si[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const float r0 = row[0];
    p.out[blockIdx.y][blockIdx.x] = (si[0] < 0 || r0 != r0) ? 0 : si[0];
  }
}

// counts[g] += #{i : a[g * n + i] == b[i]} for group g = blockIdx.y
__global__ void count_equal_multi_kernel(const int64_t* a, const int64_t* b, int n,
                                         unsigned long long* counts) {
  pdl_trigger();
  pdl_wait();
  const int64_t* ag = a + static_cast<int64_t>(blockIdx.y) * n;
  unsigned int mine = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    mine += ag[i] == b[i];
  }
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(counts + blockIdx.y, static_cast<unsigned long long>(mine));
}

__global__ void count_equal_kernel(const int64_t* a, const int64_t* b, int n,
                                   unsigned long long* count) {
  pdl_trigger();
  pdl_wait();
  unsigned int mine = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    mine += a[i] == b[i];
  }
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(count, static_cast<unsigned long long>(mine));
}

}  // namespace

void add_f32(const float* a, int64_t na, const float* b, int64_t nb, float* y, int64_t n,
             cudaStream_t s) {
  if (n <= 0) return;
  add_kernel<<<grid_for(n, 256), 256, 0, s>>>(a, na, b, nb, y, n);
  QC_CUDA_CHECK_LAUNCH();
}

void relu_f32(const float* x, float* y, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  relu_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, y, n);
  QC_CUDA_CHECK_LAUNCH();
}

void clip_f32(const float* x, float* y, int64_t n, float lo, float hi, cudaStream_t s) {
  if (n <= 0) return;
  clip_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, y, n, lo, hi);
  QC_CUDA_CHECK_LAUNCH();
}

void maxpool_f32(const float* x, float* y, int N, int C, int H, int W, int OH, int OW, int kh,
                 int kw, int sh, int sw, int ph, int pw, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(N) * C * OH * OW;
  if (total <= 0) return;
  maxpool_kernel<<<grid_for(total, 256), 256, 0, s>>>(x, y, N, C, H, W, OH, OW, kh, kw, sh, sw,
                                                      ph, pw);
  QC_CUDA_CHECK_LAUNCH();
}

void avgpool_f32(const float* x, float* y, int N, int C, int H, int W, int OH, int OW, int kh,
                 int kw, int sh, int sw, int ph, int pw, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(N) * C * OH * OW;
  if (total <= 0) return;
  const double wk = static_cast<double>(static_cast<float>(1.0 / (static_cast<double>(kh) * kw)));
  avgpool_kernel<<<grid_for(total, 256), 256, 0, s>>>(x, y, N, C, H, W, OH, OW, kh, kw, sh, sw,
                                                      ph, pw, wk);
  QC_CUDA_CHECK_LAUNCH();
}

void concat_words(const void* x, void* y, int N, int64_t inner, int64_t outer, int64_t off,
                  cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(N) * inner;
  if (total <= 0) return;
  const bool v4 = inner % 4 == 0 && outer % 4 == 0 && off % 4 == 0 &&
                  reinterpret_cast<uintptr_t>(x) % 16 == 0 && reinterpret_cast<uintptr_t>(y) % 16 == 0;
  if (v4) {
    concat_v4_kernel<<<grid_for(total / 4, 256), 256, 0, s>>>(
        static_cast<const uint4*>(x), static_cast<uint4*>(y), N, inner / 4, outer / 4, off / 4);
  } else {
    concat_kernel<<<grid_for(total, 256), 256, 0, s>>>(static_cast<const uint32_t*>(x),
                                                       static_cast<uint32_t*>(y), N, inner, outer, off);
  }
  QC_CUDA_CHECK_LAUNCH();
}

void gap_f32(const float* x, float* y, int NC, int HW, cudaStream_t s) {
  if (NC <= 0) return;
  gap_kernel<<<(NC * 32 + 255) / 256, 256, 0, s>>>(x, y, NC, HW);
  QC_CUDA_CHECK_LAUNCH();
}

void argmax_rows(const float* x, int rows, int64_t cols, int64_t* out, cudaStream_t s) {
  if (rows <= 0) return;
  launch_pdl(argmax_kernel, dim3(rows), dim3(256), 0, s, x, cols, out);
  QC_CUDA_CHECK_LAUNCH();
}

void argmax_rows_multi(const float* const* xs, int64_t* const* outs, int groups, int rows,
                       int64_t cols, cudaStream_t s) {
  if (rows <= 0 || groups <= 0 || groups > 4) return;
  RowsPack p{};
  for (int g = 0; g < groups; ++g) {
    p.x[g] = xs[g];
    p.out[g] = outs[g];
  }
  launch_pdl(argmax_multi_kernel, dim3(rows, groups), dim3(256), 0, s, p, cols);
  QC_CUDA_CHECK_LAUNCH();
}

void count_equal_multi(const int64_t* a, const int64_t* b, int n, int groups,
                       unsigned long long* counts, cudaStream_t s) {
  if (n <= 0 || groups <= 0) return;
  launch_pdl(count_equal_multi_kernel, dim3(grid_for(n, 256, 64), groups), dim3(256), 0, s, a, b,
             n, counts);
  QC_CUDA_CHECK_LAUNCH();
}

void count_equal(const int64_t* a, const int64_t* b, int n, unsigned long long* count,
                 cudaStream_t s) {
  if (n <= 0) return;
  launch_pdl(count_equal_kernel, dim3(grid_for(n, 256, 64)), dim3(256), 0, s, a, b, n, count);
  QC_CUDA_CHECK_LAUNCH();
}

}  // namespace quantc::kern
