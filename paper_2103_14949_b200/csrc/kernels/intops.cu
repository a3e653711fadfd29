// intops.cu — integer-regime kernels for realized graphs (reference
// interpreter.cpp:25-37, 238-264, 293-309, 326-336, 432-482).
//
// Storage is int32 like the reference Tensor.  Accumulation is exact int64
// (order-free), then ONE clamp to the accumulator dtype (saturate) or a trap:
// overflowing elements atomicMin their flat (n,o,oh,ow) index so the host can
// raise OverflowError for the lowest one, exactly the element the reference's
// sequential loop would throw at.
#include <climits>

#include "common.cuh"

namespace quantc::kern {

namespace {

__device__ __forceinline__ int32_t clamp_acc(int64_t v, int64_t lo, int64_t hi, int64_t flat,
                                             unsigned long long* trap) {
  if (v < lo || v > hi) {
    if (trap) atomicMin(trap, static_cast<unsigned long long>(flat));
    v = v < lo ? lo : hi;
  }
  return static_cast<int32_t>(v);
}

__device__ int64_t conv_acc(const int32_t* __restrict__ x, const int32_t* __restrict__ w,
                            const int32_t* __restrict__ bias, const ConvShape& cs, int64_t zp0,
                            int64_t zp1, int64_t flat) {
  const int ow = static_cast<int>(flat % cs.OW);
  const int oh = static_cast<int>((flat / cs.OW) % cs.OH);
  const int o = static_cast<int>((flat / (static_cast<int64_t>(cs.OW) * cs.OH)) % cs.O);
  const int64_t n = flat / (static_cast<int64_t>(cs.OW) * cs.OH * cs.O);
  // grouped convs (op-set extension): output channel o reads the C/G input
  // channels of its group; the weight is [O][C/G][KH][KW]
  const int Cg = cs.C / conv_groups(cs);
  const int cbase = (o / (cs.O / conv_groups(cs))) * Cg;
  int64_t acc = 0;
  for (int c = 0; c < Cg; ++c) {
    for (int kh = 0; kh < cs.KH; ++kh) {
      const int ih = oh * cs.sh - cs.ph + kh;
      if (ih < 0 || ih >= cs.H) continue;
      for (int kw = 0; kw < cs.KW; ++kw) {
        const int iw = ow * cs.sw - cs.pw + kw;
        if (iw < 0 || iw >= cs.W) continue;
        const int64_t dv = x[((n * cs.C + cbase + c) * cs.H + ih) * cs.W + iw] - zp0;
        const int64_t wv = w[((static_cast<int64_t>(o) * Cg + c) * cs.KH + kh) * cs.KW + kw] - zp1;
        acc += dv * wv;
      }
    }
  }
  if (bias) acc += bias[o];
  return acc;
}

__global__ void conv_int_kernel(const int32_t* __restrict__ x, const int32_t* __restrict__ w,
                                const int32_t* __restrict__ bias, int32_t* __restrict__ y,
                                ConvShape cs, int64_t zp0, int64_t zp1, int64_t lo, int64_t hi,
                                unsigned long long* trap) {
  const int64_t total = static_cast<int64_t>(cs.N) * cs.O * cs.OH * cs.OW;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    y[i] = clamp_acc(conv_acc(x, w, bias, cs, zp0, zp1, i), lo, hi, i, trap);
  }
}

__global__ void conv_int_value_kernel(const int32_t* x, const int32_t* w, const int32_t* bias,
                                      ConvShape cs, int64_t zp0, int64_t zp1, int64_t flat,
                                      long long* out) {
  *out = conv_acc(x, w, bias, cs, zp0, zp1, flat);
}

__global__ void add_int_kernel(const int32_t* a, int64_t na, const int32_t* b, int64_t nb,
                               int32_t* y, int64_t n, int64_t lo, int64_t hi,
                               unsigned long long* trap) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t v = static_cast<int64_t>(a[na == n ? i : i % na]) + b[nb == n ? i : i % nb];
    y[i] = clamp_acc(v, lo, hi, i, trap);
  }
}

__global__ void relu_int_kernel(const int32_t* x, int32_t* y, int64_t n, int32_t zp) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    y[i] = max(x[i], zp);
  }
}

__global__ void clip_int_kernel(const int32_t* x, int32_t* y, int64_t n, int32_t lo, int32_t hi) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t v = x[i];
    y[i] = v < lo ? lo : (hi < v ? hi : v);
  }
}

__global__ void maxpool_int_kernel(const int32_t* x, int32_t* y, int N, int C, int H, int W,
                                   int OH, int OW, int kh, int kw, int sh, int sw, int ph,
                                   int pw) {
  const int64_t total = static_cast<int64_t>(N) * C * OH * OW;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int ow = static_cast<int>(i % OW);
    const int oh = static_cast<int>((i / OW) % OH);
    const int64_t nc = i / (static_cast<int64_t>(OW) * OH);
    int32_t best = INT_MIN;
    for (int a = 0; a < kh; ++a) {
      const int ih = oh * sh - ph + a;
      if (ih < 0 || ih >= H) continue;
      for (int b = 0; b < kw; ++b) {
        const int iw = ow * sw - pw + b;
        if (iw < 0 || iw >= W) continue;
        best = max(best, x[(nc * H + ih) * W + iw]);
      }
    }
    y[i] = best;
  }
}

// llround(x / scale) + zp, clamped (reference interpreter.cpp:443-446)
__global__ void quantize_kernel(const float* x, int32_t* y, int64_t n, double scale, int64_t zp,
                                int64_t qmin, int64_t qmax) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const long long q = llround(__ddiv_rn(static_cast<double>(x[i]), scale)) + zp;
    y[i] = static_cast<int32_t>(q < qmin ? qmin : (q > qmax ? qmax : q));
  }
}

__global__ void dequantize_kernel(const int32_t* x, float* y, int64_t n, double scale,
                                  int64_t zp) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    // static_cast<double>(xx[i] - zp) * scale   (int32 - int64 -> int64)
    y[i] = __double2float_rn(__dmul_rn(static_cast<double>(x[i] - zp), scale));
  }
}

// fixed_point_rescale (reference interpreter.cpp:32-37), round half away
__device__ __forceinline__ int64_t fp_rescale(int64_t v, int64_t mult, int shift) {
  const int64_t p = v * mult;
  if (shift == 0) return p;
  const int64_t nudge = int64_t{1} << (shift - 1);
  return p >= 0 ? (p + nudge) >> shift : -((-p + nudge) >> shift);
}

__global__ void requantize_kernel(const int32_t* x, int32_t* y, int64_t n, int64_t mult,
                                  int shift, int64_t in_zp, int64_t out_zp, int64_t qmin,
                                  int64_t qmax) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t q = fp_rescale(static_cast<int64_t>(x[i]) - in_zp, mult, shift) + out_zp;
    y[i] = static_cast<int32_t>(q < qmin ? qmin : (q > qmax ? qmax : q));
  }
}

}  // namespace

void conv2d_int(const int32_t* x, const int32_t* w, const int32_t* bias, int32_t* y,
                const ConvShape& cs, int64_t zp0, int64_t zp1, int64_t acc_min, int64_t acc_max,
                unsigned long long* trap_flat, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(cs.N) * cs.O * cs.OH * cs.OW;
  if (total <= 0) return;
  conv_int_kernel<<<grid_for(total, 128), 128, 0, s>>>(x, w, bias, y, cs, zp0, zp1, acc_min,
                                                       acc_max, trap_flat);
  QC_CUDA_CHECK_LAUNCH();
}

int64_t conv2d_int_value_at(const int32_t* x, const int32_t* w, const int32_t* bias,
                            const ConvShape& cs, int64_t zp0, int64_t zp1, int64_t flat,
                            cudaStream_t s) {
  long long* d = nullptr;
  cudaMallocAsync(&d, sizeof(long long), s);
  conv_int_value_kernel<<<1, 1, 0, s>>>(x, w, bias, cs, zp0, zp1, flat, d);
  QC_CUDA_CHECK_LAUNCH();
  long long h = 0;
  cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(d, s);
  cudaStreamSynchronize(s);
  return h;
}

void add_int(const int32_t* a, int64_t na, const int32_t* b, int64_t nb, int32_t* y, int64_t n,
             int64_t acc_min, int64_t acc_max, unsigned long long* trap_flat, cudaStream_t s) {
  if (n <= 0) return;
  add_int_kernel<<<grid_for(n, 256), 256, 0, s>>>(a, na, b, nb, y, n, acc_min, acc_max,
                                                   trap_flat);
  QC_CUDA_CHECK_LAUNCH();
}

void relu_int(const int32_t* x, int32_t* y, int64_t n, int32_t zp, cudaStream_t s) {
  if (n <= 0) return;
  relu_int_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, y, n, zp);
  QC_CUDA_CHECK_LAUNCH();
}

void clip_int(const int32_t* x, int32_t* y, int64_t n, int32_t lo, int32_t hi, cudaStream_t s) {
  if (n <= 0) return;
  clip_int_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, y, n, lo, hi);
  QC_CUDA_CHECK_LAUNCH();
}

void maxpool_int(const int32_t* x, int32_t* y, int N, int C, int H, int W, int OH, int OW,
                 int kh, int kw, int sh, int sw, int ph, int pw, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(N) * C * OH * OW;
  if (total <= 0) return;
  maxpool_int_kernel<<<grid_for(total, 256), 256, 0, s>>>(x, y, N, C, H, W, OH, OW, kh, kw, sh,
                                                          sw, ph, pw);
  QC_CUDA_CHECK_LAUNCH();
}

void quantize_f32_int(const float* x, int32_t* y, int64_t n, double scale, int64_t zp,
                      int64_t qmin, int64_t qmax, cudaStream_t s) {
  if (n <= 0) return;
  quantize_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, y, n, scale, zp, qmin, qmax);
  QC_CUDA_CHECK_LAUNCH();
}

void dequantize_int_f32(const int32_t* x, float* y, int64_t n, double scale, int64_t zp,
                        cudaStream_t s) {
  if (n <= 0) return;
  dequantize_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, y, n, scale, zp);
  QC_CUDA_CHECK_LAUNCH();
}

void requantize_int(const int32_t* x, int32_t* y, int64_t n, int64_t mult, int shift,
                    int64_t in_zp, int64_t out_zp, int64_t qmin, int64_t qmax, cudaStream_t s) {
  if (n <= 0) return;
  requantize_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, y, n, mult, shift, in_zp, out_zp, qmin,
                                                     qmax);
  QC_CUDA_CHECK_LAUNCH();
}

}  // namespace quantc::kern
