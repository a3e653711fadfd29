// simquant.cu — the simulated_quantize operator (reference simulate.cpp:64-87).
//
// Streaming kernel: 8 B/element of HBM traffic (fp32 in + fp32 out), 128-bit
// vector loads/stores, grid sized as a multiple of the 148 SMs, grid-stride.
// Math is IEEE-double exactly as the reference (see sq_value in common.cuh).
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "common.cuh"
#include "quantc/device.hpp"

namespace quantc::kern {

bool pdl_enabled() {
  static const bool on = std::getenv("QUANTC_NO_PDL") == nullptr;
  return on;
}

void check_launch(const char* file, int line) {
  ++quantc::device::counters().kernel_launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    throw std::runtime_error(std::string("CUDA launch failed at ") + file + ":" +
                             std::to_string(line) + ": " + cudaGetErrorString(e));
  }
}

namespace {

__global__ void __launch_bounds__(256) sim_quant_kernel(const float* __restrict__ x,
                                                        float* __restrict__ y, int64_t n,
                                                        SqParams p) {
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const bool aligned = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0;
  if (aligned) {
    const int64_t n4 = n >> 2;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    float4* y4 = reinterpret_cast<float4*>(y);
    for (int64_t i = tid; i < n4; i += stride) {
      float4 v = __ldcs(x4 + i);
      v.x = sq_value(v.x, p);
      v.y = sq_value(v.y, p);
      v.z = sq_value(v.z, p);
      v.w = sq_value(v.w, p);
      __stcs(y4 + i, v);
    }
    for (int64_t i = (n4 << 2) + tid; i < n; i += stride) y[i] = sq_value(x[i], p);
  } else {
    for (int64_t i = tid; i < n; i += stride) y[i] = sq_value(x[i], p);
  }
}

// NCHW float in -> float out (same layout) + int8 codes in NHWC (channel
// padded).  One thread per (n, c, hw) element; code = q - zp.
__global__ void sim_quant_codes_kernel(const float* __restrict__ x, float* __restrict__ y,
                                       int8_t* __restrict__ codes, int N, int C, int HW,
                                       int Cpad, SqParams p) {
  const int64_t total = static_cast<int64_t>(N) * C * HW;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t hw = i % HW;
    const int64_t c = (i / HW) % C;
    const int64_t n = i / (static_cast<int64_t>(HW) * C);
    double v = static_cast<double>(x[i]);
    if (p.has_acc) v = clampd(v, p.lo, p.hi);
    const double q = sq_code(v, p);
    const double code = __dsub_rn(q, p.zp);
    if (y) y[i] = __double2float_rn(__dmul_rn(code, p.s));
    codes[(n * HW + hw) * Cpad + c] = static_cast<int8_t>(static_cast<int>(code));
  }
}

__global__ void zero_pad_channels_kernel(int8_t* codes, int64_t pixels, int C, int Cpad) {
  const int64_t total = pixels * (Cpad - C);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t px = i / (Cpad - C);
    const int64_t c = C + i % (Cpad - C);
    codes[px * Cpad + c] = 0;
  }
}

}  // namespace

void sim_quant(const float* x, float* y, int64_t n, const SqParams& p, cudaStream_t s) {
  if (n <= 0) return;
  const int block = 256;
  const int grid = grid_for((n + 3) / 4, block, 148 * 8);
  sim_quant_kernel<<<grid, block, 0, s>>>(x, y, n, p);
  QC_CUDA_CHECK_LAUNCH();
}

void sim_quant_codes_nhwc(const float* x, float* y, int8_t* codes, int N, int C, int H, int W,
                          int Cpad, const SqParams& p, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(N) * C * H * W;
  if (total <= 0) return;
  if (Cpad > C) {
    zero_pad_channels_kernel<<<grid_for(static_cast<int64_t>(N) * H * W * (Cpad - C), 256), 256,
                               0, s>>>(codes, static_cast<int64_t>(N) * H * W, C, Cpad);
    QC_CUDA_CHECK_LAUNCH();
  }
  sim_quant_codes_kernel<<<grid_for(total, 256), 256, 0, s>>>(x, y, codes, N, C, H * W, Cpad, p);
  QC_CUDA_CHECK_LAUNCH();
}

}  // namespace quantc::kern
