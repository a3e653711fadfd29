// conv_simt.cu — the CUDA-core integer conv/dense backend (BASELINE north
// star (2): "the int16-accumulation backend variant on CUDA cores with
// warp-level primitives ... followed by a fused requantize").
//
// Serves the realized-graph cases the tcgen05 kernel does not: int16 codes
// (the arm_vmlal_like (i16, i16) -> i32 signature) and the int16-accumulator
// backend ((i8, i8) -> i16).  Semantics are the reference's
// (interpreter.cpp:238-309): exact sum_k (d - zp0)(w - zp1) + bias, ONE clamp
// (or trap) to the accumulator dtype, then the optional fused requantize
// (:464-482) — int_epi_value (fused.cuh), shared with the tcgen05 epilogue.
//
// Layout: data NHWC 32-bit words (4 int8 or 2 int16 channels per word) with
// the spatial border materialised as zp0, so the inner loop has no bounds
// checks and the correction acc - zp0 * sum_k w' is exact (a padded tap
// contributes (zp0 - zp0) * w' = 0, the reference's skipped tap).  Weights
// (w - zp1) as words k-major: [taps * Cw][O].
//
// Tiling: 64 pixels x 64 output channels per 256-thread CTA, K staged through
// shared memory 16 words at a time (double-buffered via registers); each
// thread owns a 4 x 4 output block.  int8: __dp4a into int32 (exact: the
// host bounds K * 255 * 128 < 2^31).  int16: two 16x16 -> 32-bit products
// per word summed in int64.  Warp-level: the 16 k-words' A fragments are
// read as 128-bit broadcasts shared by the 16 lanes of a half-warp, and the
// dense (M small) case splits K across the warp and reduces with
// __shfl_xor_sync.
#include "common.cuh"
#include "fused.cuh"
#include "kernels.h"

namespace quantc::kern {

namespace {

constexpr int kBM = 64, kBN = 64, kBK = 16, kThreads = 256;

struct SimtArgs {
  const uint32_t* x;  // [N][HP][WP][Cw] words
  const uint32_t* w;  // [K][O] words, K = taps * Cw
  int N, HP, WP, Cw, O, KH, KW, sh, sw, OH, OW;
  int64_t M;  // N * OH * OW
  int K;
  IntEpi ie;
};

template <bool I16>
struct Acc {
  using T = typename std::conditional<I16, long long, int>::type;
};

template <bool I16, bool U8>
__device__ __forceinline__ void mac_t(typename Acc<I16>::T& acc, uint32_t a, uint32_t b) {
  if constexpr (I16) {
    const int lo = static_cast<int>(static_cast<int16_t>(a & 0xFFFFu)) *
                   static_cast<int>(static_cast<int16_t>(b & 0xFFFFu));
    const int hi = static_cast<int>(static_cast<int16_t>(a >> 16)) *
                   static_cast<int>(static_cast<int16_t>(b >> 16));
    acc += static_cast<long long>(lo) + hi;
  } else if constexpr (U8) {
    // uint8 data codes x int8 weights: dp4a's u8 x s8 form
    asm("dp4a.u32.s32 %0, %1, %2, %0;" : "+r"(acc) : "r"(a), "r"(b));
  } else {
    asm("dp4a.s32.s32 %0, %1, %2, %0;" : "+r"(acc) : "r"(a), "r"(b));
  }
}

template <bool I16, bool U8>
__global__ void __launch_bounds__(kThreads) conv_simt_kernel(SimtArgs a) {
  pdl_trigger();
  pdl_wait();
  using T = typename Acc<I16>::T;
  // A rows padded by one word: the staging stores (16 k-words x 2 pixels
  // per warp) then hit distinct banks
  __shared__ uint32_t As[kBK][kBM + 1];
  __shared__ __align__(16) uint32_t Bs[kBK][kBN];
  __shared__ int64_t rowbase[kBM];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;  // tx: 4 output channels, ty: 4 pixels
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * kBM;
  const int o0 = blockIdx.y * kBN;
  if (tid < kBM) {
    const int64_t m = m0 + tid;
    int64_t base = -1;
    if (m < a.M) {
      const int64_t ohw = static_cast<int64_t>(a.OH) * a.OW;
      const int64_t n = m / ohw;
      const int r = static_cast<int>(m - n * ohw);
      const int oh = r / a.OW, ow = r - oh * a.OW;
      base = ((n * a.HP + static_cast<int64_t>(oh) * a.sh) * a.WP + static_cast<int64_t>(ow) * a.sw) *
             a.Cw;
    }
    rowbase[tid] = base;
  }
  __syncthreads();
  T acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0;

  // each thread stages 4 A words and 4 B words per K block
  // A: word (kk = tid & 15, pixel = (tid >> 4) + 16 * q)
  // B: word (kk = tid >> 4, o = (tid & 15) * 4 + q)
  const int a_kk = tid & 15;
  const int b_kk = tid >> 4;
  uint32_t ra[4], rb[4];
  auto load = [&](int kb) {
    const int k = kb + a_kk;
    int off = 0;
    bool kok = k < a.K;
    if (kok) {
      const int tap = k / a.Cw, cw = k - tap * a.Cw;
      const int kh = tap / a.KW, kw = tap - kh * a.KW;
      off = (kh * a.WP + kw) * a.Cw + cw;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t base = rowbase[(tid >> 4) + 16 * q];
      ra[q] = (kok && base >= 0) ? __ldg(a.x + base + off) : 0u;
    }
    const int kbk = kb + b_kk;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int o = o0 + tx * 4 + q;
      rb[q] = (kbk < a.K && o < a.O) ? __ldg(a.w + static_cast<int64_t>(kbk) * a.O + o) : 0u;
    }
  };
  auto store = [&]() {
#pragma unroll
    for (int q = 0; q < 4; ++q) As[a_kk][(tid >> 4) + 16 * q] = ra[q];
    *reinterpret_cast<uint4*>(&Bs[b_kk][tx * 4]) = make_uint4(rb[0], rb[1], rb[2], rb[3]);
  };
  load(0);
  for (int kb = 0; kb < a.K; kb += kBK) {
    store();
    __syncthreads();
    if (kb + kBK < a.K) load(kb + kBK);  // next block's loads overlap this block's math
#pragma unroll
    for (int kk = 0; kk < kBK; ++kk) {
      // pixels ty, ty+16, ty+32, ty+48 (matches the A staging stride)
      uint32_t av[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty + 16 * i];
      const uint4 bv = *reinterpret_cast<const uint4*>(&Bs[kk][tx * 4]);
      const uint32_t bw[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) mac_t<I16, U8>(acc[i][j], av[i], bw[j]);
    }
    __syncthreads();
  }
  // fused epilogue: NCHW int32 stores, lanes of a half-warp write 4
  // consecutive channels of the same pixel row group
  const IntEpi& ie = a.ie;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty + 16 * i;
    if (m >= a.M) continue;
    const int64_t img = m / ie.OHW, hw = m - img * ie.OHW;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int o = o0 + tx * 4 + j;
      if (o >= a.O) continue;
      const int64_t flat = (img * a.O + o) * ie.OHW + hw;
      ie.y[flat] = int_epi_value(ie, static_cast<int64_t>(acc[i][j]), o, flat);
    }
  }
}

// dense with few rows (M <= 16): one warp per (row, output channel), K split
// across the lanes and reduced with __shfl_xor_sync
template <bool I16, bool U8>
__global__ void dense_simt_warp_kernel(const uint32_t* __restrict__ x,
                                       const uint32_t* __restrict__ w, int M, int K, int O,
                                       IntEpi ie) {
  pdl_trigger();
  pdl_wait();
  using T = typename Acc<I16>::T;
  const int lane = threadIdx.x & 31;
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (wid >= static_cast<int64_t>(M) * O) return;
  const int m = static_cast<int>(wid / O), o = static_cast<int>(wid - static_cast<int64_t>(m) * O);
  T acc = 0;
  for (int k = lane; k < K; k += 32) {
    mac_t<I16, U8>(acc, __ldg(x + static_cast<int64_t>(m) * K + k),
                   __ldg(w + static_cast<int64_t>(k) * O + o));
  }
  long long s = static_cast<long long>(acc);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, d);
  if (lane == 0) {
    const int64_t flat = static_cast<int64_t>(m) * O + o;
    ie.y[flat] = int_epi_value(ie, s, o, flat);
  }
}

// int32 NCHW values -> NHWC words, border = fill (zp0), channel pad 0
template <bool I16>
__global__ void pack_words_kernel(const int32_t* __restrict__ x, uint32_t* __restrict__ out,
                                  int64_t pixels, int C, int H, int W, int ph, int pw, int Cw,
                                  int32_t fill) {
  pdl_trigger();
  pdl_wait();
  constexpr int PER = I16 ? 2 : 4;
  constexpr uint32_t MASK = I16 ? 0xFFFFu : 0xFFu;
  const int HP = H + 2 * ph, WP = W + 2 * pw;
  const int64_t total = pixels * Cw;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t pix = i % pixels;
    const int cw = static_cast<int>(i / pixels);
    const int64_t n = pix / (static_cast<int64_t>(HP) * WP);
    const int r = static_cast<int>(pix - n * HP * WP);
    const int h = r / WP - ph, w = r % WP - pw;
    const bool border = h < 0 || h >= H || w < 0 || w >= W;
    uint32_t v = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int c = cw * PER + j;
      if (c >= C) continue;
      const int32_t e = border ? fill : x[(n * C + c) * static_cast<int64_t>(H) * W +
                                          static_cast<int64_t>(h) * W + w];
      v |= (static_cast<uint32_t>(e) & MASK) << (j * (32 / PER));
    }
    out[pix * Cw + cw] = v;
  }
}

// OIHW int32 weights -> words [taps * Cw][O] of w - zp1, wsum[o] = sum w'
template <bool I16>
__global__ void pack_weight_words_kernel(const int32_t* __restrict__ w, uint32_t* __restrict__ out,
                                         int32_t* __restrict__ wsum, int* __restrict__ bad, int O,
                                         int C, int taps, int Cw, int64_t zp1) {
  pdl_trigger();
  pdl_wait();
  constexpr int PER = I16 ? 2 : 4;
  constexpr uint32_t MASK = I16 ? 0xFFFFu : 0xFFu;
  constexpr int64_t LO = I16 ? -32768 : -128, HI = I16 ? 32767 : 127;
  const int64_t total = static_cast<int64_t>(taps) * Cw * O;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int o = static_cast<int>(i % O);
    const int k = static_cast<int>(i / O);
    const int tap = k / Cw, cw = k - tap * Cw;
    uint32_t v = 0;
    int32_t s = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int c = cw * PER + j;
      if (c >= C) continue;
      const int64_t e = static_cast<int64_t>(w[(static_cast<int64_t>(o) * C + c) * taps + tap]) - zp1;
      if (e < LO || e > HI) atomicOr(bad, 1);
      v |= (static_cast<uint32_t>(e) & MASK) << (j * (32 / PER));
      s += static_cast<int32_t>(e);
    }
    out[i] = v;
    if (s != 0) atomicAdd(wsum + o, s);
  }
}

}  // namespace

void pack_words(const int32_t* x, uint32_t* out, int N, int C, int H, int W, int ph, int pw,
                int Cw, bool i16, int32_t fill, cudaStream_t s) {
  const int64_t pixels = static_cast<int64_t>(N) * (H + 2 * ph) * (W + 2 * pw);
  const int64_t total = pixels * Cw;
  if (total <= 0) return;
  if (i16) {
    launch_pdl(pack_words_kernel<true>, dim3(grid_for(total, 256)), dim3(256), 0, s, x, out,
               pixels, C, H, W, ph, pw, Cw, fill);
  } else {
    launch_pdl(pack_words_kernel<false>, dim3(grid_for(total, 256)), dim3(256), 0, s, x, out,
               pixels, C, H, W, ph, pw, Cw, fill);
  }
  QC_CUDA_CHECK_LAUNCH();
}

void pack_weight_words(const int32_t* w, uint32_t* out, int32_t* wsum, int* bad, int O, int C,
                       int taps, int Cw, bool i16, int64_t zp1, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(taps) * Cw * O;
  if (total <= 0) return;
  if (i16) {
    launch_pdl(pack_weight_words_kernel<true>, dim3(grid_for(total, 256)), dim3(256), 0, s, w,
               out, wsum, bad, O, C, taps, Cw, zp1);
  } else {
    launch_pdl(pack_weight_words_kernel<false>, dim3(grid_for(total, 256)), dim3(256), 0, s, w,
               out, wsum, bad, O, C, taps, Cw, zp1);
  }
  QC_CUDA_CHECK_LAUNCH();
}

void conv_int_simt(const SimtConvSpec& sp, cudaStream_t s) {
  SimtArgs a{};
  a.x = sp.x;
  a.w = sp.w;
  a.N = sp.N;
  a.HP = sp.HP;
  a.WP = sp.WP;
  a.Cw = sp.Cw;
  a.O = sp.O;
  a.KH = sp.KH;
  a.KW = sp.KW;
  a.sh = sp.sh;
  a.sw = sp.sw;
  a.OH = sp.OH;
  a.OW = sp.OW;
  a.M = static_cast<int64_t>(sp.N) * sp.OH * sp.OW;
  a.K = sp.KH * sp.KW * sp.Cw;
  a.ie = sp.ie;
  if (a.M <= 0 || a.O <= 0) return;
  const bool dense_warp = sp.KH == 1 && sp.KW == 1 && sp.OH == 1 && sp.OW == 1 &&
                          sp.HP == 1 && sp.WP == 1 && a.M <= 16;
  if (dense_warp) {
    const int64_t threads = a.M * a.O * 32;
    const dim3 grid(static_cast<unsigned>((threads + 255) / 256));
#define QC_DW(I16, U8)                                                                         \
  launch_pdl(dense_simt_warp_kernel<I16, U8>, grid, dim3(256), 0, s, a.x, a.w,              \
             static_cast<int>(a.M), a.K, a.O, a.ie)
    if (sp.i16) QC_DW(true, false);
    else if (sp.u8) QC_DW(false, true);
    else QC_DW(false, false);
#undef QC_DW
  } else {
    const dim3 grid(static_cast<unsigned>((a.M + kBM - 1) / kBM),
                    static_cast<unsigned>((a.O + kBN - 1) / kBN));
    if (sp.i16) launch_pdl(conv_simt_kernel<true, false>, grid, dim3(kThreads), 0, s, a);
    else if (sp.u8) launch_pdl(conv_simt_kernel<false, true>, grid, dim3(kThreads), 0, s, a);
    else launch_pdl(conv_simt_kernel<false, false>, grid, dim3(kThreads), 0, s, a);
  }
  QC_CUDA_CHECK_LAUNCH();
}

}  // namespace quantc::kern
