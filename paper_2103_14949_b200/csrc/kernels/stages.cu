// stages.cu — non-GEMM stages of the fused int8 dataflow (engine v2):
// graph-input quantisation, max-pool on codes, global average pool, weight
// codes.  Each evaluates the stage's epilogue program on its output.
//
// Semantics: max_pool2d on codes == max_pool2d on values because the value
// map code -> code*s (s > 0) is monotone (reference interpreter.cpp:377-397,
// padded taps skipped); GAP is the reference's sequential double sum over
// h*W+w then / (H*W) (interpreter.cpp:412-417).
#include <cfloat>

#include "fused.cuh"

namespace quantc::kern {

namespace {

// one thread per (m, 16-channel group); reads NCHW (strided by HW)
__global__ void input_kernel(const float* __restrict__ x, int N, int C, int HW, ProgArgs prog) {
  pdl_trigger();
  pdl_wait();
  __shared__ StageTables T;
  load_tables(&T, prog.tables);
  __syncthreads();
  const int groups = (C + 15) / 16;
  const int64_t total = static_cast<int64_t>(N) * HW * groups;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int grp = static_cast<int>(i % groups);
    const int64_t m = i / groups;
    const int64_t n = m / HW, hw = m % HW;
    const int c0 = grp * 16;
    const int nvalid = C - c0 < 16 ? C - c0 : 16;
    float v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      v[j] = j < nvalid ? x[(n * C + c0 + j) * HW + hw] : 0.0f;
    }
    run_prog<16, 3>(v, m, c0, nvalid, T);
  }
}

template <int DEPTH>
__global__ void __launch_bounds__(256) maxpool_codes_kernel(const int8_t* __restrict__ x, int ld, float scale, int N,
                                     int C, int H, int W, int OH, int OW, int kh, int kw, int sh,
                                     int sw, int ph, int pw, ProgArgs prog) {
  pdl_trigger();
  pdl_wait();
  __shared__ StageTables T;
  load_tables(&T, prog.tables);
  __syncthreads();
  const int groups = (C + 15) / 16;
  const int64_t total = static_cast<int64_t>(N) * OH * OW * groups;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int grp = static_cast<int>(i % groups);
    const int64_t m = i / groups;
    const int ow = static_cast<int>(m % OW);
    const int oh = static_cast<int>((m / OW) % OH);
    const int64_t n = m / (static_cast<int64_t>(OW) * OH);
    const int c0 = grp * 16;
    const int nvalid = C - c0 < 16 ? C - c0 : 16;
    int best[16];
    bool any = false;
#pragma unroll
    for (int j = 0; j < 16; ++j) best[j] = -129;
    for (int a = 0; a < kh; ++a) {
      const int ih = oh * sh - ph + a;
      if (ih < 0 || ih >= H) continue;
      for (int b = 0; b < kw; ++b) {
        const int iw = ow * sw - pw + b;
        if (iw < 0 || iw >= W) continue;
        any = true;
        const int8_t* src = x + ((n * H + ih) * W + iw) * ld + c0;
        if (nvalid == 16 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
          const int4 raw = *reinterpret_cast<const int4*>(src);
          const int8_t* cc = reinterpret_cast<const int8_t*>(&raw);
#pragma unroll
          for (int j = 0; j < 16; ++j) best[j] = max(best[j], static_cast<int>(cc[j]));
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (j < nvalid) best[j] = max(best[j], static_cast<int>(src[j]));
          }
        }
      }
    }
    float v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      v[j] = any ? __fmul_rn(static_cast<float>(best[j]), scale) : -FLT_MAX;
    }
    run_prog<16, DEPTH>(v, m, c0, nvalid, T);
  }
}

// average pool of fp32 NHWC rows -> the stage program.  The op is DEFINED
// as the constant depthwise conv with weight wk = fl32(1/(kh*kw)) and zero
// padding (fixtures.py _avg_pool); the reference's double accumulation
// (x*wk exact in double, one rounding per tap) in (kh, kw) order, as the
// exact engine's avgpool_kernel (eltwise.cu), then one rounding to float.
template <bool FAST>
__global__ void __launch_bounds__(256) avgpool_f32_kernel(const float* __restrict__ x, int ld, int N, int C, int H, int W,
                                   int OH, int OW, int kh, int kw, int sh, int sw, int ph, int pw,
                                   double wk, ProgArgs prog, DwFast fast) {
  pdl_trigger();
  pdl_wait();
  __shared__ StageTables T;
  if constexpr (!FAST) {
    load_tables(&T, prog.tables);
    __syncthreads();
  }
  const bool vec = (ld & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  const int groups = (C + 15) / 16;
  const int64_t total = static_cast<int64_t>(N) * OH * OW * groups;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int grp = static_cast<int>(i % groups);
    const int64_t m = i / groups;
    const int ow = static_cast<int>(m % OW);
    const int oh = static_cast<int>((m / OW) % OH);
    const int64_t n = m / (static_cast<int64_t>(OW) * OH);
    const int c0 = grp * 16;
    const int nvalid = C - c0 < 16 ? C - c0 : 16;
    double acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0.0;
    for (int a = 0; a < kh; ++a) {
      const int ih = oh * sh - ph + a;
      if (ih < 0 || ih >= H) continue;
      for (int b = 0; b < kw; ++b) {
        const int iw = ow * sw - pw + b;
        if (iw < 0 || iw >= W) continue;
        const float* src = x + ((n * H + ih) * W + iw) * ld + c0;
        if (vec && nvalid == 16) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 f = __ldg(reinterpret_cast<const float4*>(src) + q);
            acc[4 * q + 0] = __fma_rn(static_cast<double>(f.x), wk, acc[4 * q + 0]);
            acc[4 * q + 1] = __fma_rn(static_cast<double>(f.y), wk, acc[4 * q + 1]);
            acc[4 * q + 2] = __fma_rn(static_cast<double>(f.z), wk, acc[4 * q + 2]);
            acc[4 * q + 3] = __fma_rn(static_cast<double>(f.w), wk, acc[4 * q + 3]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (j < nvalid) acc[j] = __fma_rn(static_cast<double>(__ldg(src + j)), wk, acc[j]);
          }
        }
      }
    }
    float v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __double2float_rn(acc[j]);
    if constexpr (FAST) {
      if (fast.n == 2) sq_values<16>(v, fast.fa);
      float q[16];
      sq_codes<16>(v, q, fast.fs);
      store_codes<16>(fast.buf, m, c0, nvalid, q, nullptr, 0);
    } else {
      run_prog<16, 3>(v, m, c0, nvalid, T);
    }
  }
}

// depthwise conv (groups == C == O) of int8 codes -> the stage program:
// one thread per (output pixel, 16-channel group), int32 tap sums of
// code x weight-code products, then v = RN24(acc * s_x*s_w + bias) — the
// reference's double accumulation rounded to float, exact for power-of-two
// scales (|acc| <= taps * 128 * 128 < 2^24 keeps acc * s an exact float and
// the double rounding innocuous) — and the consumers' program.  Weights are
// tap quads [ceil(taps/4)][ldw] of packed int8 codes (dw_weight_quads).
// FAST: the inline [accumulator sq,] sq_store8 program only (no table
// interpreter: ~60 instead of ~166 registers, so 4x the resident warps)
template <bool FAST>
__global__ void __launch_bounds__(256) dw_conv_kernel(const int8_t* __restrict__ x, int ld, int N, int C, int H, int W,
                               int KH, int KW, int sh, int sw, int ph, int pw, int OH, int OW,
                               const int32_t* __restrict__ wq, int ldw, const float* __restrict__ bias,
                               float scale, ProgArgs prog, DwFast fast) {
  pdl_trigger();
  pdl_wait();
  __shared__ StageTables T;
  if constexpr (!FAST) {
    load_tables(&T, prog.tables);
    __syncthreads();
  }
  const int groups = (C + 15) / 16;
  const int64_t total = static_cast<int64_t>(N) * OH * OW * groups;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int grp = static_cast<int>(i % groups);
    const int64_t m = i / groups;
    const int ow = static_cast<int>(m % OW);
    const int oh = static_cast<int>((m / OW) % OH);
    const int64_t n = m / (static_cast<int64_t>(OW) * OH);
    const int c0 = grp * 16;
    const int nvalid = C - c0 < 16 ? C - c0 : 16;
    // taps in quads: per 4 channels, the four taps' input words are byte-
    // transposed (8 PRMT) so each channel's 4 taps share one word, then one
    // dp4a per channel against its pre-packed weight quad (wq: [quad][ldw]
    // words, zero past the last tap) — 12 instructions per 16 products
    int acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0;
    const int taps = KH * KW;
    int t = 0, a = 0, b = 0;
    for (int q = 0; t < taps; ++q) {
      uint32_t X[4][4];  // [tap in quad][channel word]
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        int4 xr = make_int4(0, 0, 0, 0);
        if (t < taps) {
          const int ih = oh * sh - ph + a, iw = ow * sw - pw + b;
          if (ih >= 0 && ih < H && iw >= 0 && iw < W) {
            xr = __ldg(reinterpret_cast<const int4*>(x + ((n * H + ih) * W + iw) * ld + c0));
          }
          ++t;
          if (++b == KW) {
            b = 0;
            ++a;
          }
        }
        X[k][0] = static_cast<uint32_t>(xr.x);
        X[k][1] = static_cast<uint32_t>(xr.y);
        X[k][2] = static_cast<uint32_t>(xr.z);
        X[k][3] = static_cast<uint32_t>(xr.w);
      }
      const int4* wp = reinterpret_cast<const int4*>(wq + static_cast<int64_t>(q) * ldw + c0);
#pragma unroll
      for (int g4 = 0; g4 < 4; ++g4) {
        const int4 wr = __ldg(wp + g4);
        const uint32_t t0 = __byte_perm(X[0][g4], X[1][g4], 0x5140);
        const uint32_t t1 = __byte_perm(X[2][g4], X[3][g4], 0x5140);
        const uint32_t t2 = __byte_perm(X[0][g4], X[1][g4], 0x7362);
        const uint32_t t3 = __byte_perm(X[2][g4], X[3][g4], 0x7362);
        acc[4 * g4 + 0] = __dp4a(static_cast<int>(__byte_perm(t0, t1, 0x5410)), wr.x, acc[4 * g4 + 0]);
        acc[4 * g4 + 1] = __dp4a(static_cast<int>(__byte_perm(t0, t1, 0x7632)), wr.y, acc[4 * g4 + 1]);
        acc[4 * g4 + 2] = __dp4a(static_cast<int>(__byte_perm(t2, t3, 0x5410)), wr.z, acc[4 * g4 + 2]);
        acc[4 * g4 + 3] = __dp4a(static_cast<int>(__byte_perm(t2, t3, 0x7632)), wr.w, acc[4 * g4 + 3]);
      }
    }
    float v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float b = (bias && j < nvalid) ? __ldg(bias + c0 + j) : 0.0f;
      v[j] = __fadd_rn(__fmul_rn(static_cast<float>(acc[j]), scale), b);
    }
    if constexpr (FAST) {
      // the program [passthrough accumulator sq,] sq_store8 without the
      // interpreter: the same device functions run_prog calls for them
      if (fast.n == 2) sq_values<16>(v, fast.fa);
      float q[16];
      sq_codes<16>(v, q, fast.fs);
      store_codes<16>(fast.buf, m, c0, nvalid, q, nullptr, 0);
    } else {
      run_prog<16, 3>(v, m, c0, nvalid, T);
    }
  }
}

// one thread per (n, c): sequential double sum in h*W+w order (coalesced
// across c), then the stage program on that one value
__global__ void gap_rows_kernel(const float* __restrict__ x, int64_t ld, int N, int C, int HW,
                                ProgArgs prog) {
  pdl_trigger();
  pdl_wait();
  __shared__ StageTables T;
  load_tables(&T, prog.tables);
  __syncthreads();
  const int64_t total = static_cast<int64_t>(N) * C;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % C);
    const int64_t n = i / C;
    const float* col = x + n * HW * ld + c;
    double acc = 0.0;
    for (int hw = 0; hw < HW; ++hw) acc = __dadd_rn(acc, static_cast<double>(__ldg(col + hw * ld)));
    float v[1] = {__double2float_rn(__ddiv_rn(acc, static_cast<double>(HW)))};
    run_prog<1, 3>(v, n, c, 1, T);
  }
}

// max-pool -> code stores: signed byte max over the window, then each store's
// folded sq (codes are exact floats; no conversion-pipe instructions)
template <int NOUT, bool K3>
__global__ void maxpool_stores_kernel(const int8_t* __restrict__ x, int ld, int N, int C, int H,
                                      int W, int OH, int OW, int kh, int kw, int sh, int sw, int ph,
                                      int pw, PoolStores e) {
  pdl_trigger();
  pdl_wait();
  const int groups = C / 16;
  const int64_t total = static_cast<int64_t>(N) * OH * OW * groups;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    // 32-bit index decomposition when the space fits (64-bit divisions are
    // ~100 instructions each: four of them per item dominated this kernel)
    int grp, ow, oh;
    int64_t m, n;
    if (total <= 0xFFFFFFFFll) {
      const uint32_t ii = static_cast<uint32_t>(i);
      const uint32_t mm = ii / static_cast<uint32_t>(groups);
      grp = static_cast<int>(ii - mm * static_cast<uint32_t>(groups));
      const uint32_t t = mm / static_cast<uint32_t>(OW);
      ow = static_cast<int>(mm - t * static_cast<uint32_t>(OW));
      const uint32_t nn = t / static_cast<uint32_t>(OH);
      oh = static_cast<int>(t - nn * static_cast<uint32_t>(OH));
      m = mm;
      n = nn;
    } else {
      grp = static_cast<int>(i % groups);
      m = i / groups;
      ow = static_cast<int>(m % OW);
      oh = static_cast<int>((m / OW) % OH);
      n = m / (static_cast<int64_t>(OW) * OH);
    }
    uint32_t best[4] = {0x80808080u, 0x80808080u, 0x80808080u, 0x80808080u};
    if constexpr (K3) {
      // 3x3 window: the nine (masked) 16-byte loads are issued together
      int4 raw[9];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const int ih = oh * sh - ph + a;
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          const int iw = ow * sw - pw + b;
          const bool ok = ih >= 0 && ih < H && iw >= 0 && iw < W;
          raw[a * 3 + b] = ok ? __ldg(reinterpret_cast<const int4*>(
                                    x + ((n * H + ih) * W + iw) * ld + grp * 16))
                              : make_int4(static_cast<int>(0x80808080u), static_cast<int>(0x80808080u),
                                          static_cast<int>(0x80808080u), static_cast<int>(0x80808080u));
        }
      }
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        best[0] = __vmaxs4(best[0], static_cast<uint32_t>(raw[k].x));
        best[1] = __vmaxs4(best[1], static_cast<uint32_t>(raw[k].y));
        best[2] = __vmaxs4(best[2], static_cast<uint32_t>(raw[k].z));
        best[3] = __vmaxs4(best[3], static_cast<uint32_t>(raw[k].w));
      }
    } else {
      for (int a = 0; a < kh; ++a) {
        const int ih = oh * sh - ph + a;
        if (ih < 0 || ih >= H) continue;
        for (int b = 0; b < kw; ++b) {
          const int iw = ow * sw - pw + b;
          if (iw < 0 || iw >= W) continue;
          const int4 raw = __ldg(reinterpret_cast<const int4*>(x + ((n * H + ih) * W + iw) * ld + grp * 16));
          best[0] = __vmaxs4(best[0], static_cast<uint32_t>(raw.x));
          best[1] = __vmaxs4(best[1], static_cast<uint32_t>(raw.y));
          best[2] = __vmaxs4(best[2], static_cast<uint32_t>(raw.z));
          best[3] = __vmaxs4(best[3], static_cast<uint32_t>(raw.w));
        }
      }
    }
    float r[16];
    codes_to_floats(best, r);
#pragma unroll
    for (int o = 0; o < NOUT; ++o) {
      float y[16];
      epi_next(r, y, e.q[o]);
      *reinterpret_cast<int4*>(e.out[o] + m * e.ld[o] + grp * 16) = epi_pack(y, e.q[o]);
    }
  }
}

// DEPTH: the program's push depth (prog.depth); a shallow program needs
// fewer stack registers, so more warps stay resident
template <int DEPTH>
__global__ void __launch_bounds__(256) ew_kernel(ProgBuf src, int64_t M, int C, ProgArgs prog) {
  pdl_trigger();
  pdl_wait();
  __shared__ StageTables T;
  load_tables(&T, prog.tables);
  __syncthreads();
  const int groups = (C + 15) / 16;
  const int64_t total = M * groups;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int grp = static_cast<int>(i % groups);
    const int64_t m = i / groups;
    const int c0 = grp * 16;
    const int nvalid = C - c0 < 16 ? C - c0 : 16;
    float v[16];
    load_values<16>(src, m, c0, nvalid, v);
    run_prog<16, DEPTH>(v, m, c0, nvalid, T);
  }
}

__global__ void weight_codes_v2_kernel(const float* __restrict__ w, int8_t* __restrict__ codes,
                                       int O, int C, int taps, int ldk, int Kpad, FSq p) {
  pdl_trigger();
  pdl_wait();
  const int64_t total = static_cast<int64_t>(O) * Kpad;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(i % Kpad);
    const int o = static_cast<int>(i / Kpad);
    const int tap = k / ldk, c = k - (k / ldk) * ldk;
    int8_t code = 0;
    if (tap < taps && c < C) {
      const float v = w[(static_cast<int64_t>(o) * C + c) * taps + tap];
      code = static_cast<int8_t>(static_cast<int>(__fsub_rn(fsq_code(v, p), p.zp)));
    }
    codes[i] = code;
  }
}

// graph input NCHW fp32 -> space-to-depth int8 codes (fastplan Val::s2d): one
// thread per 2x2 pixel block, its 4*C codes (zero-padded to 16) as one store
__global__ void input_s2d_kernel(const float* __restrict__ x, int N, int C, int H, int W, int H2,
                                 int W2, FSq p, int8_t* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int64_t total = static_cast<int64_t>(N) * H2 * W2;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int w2, h2;
    int64_t n;
    if (total <= 0xFFFFFFFFll) {  // 32-bit decomposition (see maxpool_stores_kernel)
      const uint32_t ii = static_cast<uint32_t>(i);
      const uint32_t t = ii / static_cast<uint32_t>(W2);
      w2 = static_cast<int>(ii - t * static_cast<uint32_t>(W2));
      const uint32_t nn = t / static_cast<uint32_t>(H2);
      h2 = static_cast<int>(t - nn * static_cast<uint32_t>(H2));
      n = nn;
    } else {
      w2 = static_cast<int>(i % W2);
      const int64_t t = i / W2;
      h2 = static_cast<int>(t % H2);
      n = t / H2;
    }
    uint32_t word[4] = {0, 0, 0, 0};
    const bool pair = (W & 1) == 0;  // the two pixels of a row are one 8-byte load
    for (int c = 0; c < C; ++c) {
      const float* plane = x + (n * C + c) * H * W;
#pragma unroll
      for (int dy = 0; dy < 2; ++dy) {
        const int h = 2 * h2 + dy;
        if (h >= H) continue;
        float v[2];
        if (pair) {
          const float2 v2 = __ldg(reinterpret_cast<const float2*>(plane + h * W + 2 * w2));
          v[0] = v2.x;
          v[1] = v2.y;
        } else {
          v[0] = plane[h * W + 2 * w2];
          v[1] = 2 * w2 + 1 < W ? plane[h * W + 2 * w2 + 1] : 0.0f;
        }
#pragma unroll
        for (int dx = 0; dx < 2; ++dx) {
          const int w = 2 * w2 + dx;
          if (w < W) {
            const float q = __fsub_rn(fsq_code(v[dx], p), p.zp);
            const int b = (dy * 2 + dx) * C + c;
            word[b >> 2] |= static_cast<uint32_t>(static_cast<uint8_t>(static_cast<int8_t>(
                                __float2int_rn(q))))
                            << (8 * (b & 3));
          }
        }
      }
    }
    *reinterpret_cast<int4*>(out + i * 16) =
        make_int4(static_cast<int>(word[0]), static_cast<int>(word[1]), static_cast<int>(word[2]),
                  static_cast<int>(word[3]));
  }
}
// the same images quantized under up to four bindings (grouped candidate
// evaluation): each pixel is read once and written once per binding
struct S2dMulti {
  FSq p[4];
  int8_t* out[4];
};
__global__ void input_s2d_multi_kernel(const float* __restrict__ x, int N, int C, int H, int W,
                                       int H2, int W2, S2dMulti m, int groups) {
  pdl_trigger();
  pdl_wait();
  const int64_t total = static_cast<int64_t>(N) * H2 * W2;
  const bool pair = (W & 1) == 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int w2, h2;
    int64_t n;
    if (total <= 0xFFFFFFFFll) {  // 32-bit decomposition (see maxpool_stores_kernel)
      const uint32_t ii = static_cast<uint32_t>(i);
      const uint32_t t = ii / static_cast<uint32_t>(W2);
      w2 = static_cast<int>(ii - t * static_cast<uint32_t>(W2));
      const uint32_t nn = t / static_cast<uint32_t>(H2);
      h2 = static_cast<int>(t - nn * static_cast<uint32_t>(H2));
      n = nn;
    } else {
      w2 = static_cast<int>(i % W2);
      const int64_t t = i / W2;
      h2 = static_cast<int>(t % H2);
      n = t / H2;
    }
    float v[4][4] = {};  // [c][dy*2 + dx], C <= 4 (fully unrolled: registers)
    bool ok[4] = {false, false, false, false};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (c >= C) break;
      const float* plane = x + (n * C + c) * H * W;
#pragma unroll
      for (int dy = 0; dy < 2; ++dy) {
        const int h = 2 * h2 + dy;
        ok[dy * 2] = h < H;
        ok[dy * 2 + 1] = h < H && 2 * w2 + 1 < W;
        if (h >= H) continue;
        if (pair) {
          const float2 v2 = __ldg(reinterpret_cast<const float2*>(plane + h * W + 2 * w2));
          v[c][dy * 2] = v2.x;
          v[c][dy * 2 + 1] = v2.y;
        } else {
          v[c][dy * 2] = plane[h * W + 2 * w2];
          v[c][dy * 2 + 1] = 2 * w2 + 1 < W ? plane[h * W + 2 * w2 + 1] : 0.0f;
        }
      }
    }
    for (int g = 0; g < groups; ++g) {
      uint32_t word[4] = {0, 0, 0, 0};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (c >= C) break;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (!ok[k]) continue;
          const float q = __fsub_rn(fsq_code(v[c][k], m.p[g]), m.p[g].zp);
          const int b = k * C + c;
          word[b >> 2] |= static_cast<uint32_t>(static_cast<uint8_t>(static_cast<int8_t>(
                              __float2int_rn(q))))
                          << (8 * (b & 3));
        }
      }
      *reinterpret_cast<int4*>(m.out[g] + i * 16) =
          make_int4(static_cast<int>(word[0]), static_cast<int>(word[1]), static_cast<int>(word[2]),
                    static_cast<int>(word[3]));
    }
  }
}


// weight codes of the space-to-depth conv: k = tap*16 + ch, tap = ka*KW2 + kb,
// ch = (dy*2 + dx)*C + c  <->  original tap (2*ka + dy - dh, 2*kb + dx - dw)
__global__ void weight_codes_s2d_kernel(const float* __restrict__ w, int8_t* __restrict__ codes,
                                        int O, int C, int KH, int KW, int KH2, int KW2, int dh,
                                        int dw, int Kpad, FSq p) {
  pdl_trigger();
  pdl_wait();
  const int64_t total = static_cast<int64_t>(O) * Kpad;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(i % Kpad);
    const int o = static_cast<int>(i / Kpad);
    const int tap = k >> 4, ch = k & 15;
    int8_t code = 0;
    if (tap < KH2 * KW2 && ch < 4 * C) {
      const int ka = tap / KW2, kb = tap - (tap / KW2) * KW2;
      const int sub = ch / C, c = ch - sub * C;
      const int kh = 2 * ka + (sub >> 1) - dh, kw = 2 * kb + (sub & 1) - dw;
      if (kh >= 0 && kh < KH && kw >= 0 && kw < KW) {
        const float v = w[((static_cast<int64_t>(o) * C + c) * KH + kh) * KW + kw];
        code = static_cast<int8_t>(static_cast<int>(__fsub_rn(fsq_code(v, p), p.zp)));
      }
    }
    codes[i] = code;
  }
}

// one warp per weight row: sum |code| with byte SIMD, max over rows
__global__ void weight_l1_kernel(const int8_t* __restrict__ codes, int O, int Kpad,
                                 int* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int o = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; o < O; o += warps) {
    const uint32_t* row = reinterpret_cast<const uint32_t*>(codes + static_cast<int64_t>(o) * Kpad);
    uint32_t acc = 0;
    for (int i = lane; i < Kpad / 4; i += 32) acc += __vsadu4(__vabsss4(row[i]), 0u);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
    if (lane == 0) atomicMax(out, static_cast<int>(acc));
  }
}

// int32 NCHW (8-bit value range) -> 8-bit NHWC rows: one thread per (pixel,
// 16-channel group), coalesced over pixels, one 16-byte store
__global__ void pack_i32_nhwc_kernel(const int32_t* __restrict__ x, uint8_t* __restrict__ out,
                                     int64_t pixels, int C, int H, int W, int ph, int pw,
                                     int ld, uint32_t fill) {
  pdl_trigger();
  pdl_wait();
  const int groups = ld / 16;
  const int64_t total = pixels * groups;
  const int HP = H + 2 * ph, WP = W + 2 * pw;
  const uint32_t fill4 = (fill & 0xFFu) * 0x01010101u;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t pix = i % pixels;  // (padded) pixel fastest: coalesced reads per channel
    const int g = static_cast<int>(i / pixels);
    const int64_t n = pix / (static_cast<int64_t>(HP) * WP);
    const int r = static_cast<int>(pix - n * HP * WP);
    const int h = r / WP - ph, w = r % WP - pw;
    uint32_t v[4] = {0, 0, 0, 0};
    if (h < 0 || h >= H || w < 0 || w >= W) {
      v[0] = v[1] = v[2] = v[3] = fill4;  // the padding value the zp0 correction assumes
    } else {
      const int64_t base = n * C * H * W + static_cast<int64_t>(h) * W + w;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int c = g * 16 + j;
        if (c < C) v[j >> 2] |= (static_cast<uint32_t>(x[base + static_cast<int64_t>(c) * H * W]) & 0xFFu) << (8 * (j & 3));
      }
    }
    *reinterpret_cast<int4*>(out + pix * ld + g * 16) =
        make_int4(static_cast<int>(v[0]), static_cast<int>(v[1]), static_cast<int>(v[2]),
                  static_cast<int>(v[3]));
  }
}

__global__ void pack_i32_weights_kernel(const int32_t* __restrict__ w, int8_t* __restrict__ codes,
                                        int32_t* __restrict__ wsum, int* __restrict__ bad, int O,
                                        int C, int taps, int ld, int Kpad, int64_t zp1) {
  pdl_trigger();
  pdl_wait();
  const int64_t total = static_cast<int64_t>(O) * Kpad;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(i % Kpad);
    const int o = static_cast<int>(i / Kpad);
    const int tap = k / ld, c = k - tap * ld;
    int8_t code = 0;
    if (tap < taps && c < C) {
      const int64_t v = static_cast<int64_t>(w[(static_cast<int64_t>(o) * C + c) * taps + tap]) - zp1;
      if (v < -128 || v > 127) atomicOr(bad, 1);
      code = static_cast<int8_t>(v);
      if (v != 0) atomicAdd(wsum + o, static_cast<int32_t>(v));
    }
    codes[i] = code;
  }
}

// one thread per output row: walks (kh, kw, c) with incremental counters and
// emits the row as 16-byte stores
__global__ void pack_im2col_kernel(const int8_t* __restrict__ x, int8_t* __restrict__ out, int N,
                                   int H, int W, int C, int ld, int KH, int KW, int sh, int sw,
                                   int ph, int pw, int OH, int OW, int Ktrue, int Kpad) {
  pdl_trigger();
  pdl_wait();
  const int64_t rows = static_cast<int64_t>(N) * OH * OW;
  for (int64_t m = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; m < rows;
       m += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int ow = static_cast<int>(m % OW);
    const int oh = static_cast<int>((m / OW) % OH);
    const int64_t n = m / (static_cast<int64_t>(OW) * OH);
    const int8_t* img = x + n * H * W * ld;
    const int ih0 = oh * sh - ph, iw0 = ow * sw - pw;
    int c = 0, kw = 0, kh = 0, k = 0;
    int4* dst = reinterpret_cast<int4*>(out + m * Kpad);
    for (int chunk = 0; chunk < Kpad / 16; ++chunk) {
      uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
      for (int b = 0; b < 16; ++b, ++k) {
        if (k < Ktrue) {
          const int ih = ih0 + kh, iw = iw0 + kw;
          int8_t v = 0;
          if (ih >= 0 && ih < H && iw >= 0 && iw < W) v = img[(ih * W + iw) * ld + c];
          w[b >> 2] |= static_cast<uint32_t>(static_cast<uint8_t>(v)) << (8 * (b & 3));
          if (++c == C) {
            c = 0;
            if (++kw == KW) {
              kw = 0;
              ++kh;
            }
          }
        }
      }
      dst[chunk] = make_int4(static_cast<int>(w[0]), static_cast<int>(w[1]),
                             static_cast<int>(w[2]), static_cast<int>(w[3]));
    }
  }
}

}  // namespace

void pack_im2col(const int8_t* x, int8_t* out, int N, int H, int W, int C, int ld, int KH, int KW,
                 int sh, int sw, int ph, int pw, int OH, int OW, int Ktrue, int Kpad,
                 cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(N) * OH * OW;
  if (total <= 0) return;
  launch_pdl(pack_im2col_kernel, dim3(grid_for(total, 128, 148 * 32)), dim3(128), 0, s, x, out, N, H, W, C, ld, KH, KW,
                                                                     sh, sw, ph, pw, OH, OW, Ktrue,
                                                                     Kpad);
  QC_CUDA_CHECK_LAUNCH();
}

void pack_i32_nhwc(const int32_t* x, uint8_t* out, int N, int C, int H, int W, int ph, int pw,
                   int ld, int32_t fill, cudaStream_t s) {
  const int64_t pixels = static_cast<int64_t>(N) * (H + 2 * ph) * (W + 2 * pw);
  const int64_t total = pixels * (ld / 16);
  if (total <= 0) return;
  launch_pdl(pack_i32_nhwc_kernel, dim3(grid_for(total, 256)), dim3(256), 0, s, x, out, pixels,
             C, H, W, ph, pw, ld, static_cast<uint32_t>(fill));
  QC_CUDA_CHECK_LAUNCH();
}

void pack_i32_weights(const int32_t* w, int8_t* codes, int32_t* wsum, int* bad, int O, int C,
                      int taps, int ld, int Kpad, int64_t zp1, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(O) * Kpad;
  if (total <= 0) return;
  launch_pdl(pack_i32_weights_kernel, dim3(grid_for(total, 256)), dim3(256), 0, s, w, codes,
             wsum, bad, O, C, taps, ld, Kpad, zp1);
  QC_CUDA_CHECK_LAUNCH();
}

void weight_l1_max(const int8_t* codes, int O, int Kpad, int* out, cudaStream_t s) {
  if (O <= 0) return;
  launch_pdl(weight_l1_kernel, dim3((O + 7) / 8), dim3(256), 0, s, codes, O, Kpad, out);
  QC_CUDA_CHECK_LAUNCH();
}

void stage_input_s2d(const float* x, int N, int C, int H, int W, const FSq& p, int8_t* out,
                     cudaStream_t s) {
  const int H2 = (H + 1) / 2, W2 = (W + 1) / 2;
  const int64_t total = static_cast<int64_t>(N) * H2 * W2;
  if (total <= 0) return;
  launch_pdl(input_s2d_kernel, dim3(static_cast<unsigned>((total + 255) / 256)), dim3(256), 0, s, x,
             N, C, H, W, H2, W2, p, out);
  QC_CUDA_CHECK_LAUNCH();
}

void stage_input_s2d_multi(const float* x, int N, int C, int H, int W, const FSq* ps,
                           int8_t* const* outs, int groups, cudaStream_t s) {
  const int H2 = (H + 1) / 2, W2 = (W + 1) / 2;
  const int64_t total = static_cast<int64_t>(N) * H2 * W2;
  if (total <= 0 || groups <= 0 || groups > 4 || C > 4) return;
  S2dMulti m{};
  for (int g = 0; g < groups; ++g) {
    m.p[g] = ps[g];
    m.out[g] = outs[g];
  }
  launch_pdl(input_s2d_multi_kernel, dim3(static_cast<unsigned>((total + 255) / 256)), dim3(256), 0,
             s, x, N, C, H, W, H2, W2, m, groups);
  QC_CUDA_CHECK_LAUNCH();
}

void weight_codes_s2d(const float* w, int8_t* codes, int O, int C, int KH, int KW, int KH2,
                      int KW2, int dh, int dw, int Kpad, const FSq& p, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(O) * Kpad;
  if (total <= 0) return;
  launch_pdl(weight_codes_s2d_kernel, dim3(grid_for(total, 256)), dim3(256), 0, s, w, codes, O, C, KH, KW, KH2, KW2,
                                                                dh, dw, Kpad, p);
  QC_CUDA_CHECK_LAUNCH();
}

void stage_input(const float* x, int N, int C, int HW, const ProgArgs& prog, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(N) * HW * ((C + 15) / 16);
  if (total <= 0) return;
  launch_pdl(input_kernel, dim3(grid_for(total, 256)), dim3(256), 0, s, x, N, C, HW, prog);
  QC_CUDA_CHECK_LAUNCH();
}

void stage_maxpool(const int8_t* x, int ld, float scale, int N, int C, int H, int W, int OH,
                   int OW, int kh, int kw, int sh, int sw, int ph, int pw, const ProgArgs& prog,
                   cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(N) * OH * OW * ((C + 15) / 16);
  if (total <= 0) return;
  if (prog.depth <= 1) {
    launch_pdl(maxpool_codes_kernel<1>, dim3(grid_for(total, 256)), dim3(256), 0, s, x, ld, scale, N, C, H, W, OH,
               OW, kh, kw, sh, sw, ph, pw, prog);
  } else {
    launch_pdl(maxpool_codes_kernel<3>, dim3(grid_for(total, 256)), dim3(256), 0, s, x, ld, scale, N, C, H, W, OH,
               OW, kh, kw, sh, sw, ph, pw, prog);
  }
  QC_CUDA_CHECK_LAUNCH();
}

void stage_avgpool_f32(const float* x, int ld, int N, int C, int H, int W, int OH, int OW, int kh,
                       int kw, int sh, int sw, int ph, int pw, double wk, const ProgArgs& prog,
                       const DwFast& fast, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(N) * OH * OW * ((C + 15) / 16);
  if (total <= 0) return;
  if (fast.n > 0) {
    launch_pdl(avgpool_f32_kernel<true>, dim3(grid_for(total, 256)), dim3(256), 0, s, x, ld, N, C, H, W, OH,
               OW, kh, kw, sh, sw, ph, pw, wk, prog, fast);
  } else {
    launch_pdl(avgpool_f32_kernel<false>, dim3(grid_for(total, 256)), dim3(256), 0, s, x, ld, N, C, H, W,
               OH, OW, kh, kw, sh, sw, ph, pw, wk, prog, fast);
  }
  QC_CUDA_CHECK_LAUNCH();
}

// [tap][ldw] int8 codes -> [quad][ldw] words of 4 consecutive taps' codes
__global__ void dw_weight_quads_kernel(const int8_t* __restrict__ codes, int taps, int ldw,
                                       int32_t* __restrict__ quads) {
  pdl_trigger();
  pdl_wait();
  const int nq = (taps + 3) / 4;
  const int64_t total = static_cast<int64_t>(nq) * ldw;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int q = static_cast<int>(i / ldw), c = static_cast<int>(i % ldw);
    uint32_t w = 0;
    for (int k = 0; k < 4; ++k) {
      const int t = 4 * q + k;
      if (t < taps) w |= static_cast<uint32_t>(static_cast<uint8_t>(codes[static_cast<int64_t>(t) * ldw + c])) << (8 * k);
    }
    quads[i] = static_cast<int32_t>(w);
  }
}

void dw_weight_quads(const int8_t* codes, int taps, int ldw, int32_t* quads, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>((taps + 3) / 4) * ldw;
  if (total <= 0) return;
  launch_pdl(dw_weight_quads_kernel, dim3(grid_for(total, 256)), dim3(256), 0, s, codes, taps, ldw, quads);
  QC_CUDA_CHECK_LAUNCH();
}

void stage_dw_conv(const int8_t* x, int ld, int N, int C, int H, int W, int KH, int KW, int sh,
                   int sw, int ph, int pw, int OH, int OW, const int32_t* wquads, int ldw,
                   const float* bias, float scale, const ProgArgs& prog, const DwFast& fast,
                   cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(N) * OH * OW * ((C + 15) / 16);
  if (total <= 0) return;
  if (fast.n > 0) {
    launch_pdl(dw_conv_kernel<true>, dim3(grid_for(total, 256)), dim3(256), 0, s, x, ld, N, C, H, W, KH, KW,
               sh, sw, ph, pw, OH, OW, wquads, ldw, bias, scale, prog, fast);
  } else {
    launch_pdl(dw_conv_kernel<false>, dim3(grid_for(total, 256)), dim3(256), 0, s, x, ld, N, C, H, W, KH, KW,
               sh, sw, ph, pw, OH, OW, wquads, ldw, bias, scale, prog, fast);
  }
  QC_CUDA_CHECK_LAUNCH();
}

void stage_gap(const float* x, int64_t ld, int N, int C, int HW, const ProgArgs& prog,
               cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(N) * C;
  if (total <= 0) return;
  launch_pdl(gap_rows_kernel, dim3(grid_for(total, 256)), dim3(256), 0, s, x, ld, N, C, HW, prog);
  QC_CUDA_CHECK_LAUNCH();
}

void stage_maxpool_stores(const int8_t* x, int ld, int N, int C, int H, int W, int OH, int OW,
                          int kh, int kw, int sh, int sw, int ph, int pw, const PoolStores& e,
                          cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(N) * OH * OW * (C / 16);
  if (total <= 0) return;
  const dim3 grid(static_cast<unsigned>((total + 255) / 256));  // one item per thread
  const bool k3 = kh == 3 && kw == 3;
#define QC_POOL(NO, K3)                                                                       \
  launch_pdl(maxpool_stores_kernel<NO, K3>, grid, dim3(256), 0, s, x, ld, N, C, H, W, OH, OW, \
             kh, kw, sh, sw, ph, pw, e)
  if (e.n_out == 2) {
    if (k3) QC_POOL(2, true); else QC_POOL(2, false);
  } else {
    if (k3) QC_POOL(1, true); else QC_POOL(1, false);
  }
#undef QC_POOL
  QC_CUDA_CHECK_LAUNCH();
}

void stage_ew(const ProgBuf& src, int64_t M, int C, const ProgArgs& prog, cudaStream_t s) {
  const int64_t total = M * ((C + 15) / 16);
  if (total <= 0) return;
  if (prog.depth <= 1) {
    launch_pdl(ew_kernel<1>, dim3(grid_for(total, 256)), dim3(256), 0, s, src, M, C, prog);
  } else if (prog.depth == 2) {
    launch_pdl(ew_kernel<2>, dim3(grid_for(total, 256)), dim3(256), 0, s, src, M, C, prog);
  } else {
    launch_pdl(ew_kernel<3>, dim3(grid_for(total, 256)), dim3(256), 0, s, src, M, C, prog);
  }
  QC_CUDA_CHECK_LAUNCH();
}

void weight_codes_v2(const float* w, int8_t* codes, int O, int C, int taps, int ldk, int Kpad,
                     const FSq& p, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(O) * Kpad;
  if (total <= 0) return;
  launch_pdl(weight_codes_v2_kernel, dim3(grid_for(total, 256)), dim3(256), 0, s, w, codes, O, C, taps, ldk, Kpad, p);
  QC_CUDA_CHECK_LAUNCH();
}

}  // namespace quantc::kern
