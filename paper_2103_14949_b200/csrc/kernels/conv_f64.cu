// conv_f64.cu — exact-order fp32 conv2d / dense (reference interpreter.cpp:
// 210-236 and 276-291).
//
// The reference accumulates every output in double, sequentially over
// k = (c, kh, kw), skipping padded taps, adds the bias in double and rounds to
// float once.  Products of two floats are exact in double, so a DFMA chain in
// the same k order reproduces every partial sum bit for bit; padded taps are
// fed as 0.0, which leaves the accumulator unchanged (it can never be -0.0:
// it starts at +0.0 and exact cancellation rounds to +0.0).  Therefore this
// kernel is bit-identical to the reference for all finite inputs.
//
// Implicit GEMM on CUDA-core FP64: M = N*OH*OW output pixels, N = O output
// channels, K = C*KH*KW.  CTA tile (16*TM) x (16*TN) with 256 threads, each
// owning a TM x TN register tile (rows ty+16i, cols tx+16j: conflict-free
// shared-memory reads), BK = 8, double-buffered shared memory with register
// prefetch of the next im2col/weight slice.  K is never split (order!).
//
// Grouped convs (op-set extension): grid.z = group; the
// GEMM runs over the group's C/G input channels and O/G output channels.
// Depthwise-like layers (O/G < 16, where a 16-wide channel tile would idle)
// take the direct kernel: one thread per output, the same (c, kh, kw) DFMA
// chain.  Both are what the reference computes on the block-diagonal dense
// rewrite of the layer (fixtures.py _depthwise; tests/test_rewrites.py): the
// off-group zero weights add signed zeros to an accumulator that is never
// -0.0, so skipping them leaves every partial sum unchanged.
#include <algorithm>

#include "common.cuh"

namespace quantc::kern {

namespace {

constexpr int BK = 8;

template <int TM, int TN>
__global__ void __launch_bounds__(256) conv_f64_kernel(const float* __restrict__ x,
                                                       const float* __restrict__ w,
                                                       const float* __restrict__ bias,
                                                       float* __restrict__ y, ConvShape cs) {
  constexpr int BM = 16 * TM, BN = 16 * TN;
  constexpr int A_PER = BM * BK / 256;  // im2col elements loaded per thread per tile
  constexpr int B_PER = (BN * BK + 255) / 256;
  __shared__ double As[2][BK][BM];
  __shared__ double Bs[2][BK][BN];

  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t M = static_cast<int64_t>(cs.N) * cs.OH * cs.OW;
  const int G = conv_groups(cs);
  const int Cg = cs.C / G, Og = cs.O / G;
  const int grp = blockIdx.z;
  const int K = Cg * cs.KH * cs.KW;
  const int khw = cs.KH * cs.KW;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * BM;
  const int n0 = blockIdx.y * BN;  // within the group
  w += static_cast<int64_t>(grp) * Og * K;

  // A loader: thread owns pixel column am = tid % BM and rows ak + (256/BM)*r
  const int am = tid % BM;
  const int ak0 = tid / BM;
  constexpr int AK_STEP = 256 / BM;
  const int64_t mg = m0 + am;
  const bool m_ok = mg < M;
  int img = 0, ih0 = 0, iw0 = 0;
  if (m_ok) {
    const int64_t ohw = static_cast<int64_t>(cs.OH) * cs.OW;
    img = static_cast<int>(mg / ohw);
    const int rem = static_cast<int>(mg % ohw);
    ih0 = (rem / cs.OW) * cs.sh - cs.ph;
    iw0 = (rem % cs.OW) * cs.sw - cs.pw;
  }
  const float* ximg = x + (static_cast<int64_t>(img) * cs.C + static_cast<int64_t>(grp) * Cg) * cs.H * cs.W;

  // this thread's A elements k = k0 + ak0 + r*AK_STEP as (c, kh, kw), walked
  // incrementally by BK per tile (mixed radix KH*KW, KW with one carry each):
  // no integer division in the K loop (it made the loader latency-bound)
  int ac[A_PER], akh[A_PER], akw[A_PER];
#pragma unroll
  for (int r = 0; r < A_PER; ++r) {
    const int k = ak0 + r * AK_STEP;
    ac[r] = k / khw;
    akh[r] = (k - ac[r] * khw) / cs.KW;
    akw[r] = k - ac[r] * khw - akh[r] * cs.KW;
  }
  const int step_c = BK / khw, step_kh = (BK % khw) / cs.KW, step_kw = BK % cs.KW;
  auto advance_a = [&]() {
#pragma unroll
    for (int r = 0; r < A_PER; ++r) {
      akw[r] += step_kw;
      int carry = akw[r] >= cs.KW;
      akw[r] -= carry ? cs.KW : 0;
      akh[r] += step_kh + carry;
      carry = akh[r] >= cs.KH;
      akh[r] -= carry ? cs.KH : 0;
      ac[r] += step_c + carry;
    }
  };
  const int64_t plane = static_cast<int64_t>(cs.H) * cs.W;
  auto load_a = [&](double (&ra)[A_PER]) {
#pragma unroll
    for (int r = 0; r < A_PER; ++r) {
      double v = 0.0;
      const int ih = ih0 + akh[r], iw = iw0 + akw[r];
      if (m_ok && ac[r] < Cg && static_cast<unsigned>(ih) < static_cast<unsigned>(cs.H) &&
          static_cast<unsigned>(iw) < static_cast<unsigned>(cs.W)) {
        v = static_cast<double>(__ldg(ximg + ac[r] * plane + ih * cs.W + iw));
      }
      ra[r] = v;
    }
  };
  // B loader: element e = tid + 256*r -> (bk = e % BK, bn = e / BK)
  auto load_b = [&](int k0, double (&rb)[B_PER]) {
#pragma unroll
    for (int r = 0; r < B_PER; ++r) {
      const int e = tid + 256 * r;
      const int bk = e % BK, bn = e / BK;
      const int k = k0 + bk, o = n0 + bn;
      double v = 0.0;
      if (bn < BN && k < K && o < Og) v = static_cast<double>(__ldg(w + static_cast<int64_t>(o) * K + k));
      rb[r] = v;
    }
  };
  auto store = [&](int buf, const double (&ra)[A_PER], const double (&rb)[B_PER]) {
#pragma unroll
    for (int r = 0; r < A_PER; ++r) As[buf][ak0 + r * AK_STEP][am] = ra[r];
#pragma unroll
    for (int r = 0; r < B_PER; ++r) {
      const int e = tid + 256 * r;
      if (e / BK < BN) Bs[buf][e % BK][e / BK] = rb[r];
    }
  };

  double acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0;

  double ra[A_PER], rb[B_PER];
  load_a(ra);
  advance_a();
  load_b(0, rb);
  store(0, ra, rb);
  __syncthreads();

  const int ntiles = (K + BK - 1) / BK;
  for (int t = 0; t < ntiles; ++t) {
    const int cur = t & 1;
    if (t + 1 < ntiles) {
      load_a(ra);
      advance_a();
      load_b((t + 1) * BK, rb);
    }
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      double a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[cur][kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[cur][kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = __fma_rn(a[i], b[j], acc[i][j]);
    }
    if (t + 1 < ntiles) store(cur ^ 1, ra, rb);
    __syncthreads();
  }

  const int64_t ohw = static_cast<int64_t>(cs.OH) * cs.OW;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t m = m0 + ty + 16 * i;
    if (m >= M) continue;
    const int64_t im = m / ohw, pix = m % ohw;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int ol = n0 + tx + 16 * j;
      if (ol >= Og) continue;
      const int o = grp * Og + ol;
      double v = acc[i][j];
      if (bias) v = __dadd_rn(v, static_cast<double>(__ldg(bias + o)));
      y[(im * cs.O + o) * ohw + pix] = __double2float_rn(v);
    }
  }
}

// direct grouped conv: one thread per output element (n, o, oh, ow), NCHW
// order (consecutive threads: consecutive ow, coalesced input rows)
__global__ void __launch_bounds__(256) conv_f64_direct_kernel(const float* __restrict__ x,
                                                              const float* __restrict__ w,
                                                              const float* __restrict__ bias,
                                                              float* __restrict__ y, ConvShape cs) {
  const int G = conv_groups(cs);
  const int Cg = cs.C / G, Og = cs.O / G;
  const int64_t ohw = static_cast<int64_t>(cs.OH) * cs.OW;
  const int64_t total = static_cast<int64_t>(cs.N) * cs.O * ohw;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t pix = i % ohw;
    const int64_t no = i / ohw;
    const int o = static_cast<int>(no % cs.O);
    const int64_t n = no / cs.O;
    const int oh = static_cast<int>(pix / cs.OW), ow = static_cast<int>(pix % cs.OW);
    const int c0 = (o / Og) * Cg;
    const float* wo = w + static_cast<int64_t>(o) * Cg * cs.KH * cs.KW;
    double acc = 0.0;
    for (int c = 0; c < Cg; ++c) {
      const float* xc = x + ((n * cs.C + c0 + c) * cs.H) * cs.W;
      for (int kh = 0; kh < cs.KH; ++kh) {
        const int ih = oh * cs.sh - cs.ph + kh;
        if (ih < 0 || ih >= cs.H) continue;
        for (int kw = 0; kw < cs.KW; ++kw) {
          const int iw = ow * cs.sw - cs.pw + kw;
          if (iw < 0 || iw >= cs.W) continue;
          acc = __fma_rn(static_cast<double>(__ldg(xc + static_cast<int64_t>(ih) * cs.W + iw)),
                         static_cast<double>(__ldg(wo + (c * cs.KH + kh) * cs.KW + kw)), acc);
        }
      }
    }
    if (bias) acc = __dadd_rn(acc, static_cast<double>(__ldg(bias + o)));
    y[i] = __double2float_rn(acc);
  }
}

template <int TM, int TN>
void launch(const float* x, const float* w, const float* bias, float* y, const ConvShape& cs,
            cudaStream_t s) {
  const int64_t M = static_cast<int64_t>(cs.N) * cs.OH * cs.OW;
  const int Og = cs.O / conv_groups(cs);
  dim3 grid(static_cast<unsigned>((M + 16 * TM - 1) / (16 * TM)),
            static_cast<unsigned>((Og + 16 * TN - 1) / (16 * TN)),
            static_cast<unsigned>(conv_groups(cs)));
  conv_f64_kernel<TM, TN><<<grid, 256, 0, s>>>(x, w, bias, y, cs);
  QC_CUDA_CHECK_LAUNCH();
}

}  // namespace

void conv2d_f64acc(const float* x, const float* w, const float* bias, float* y,
                   const ConvShape& cs, cudaStream_t s) {
  const int64_t M = static_cast<int64_t>(cs.N) * cs.OH * cs.OW;
  if (M <= 0 || cs.O <= 0) return;
  const int G = conv_groups(cs);
  const int Og = cs.O / G;
  if (G > 1 && Og < 16) {
    const int64_t total = M * cs.O;
    conv_f64_direct_kernel<<<static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 148 * 16)),
                             256, 0, s>>>(x, w, bias, y, cs);
    QC_CUDA_CHECK_LAUNCH();
    return;
  }
  // Pick the channel tile; shrink the pixel tile when the grid would not fill
  // the 148 SMs.
  if (Og <= 16) {
    launch<8, 1>(x, w, bias, y, cs, s);
  } else if (Og <= 32) {
    launch<8, 2>(x, w, bias, y, cs, s);
  } else if (Og <= 64) {
    launch<8, 4>(x, w, bias, y, cs, s);
  } else if ((M + 127) / 128 * ((Og + 127) / 128) * G >= 148) {
    launch<8, 8>(x, w, bias, y, cs, s);
  } else if ((M + 63) / 64 * ((Og + 127) / 128) * G >= 148) {
    launch<4, 8>(x, w, bias, y, cs, s);
  } else {
    launch<2, 8>(x, w, bias, y, cs, s);
  }
}

}  // namespace quantc::kern
