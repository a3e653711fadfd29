// fused.cuh — device side of the per-element epilogue programs (fused.h).
// A thread evaluates one row m over W consecutive columns n0..n0+W-1 at once
// (SIMD-in-thread), so codes leave as one W-byte vector store.
#pragma once

#include "common.cuh"
#include "fused.h"

namespace quantc::kern {

// fp32 simulated quantize with host-rounded bounds (exact for pow2 scales)
__device__ __forceinline__ float fsq_code(float v, const FSq& p) {
  if (p.has_acc) {
    if (v < p.lo_up) return p.q_lo;
    if (v > p.hi_dn) return p.q_hi;
  }
  float q = __fadd_rn(roundf(__fmul_rn(v, p.inv_s)), p.zp);
  q = (q < p.qmin) ? p.qmin : ((p.qmax < q) ? p.qmax : q);
  return q;
}

__device__ __forceinline__ float fsq_value(float v, const FSq& p) {
  if (p.passthrough) {
    if (p.has_acc) {
      if (v < p.lo_up) return p.lo_rn;
      if (v > p.hi_dn) return p.hi_rn;
    }
    return v;
  }
  return __fmul_rn(__fsub_rn(fsq_code(v, p), p.zp), p.s);
}

__device__ __forceinline__ int64_t buf_off(const ProgBuf& b, int64_t m, int n) {
  return (m / b.hw) * b.ld + (m % b.hw) * b.cs + n;
}

template <int W>
__device__ __forceinline__ void store_codes(const ProgBuf& b, int64_t m, int n0, int nvalid,
                                            const float (&q)[W]) {
  int8_t* dst = static_cast<int8_t*>(b.ptr) + buf_off(b, m, n0);
  if (W == 16 && nvalid == 16 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      w[i] = (static_cast<uint32_t>(static_cast<uint8_t>(static_cast<int8_t>(static_cast<int>(q[4 * i])))) |
              (static_cast<uint32_t>(static_cast<uint8_t>(static_cast<int8_t>(static_cast<int>(q[4 * i + 1])))) << 8) |
              (static_cast<uint32_t>(static_cast<uint8_t>(static_cast<int8_t>(static_cast<int>(q[4 * i + 2])))) << 16) |
              (static_cast<uint32_t>(static_cast<uint8_t>(static_cast<int8_t>(static_cast<int>(q[4 * i + 3])))) << 24));
    }
    *reinterpret_cast<int4*>(dst) = make_int4(static_cast<int>(w[0]), static_cast<int>(w[1]),
                                              static_cast<int>(w[2]), static_cast<int>(w[3]));
  } else {
#pragma unroll
    for (int j = 0; j < W; ++j) {
      if (j < nvalid) dst[j] = static_cast<int8_t>(static_cast<int>(q[j]));
    }
  }
}

template <int W>
__device__ __forceinline__ void load_values(const ProgBuf& b, int64_t m, int n0, int nvalid,
                                            float (&o)[W]) {
  if (b.kind == 0) {
    const int8_t* src = static_cast<const int8_t*>(b.ptr) + buf_off(b, m, n0);
    if (W == 16 && nvalid == 16 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
      const int4 raw = *reinterpret_cast<const int4*>(src);
      const int8_t* c = reinterpret_cast<const int8_t*>(&raw);
#pragma unroll
      for (int j = 0; j < W; ++j) o[j] = __fmul_rn(static_cast<float>(c[j]), b.scale);
    } else {
#pragma unroll
      for (int j = 0; j < W; ++j) o[j] = j < nvalid ? __fmul_rn(static_cast<float>(src[j]), b.scale) : 0.0f;
    }
  } else {
    const float* src = static_cast<const float*>(b.ptr) + buf_off(b, m, n0);
#pragma unroll
    for (int j = 0; j < W; ++j) o[j] = j < nvalid ? src[j] : 0.0f;
  }
}

template <int W>
__device__ __forceinline__ void run_prog(float (&v)[W], int64_t m, int n0, int nvalid,
                                         const ProgArgs& a) {
  float s0[W], s1[W], s2[W];
  int sp = 0;
  for (int pc = 0; pc < a.n_code; ++pc) {
    const ProgInstr ins = a.code[pc];
    switch (ins.op) {
      case kPSq: {
        const FSq p = a.sq[ins.a];
#pragma unroll
        for (int j = 0; j < W; ++j) v[j] = fsq_value(v[j], p);
        break;
      }
      case kPSqStore8: {
        const FSq p = a.sq[ins.a];
        float q[W];
#pragma unroll
        for (int j = 0; j < W; ++j) {
          q[j] = __fsub_rn(fsq_code(v[j], p), p.zp);
          v[j] = __fmul_rn(q[j], p.s);
        }
        store_codes<W>(a.bufs[ins.b], m, n0, nvalid, q);
        break;
      }
      case kPRelu:
#pragma unroll
        for (int j = 0; j < W; ++j) v[j] = (v[j] < 0.0f) ? 0.0f : v[j];
        break;
      case kPClip: {
        const float2 c = a.clip[ins.a];
#pragma unroll
        for (int j = 0; j < W; ++j) v[j] = (v[j] < c.x) ? c.x : ((c.y < v[j]) ? c.y : v[j]);
        break;
      }
      case kPAdd: {
        float o[W];
        load_values<W>(a.bufs[ins.b], m, n0, nvalid, o);
#pragma unroll
        for (int j = 0; j < W; ++j) v[j] = __fadd_rn(v[j], o[j]);
        break;
      }
      case kPStoreF32: {
        const ProgBuf& b = a.bufs[ins.b];
        float* dst = static_cast<float*>(b.ptr) + buf_off(b, m, n0);
#pragma unroll
        for (int j = 0; j < W; ++j) {
          if (j < nvalid) dst[j] = v[j];
        }
        break;
      }
      case kPPush:
        if (sp == 0) {
#pragma unroll
          for (int j = 0; j < W; ++j) s0[j] = v[j];
        } else if (sp == 1) {
#pragma unroll
          for (int j = 0; j < W; ++j) s1[j] = v[j];
        } else {
#pragma unroll
          for (int j = 0; j < W; ++j) s2[j] = v[j];
        }
        ++sp;
        break;
      case kPPop:
        --sp;
        if (sp == 0) {
#pragma unroll
          for (int j = 0; j < W; ++j) v[j] = s0[j];
        } else if (sp == 1) {
#pragma unroll
          for (int j = 0; j < W; ++j) v[j] = s1[j];
        } else {
#pragma unroll
          for (int j = 0; j < W; ++j) v[j] = s2[j];
        }
        break;
      default:
        break;
    }
  }
}

}  // namespace quantc::kern
