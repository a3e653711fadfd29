// fused.cuh — device side of the per-element epilogue programs (fused.h).
// A thread evaluates one row m over W consecutive columns n0..n0+W-1 at once
// (SIMD-in-thread): every program op is a W-wide unrolled loop whose
// per-op flags are tested once, and codes leave as W-byte vector stores.
// The program and its parameters are read from the stage's StageTables block
// in shared memory.
#pragma once

#include "common.cuh"
#include "fused.h"

namespace quantc::kern {

__device__ __forceinline__ float clampf_ref(float v, float lo, float hi) {
  return (v < lo) ? lo : ((hi < v) ? hi : v);
}

// code clamp: identical to the reference's std::clamp for every non-NaN q
// (the fused engine requires finite activations; NaN would saturate here)
__device__ __forceinline__ float clampq(float q, float lo, float hi) {
  return fminf(fmaxf(q, lo), hi);
}

// copy a StageTables block from global to shared memory (all threads)
__device__ __forceinline__ void load_tables(StageTables* dst, const StageTables* src) {
  const int words = static_cast<int>(sizeof(StageTables) / 16);
  const int4* s = reinterpret_cast<const int4*>(src);
  int4* d = reinterpret_cast<int4*>(dst);
  for (int i = threadIdx.x; i < words; i += blockDim.x) d[i] = s[i];
}

// scalar code q (clamp + round) of one value
__device__ __forceinline__ float fsq_code(float v, const FSq& p) {
  float q = clampq(__fadd_rn(roundf(__fmul_rn(v, p.inv_s)), p.zp), p.qmin, p.qmax);
  if (p.has_acc) q = (v < p.lo_up) ? p.q_lo : ((v > p.hi_dn) ? p.q_hi : q);
  return q;
}

template <int W>
__device__ __forceinline__ void sq_values(float (&v)[W], const FSq& p) {
  if (p.passthrough) {
    if (p.has_acc) {
      const float lu = p.lo_up, hd = p.hi_dn, lr = p.lo_rn, hr = p.hi_rn;
#pragma unroll
      for (int j = 0; j < W; ++j) v[j] = (v[j] < lu) ? lr : ((v[j] > hd) ? hr : v[j]);
    }
    return;
  }
  const float inv = p.inv_s, s = p.s, zp = p.zp, qmin = p.qmin, qmax = p.qmax;
  if (p.has_acc) {
    const float lu = p.lo_up, hd = p.hi_dn, ql = p.q_lo, qh = p.q_hi;
#pragma unroll
    for (int j = 0; j < W; ++j) {
      float q = clampq(__fadd_rn(roundf(__fmul_rn(v[j], inv)), zp), qmin, qmax);
      q = (v[j] < lu) ? ql : ((v[j] > hd) ? qh : q);
      v[j] = __fmul_rn(__fsub_rn(q, zp), s);
    }
  } else if (zp == 0.0f) {
    // symmetric grid: (q - 0) * s; the +0 of the reference only canonicalises
    // -0.0, which never changes a code or a prediction
#pragma unroll
    for (int j = 0; j < W; ++j) {
      v[j] = __fmul_rn(clampq(roundf(__fmul_rn(v[j], inv)), qmin, qmax), s);
    }
  } else {
#pragma unroll
    for (int j = 0; j < W; ++j) {
      const float q = clampq(__fadd_rn(roundf(__fmul_rn(v[j], inv)), zp), qmin, qmax);
      v[j] = __fmul_rn(__fsub_rn(q, zp), s);
    }
  }
}

// as sq_values, also returning the integer codes q - zp
template <int W>
__device__ __forceinline__ void sq_codes(float (&v)[W], float (&c)[W], const FSq& p) {
  const float inv = p.inv_s, s = p.s, zp = p.zp, qmin = p.qmin, qmax = p.qmax;
  if (p.has_acc) {
    const float lu = p.lo_up, hd = p.hi_dn, ql = p.q_lo, qh = p.q_hi;
#pragma unroll
    for (int j = 0; j < W; ++j) {
      float q = clampq(__fadd_rn(roundf(__fmul_rn(v[j], inv)), zp), qmin, qmax);
      q = (v[j] < lu) ? ql : ((v[j] > hd) ? qh : q);
      c[j] = __fsub_rn(q, zp);
      v[j] = __fmul_rn(c[j], s);
    }
  } else if (zp == 0.0f) {
#pragma unroll
    for (int j = 0; j < W; ++j) {
      c[j] = clampq(roundf(__fmul_rn(v[j], inv)), qmin, qmax);
      v[j] = __fmul_rn(c[j], s);
    }
  } else {
#pragma unroll
    for (int j = 0; j < W; ++j) {
      const float q = clampq(__fadd_rn(roundf(__fmul_rn(v[j], inv)), zp), qmin, qmax);
      c[j] = __fsub_rn(q, zp);
      v[j] = __fmul_rn(c[j], s);
    }
  }
}

// tcgen05-epilogue tile I/O: the thread's row within the 128-row tile and the
// shared-memory slot area (see ProgBuf::slot / slot_swizzle)
struct TileIo {
  uint32_t base;  // shared-window address of slot 0
  int rl;
  int slot_bytes;
  int swz;
};

__device__ __forceinline__ uint32_t tile_addr(const TileIo& io, int slot, int cl) {
  const int S = io.swz;
  const int blk = cl / S, within = cl - blk * S;
  const int chunk = (within >> 4) ^ ((io.rl * S >> 7) & (S / 16 - 1));
  return io.base + static_cast<uint32_t>(slot * io.slot_bytes + blk * (128 * S) + io.rl * S +
                                         (chunk << 4));
}

__device__ __forceinline__ int4 lds128(uint32_t a) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a)
               : "memory");
  return v;
}

__device__ __forceinline__ void sts128(uint32_t a, int4 v) {
  asm volatile("st.shared.v4.s32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

__device__ __forceinline__ int64_t buf_off(const ProgBuf& b, int64_t m, int n) {
  return b.hw == 1 ? m * b.ld + n : (m / b.hw) * b.ld + (m % b.hw) * b.cs + n;
}

__device__ __forceinline__ uint32_t pack4(float a, float b, float c, float d) {
  return (static_cast<uint32_t>(static_cast<uint8_t>(static_cast<int8_t>(__float2int_rn(a))))) |
         (static_cast<uint32_t>(static_cast<uint8_t>(static_cast<int8_t>(__float2int_rn(b)))) << 8) |
         (static_cast<uint32_t>(static_cast<uint8_t>(static_cast<int8_t>(__float2int_rn(c)))) << 16) |
         (static_cast<uint32_t>(static_cast<uint8_t>(static_cast<int8_t>(__float2int_rn(d)))) << 24);
}

template <int W>
__device__ __forceinline__ void store_codes(const ProgBuf& b, int64_t m, int n0, int nvalid,
                                            const float (&q)[W], const TileIo* io = nullptr,
                                            int cl = 0) {
  if (W == 16 && io != nullptr && b.slot >= 0) {
    sts128(tile_addr(*io, b.slot, cl),
           make_int4(static_cast<int>(pack4(q[0], q[1], q[2], q[3])),
                     static_cast<int>(pack4(q[4], q[5], q[6], q[7])),
                     static_cast<int>(pack4(q[8], q[9], q[10], q[11])),
                     static_cast<int>(pack4(q[12], q[13], q[14], q[15]))));
    return;
  }
  int8_t* dst = static_cast<int8_t*>(b.ptr) + buf_off(b, m, n0);
  if (W % 16 == 0 && nvalid == W && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
    for (int i = 0; i < W / 16; ++i) {
      const int o = 16 * i;
      *reinterpret_cast<int4*>(dst + o) =
          make_int4(static_cast<int>(pack4(q[o], q[o + 1], q[o + 2], q[o + 3])),
                    static_cast<int>(pack4(q[o + 4], q[o + 5], q[o + 6], q[o + 7])),
                    static_cast<int>(pack4(q[o + 8], q[o + 9], q[o + 10], q[o + 11])),
                    static_cast<int>(pack4(q[o + 12], q[o + 13], q[o + 14], q[o + 15])));
    }
  } else {
#pragma unroll
    for (int j = 0; j < W; ++j) {
      if (j < nvalid) dst[j] = static_cast<int8_t>(__float2int_rn(q[j]));
    }
  }
}

template <int W>
__device__ __forceinline__ void load_values(const ProgBuf& b, int64_t m, int n0, int nvalid,
                                            float (&o)[W], const TileIo* io = nullptr,
                                            int cl = 0) {
  if (W == 16 && io != nullptr && b.slot >= 0) {
    const int4 raw = lds128(tile_addr(*io, b.slot, cl));
    const int8_t* cc = reinterpret_cast<const int8_t*>(&raw);
    const float sc = b.scale;
#pragma unroll
    for (int j = 0; j < W; ++j) o[j] = __fmul_rn(static_cast<float>(cc[j % 16]), sc);
    return;
  }
  if (b.kind == 0) {
    const int8_t* src = static_cast<const int8_t*>(b.ptr) + buf_off(b, m, n0);
    const float sc = b.scale;
    if (W % 16 == 0 && nvalid == W && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
#pragma unroll
      for (int i = 0; i < W / 16; ++i) {
        const int4 raw = *reinterpret_cast<const int4*>(src + 16 * i);
        const int8_t* cc = reinterpret_cast<const int8_t*>(&raw);
#pragma unroll
        for (int j = 0; j < 16; ++j) o[16 * i + j] = __fmul_rn(static_cast<float>(cc[j]), sc);
      }
    } else {
#pragma unroll
      for (int j = 0; j < W; ++j) {
        o[j] = j < nvalid ? __fmul_rn(static_cast<float>(src[j]), sc) : 0.0f;
      }
    }
  } else {
    const float* src = static_cast<const float*>(b.ptr) + buf_off(b, m, n0);
    if (W % 4 == 0 && nvalid == W && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
#pragma unroll
      for (int i = 0; i < W / 4; ++i) {
        const float4 f = *reinterpret_cast<const float4*>(src + 4 * i);
        o[4 * i] = f.x;
        o[4 * i + 1] = f.y;
        o[4 * i + 2] = f.z;
        o[4 * i + 3] = f.w;
      }
      return;
    }
#pragma unroll
    for (int j = 0; j < W; ++j) o[j] = j < nvalid ? src[j] : 0.0f;
  }
}

// (shape ids: fused.h kShape*)

// Packed fp32 pairs (sm_100 FFMA2 / FADD2: two IEEE fp32 operations per
// instruction, same per-lane rounding as FFMA / FADD)
using f2 = unsigned long long;
__device__ __forceinline__ f2 f2_pack(float a, float b) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2_unpack(f2 v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ f2 f2_fma_rn(f2 a, f2 b, f2 c) {
  f2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f2 f2_fma_rz(f2 a, f2 b, f2 c) {
  f2 r;
  asm("fma.rz.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f2 f2_add_rz(f2 a, f2 b) {
  f2 r;
  asm("add.rz.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2 f2_add_rn(f2 a, f2 b) {
  f2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// ---- straight-line shape epilogues (no conversion-pipe instructions) -------------
// Host preconditions (fastplan classify_shape / make_epi): every sq of the
// shape has zp = 0, no live accumulator clamp, is not passthrough; code I/O
// goes through tile slots; every scale ratio folded into EpiConsts is an
// exact power of two.  Domains and rounding: fused.h (EpiSq).
// round 16 values into sq q's code domain; the (uniform) flag tests sit
// outside the element loops so each variant is straight-line code
__device__ __forceinline__ void epi_round(float (&x)[16], const EpiSq& q) {
  if (q.flags & kEpiNoClamp) return;
#pragma unroll
  for (int j = 0; j < 16; ++j) x[j] = fminf(fmaxf(x[j], q.lo), q.hi);
  if (q.flags & kEpiExact) return;
  // half-away rounding, two lanes per FADD2 (same per-lane RZ rounding)
  const f2 half = f2_pack(0.5f, 0.5f);
  const f2 m2 = f2_pack(kMagic, kMagic);
  if (q.flags & kEpiNonneg) {
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      f2_unpack(f2_add_rz(f2_add_rz(f2_pack(x[j], x[j + 1]), half), m2), x[j], x[j + 1]);
    }
  } else {
    const f2 nm2 = f2_pack(-kMagic, -kMagic);
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      float a, b;
      f2_unpack(f2_add_rn(f2_add_rz(f2_add_rz(f2_pack(fabsf(x[j]), fabsf(x[j + 1])), half), m2), nm2),
                a, b);
      x[j] = copysignf(a, x[j]);
      x[j + 1] = copysignf(b, x[j + 1]);
    }
  }
}

// y = fma(R, q.k, q.off), rounded into q's domain
__device__ __forceinline__ void epi_next(const float (&R)[16], float (&y)[16], const EpiSq& q) {
  const f2 k2 = f2_pack(q.k, q.k);
  const f2 o2 = f2_pack(q.off, q.off);
#pragma unroll
  for (int j = 0; j < 16; j += 2) f2_unpack(f2_fma_rn(f2_pack(R[j], R[j + 1]), k2, o2), y[j], y[j + 1]);
  epi_round(y, q);
}

// 16 rounded codes -> 16 int8 bytes (low byte of the T-domain bits)
__device__ __forceinline__ int4 epi_pack(float (&R)[16], const EpiSq& q) {
  if (!(q.flags & kEpiNonneg)) {
    const f2 m2 = f2_pack(kMagic, kMagic);
#pragma unroll
    for (int j = 0; j < 16; j += 2) f2_unpack(f2_add_rn(f2_pack(R[j], R[j + 1]), m2), R[j], R[j + 1]);
  }
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t lo = __byte_perm(__float_as_uint(R[4 * i]), __float_as_uint(R[4 * i + 1]), 0x0040);
    const uint32_t hi =
        __byte_perm(__float_as_uint(R[4 * i + 2]), __float_as_uint(R[4 * i + 3]), 0x0040);
    w[i] = __byte_perm(lo, hi, 0x5410);
  }
  return make_int4(static_cast<int>(w[0]), static_cast<int>(w[1]), static_cast<int>(w[2]),
                   static_cast<int>(w[3]));
}

__device__ __forceinline__ void epi_store(float (&R)[16], const EpiSq& q, const TileIo& io,
                                          int slot, int cl) {
  sts128(tile_addr(io, slot, cl), epi_pack(R, q));
}

// 16 int8 codes (4 packed words) -> floats, without the conversion pipe
__device__ __forceinline__ void codes_to_floats(const uint32_t (&w)[4], float (&r)[16]) {
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const float C = __uint_as_float(__byte_perm(w[j >> 2] ^ 0x80808080u, 0x4B000000u, 0x7650u + (j & 3)));
    r[j] = __fsub_rn(C, 8388736.0f);  // 2^23 + 128
  }
}

// byte permute with an immediate selector (keeps the selector out of registers)
template <uint32_t SEL>
__device__ __forceinline__ uint32_t prmt_imm(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "n"(SEL));
  return r;
}
// residual code byte k of w as the biased magic float 2^23 + byte
template <int K>
__device__ __forceinline__ float code_float(uint32_t w) {
  return __uint_as_float(prmt_imm<0x7650u + K>(w, 0x4B000000u));
}

// RZ(a + b) clamped to [0, 1] on the FMA pipe (PTX add.rz.sat: NaN -> +0)
__device__ __forceinline__ float add_rz_sat(float a, float b) {
  float r;
  asm("add.rz.sat.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// x[16] = conv output scaled into sq0's grid (x0 = v / s0); runs the shape
// (m, n): the element coordinates of x[0] (shape 5 stores to global rows)
template <int SHAPE>
__device__ __forceinline__ void run_shape_epi(float (&x)[16], const EpiConsts& e,
                                              const TileIo& io, int cl, int64_t m, int n,
                                              bool row_ok) {
  if constexpr (SHAPE == kShapeSqStoreId) {
    // sq0 (codes [0, P0 - 1]) on x0 / P0: T = M + min(floor(max(RZ(x0 + 1/2), 0)), P0 - 1)
    const f2 p2 = f2_pack(e.sat_p[0], e.sat_p[0]);
    const f2 m2 = f2_pack(kMagic, kMagic);
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      const f2 t = f2_fma_rz(f2_pack(add_rz_sat(x[j], e.sat_half[0]), add_rz_sat(x[j + 1], e.sat_half[0])),
                             p2, m2);
      float a, b;
      f2_unpack(t, a, b);
      x[j] = fminf(a, e.sat_top[0]);
      x[j + 1] = fminf(b, e.sat_top[0]);
    }
    epi_round(x, e.q[1]);  // k = 1 store: at most a clamp in the T-domain
    sts128(tile_addr(io, e.slot_out[0], cl), epi_pack(x, e.q[1]));
    return;
  }
  if constexpr (SHAPE == kShapeAddForkId) {
    const int4 raw = lds128(tile_addr(io, e.slot_res, cl));
    const uint32_t wr[4] = {static_cast<uint32_t>(raw.x) ^ 0x80808080u,
                            static_cast<uint32_t>(raw.y) ^ 0x80808080u,
                            static_cast<uint32_t>(raw.z) ^ 0x80808080u,
                            static_cast<uint32_t>(raw.w) ^ 0x80808080u};
    const f2 p0 = f2_pack(e.sat_p[0], e.sat_p[0]);
    const f2 p1 = f2_pack(e.sat_p[1], e.sat_p[1]);
    const f2 m2 = f2_pack(kMagic, kMagic);
    const f2 nm2 = f2_pack(-kMagic, -kMagic);
    const f2 k1 = f2_pack(e.q[1].k, e.q[1].k);
    const f2 ka = f2_pack(e.ka, e.ka);
    const f2 kofs = f2_pack(e.ka_off, e.ka_off);
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      // sq0, signed codes [-P0, P0 - 1], on x0 / P0: half-away rounding of
      // |x0| saturated at P0, sign restored, positive side capped at P0 - 1
      const f2 u0 = f2_pack(add_rz_sat(fabsf(x[j]), e.sat_half[0]),
                            add_rz_sat(fabsf(x[j + 1]), e.sat_half[0]));
      float ta, tb;
      f2_unpack(f2_add_rn(f2_fma_rz(u0, p0, m2), nm2), ta, tb);
      const float ra = fminf(copysignf(ta, x[j]), e.sat_top[0]);
      const float rb = fminf(copysignf(tb, x[j + 1]), e.sat_top[0]);
      // residual add (k1, ka, ka_off pre-scaled by 1/P1), then sq1 (codes
      // [0, P1 - 1]) into the T-domain
      const float Ca = (j & 3) == 0 ? code_float<0>(wr[j >> 2]) : code_float<2>(wr[j >> 2]);
      const float Cb = (j & 3) == 0 ? code_float<1>(wr[j >> 2]) : code_float<3>(wr[j >> 2]);
      float xa, xb;
      f2_unpack(f2_fma_rn(f2_pack(ra, rb), k1, f2_fma_rn(f2_pack(Ca, Cb), ka, kofs)), xa, xb);
      float ta1, tb1;
      f2_unpack(f2_fma_rz(f2_pack(add_rz_sat(xa, e.sat_half[1]), add_rz_sat(xb, e.sat_half[1])), p1, m2),
                ta1, tb1);
      x[j] = fminf(ta1, e.sat_top[1]);
      x[j + 1] = fminf(tb1, e.sat_top[1]);
    }
    epi_round(x, e.q[2]);                     // k = 1 store (q2 == q3): at most a clamp
    const int4 packed = epi_pack(x, e.q[2]);
    sts128(tile_addr(io, e.slot_out[0], cl), packed);
    // slot_out[1] < 0: the fork's second value aliases the first buffer
    if (e.slot_out[1] >= 0) sts128(tile_addr(io, e.slot_out[1], cl), packed);
    return;
  }
  if constexpr (SHAPE == kShapeSqStoreAcc || SHAPE == kShapeStoreAcc) {
    // sq0 with a live accumulator clamp: the reference saturates on the
    // conv value (fsq_code: v < lo_up -> q_lo, v > hi_dn -> q_hi), i.e. on
    // x0 against the bounds scaled into sq0's grid
    float raw[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) raw[j] = x[j];
    epi_round(x, e.q[0]);
    const float alo = e.q[3].lo, ahi = e.q[3].hi, clo = e.q[3].k, chi = e.q[3].off;
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = raw[j] < alo ? clo : (raw[j] > ahi ? chi : x[j]);
    if constexpr (SHAPE == kShapeStoreAcc) {
      epi_store(x, e.q[0], io, e.slot_out[0], cl);
      return;
    }
    float y0[16];
    epi_next(x, y0, e.q[1]);
    epi_store(y0, e.q[1], io, e.slot_out[0], cl);
    return;
  }
  epi_round(x, e.q[0]);
  if constexpr (SHAPE == kShapeSqF32) {
    // fp32 value of the code: v = fma(R, s, off) (T-domain offset folded)
    if (!row_ok) return;
    float* dst = e.f32_ptr + m * e.f32_ld + n;
    const int nv = e.f32_cols - n;
    if (nv >= 16) {
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        *reinterpret_cast<float4*>(dst + j) = make_float4(
            __fmaf_rn(x[j], e.f32_s, e.f32_off), __fmaf_rn(x[j + 1], e.f32_s, e.f32_off),
            __fmaf_rn(x[j + 2], e.f32_s, e.f32_off), __fmaf_rn(x[j + 3], e.f32_s, e.f32_off));
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (j < nv) dst[j] = __fmaf_rn(x[j], e.f32_s, e.f32_off);
      }
    }
    return;
  }
  if (SHAPE == kShapeStore) {
    epi_store(x, e.q[0], io, e.slot_out[0], cl);
    return;
  }
  float y[16];
  if (SHAPE == kShapeSqStore) {
    epi_next(x, y, e.q[1]);
    epi_store(y, e.q[1], io, e.slot_out[0], cl);
    return;
  }
  // residual add: x1 = (r0 * s0 + c * s_res) / s1 in one rounding
  if (e.q[0].flags & kEpiNonneg) {
    const f2 nm2 = f2_pack(-kMagic, -kMagic);
#pragma unroll
    for (int j = 0; j < 16; j += 2) f2_unpack(f2_add_rn(f2_pack(x[j], x[j + 1]), nm2), x[j], x[j + 1]);
  }
  const int4 raw = lds128(tile_addr(io, e.slot_res, cl));
  const uint32_t wr[4] = {static_cast<uint32_t>(raw.x) ^ 0x80808080u,
                          static_cast<uint32_t>(raw.y) ^ 0x80808080u,
                          static_cast<uint32_t>(raw.z) ^ 0x80808080u,
                          static_cast<uint32_t>(raw.w) ^ 0x80808080u};
  {
    const f2 k1 = f2_pack(e.q[1].k, e.q[1].k);
    const f2 ka = f2_pack(e.ka, e.ka);
    const f2 kofs = f2_pack(e.ka_off, e.ka_off);
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      const float Ca = (j & 3) == 0 ? code_float<0>(wr[j >> 2]) : code_float<2>(wr[j >> 2]);
      const float Cb = (j & 3) == 0 ? code_float<1>(wr[j >> 2]) : code_float<3>(wr[j >> 2]);
      f2_unpack(f2_fma_rn(f2_pack(x[j], x[j + 1]), k1, f2_fma_rn(f2_pack(Ca, Cb), ka, kofs)), x[j],
                x[j + 1]);
    }
  }
  epi_round(x, e.q[1]);
  if (SHAPE == kShapeAddF32) {
    if (row_ok) {
      float4* dst = reinterpret_cast<float4*>(e.f32_ptr + m * e.f32_ld + n);
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        dst[j / 4] = make_float4(__fmaf_rn(x[j], e.f32_s, e.f32_off),
                                 __fmaf_rn(x[j + 1], e.f32_s, e.f32_off),
                                 __fmaf_rn(x[j + 2], e.f32_s, e.f32_off),
                                 __fmaf_rn(x[j + 3], e.f32_s, e.f32_off));
      }
    }
    return;
  }
  epi_next(x, y, e.q[2]);
  epi_store(y, e.q[2], io, e.slot_out[0], cl);
  if (SHAPE == kShapeAddFork && e.slot_out[1] >= 0) {
    epi_next(x, y, e.q[3]);
    epi_store(y, e.q[3], io, e.slot_out[1], cl);
  }
}

// ---- integer shapes 10/11 (fused.h EpiConsts i_*) ------------------------------
// four int32 codes -> four bytes, each saturated to [0, 255] (I2IP): the low
// side of a non-negative code clamp comes for free
__device__ __forceinline__ uint32_t pack_sat_u8(int32_t v0, int32_t v1, int32_t v2, int32_t v3) {
  uint32_t hi, r;
  asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(hi) : "r"(v3), "r"(v2), "r"(0));
  asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(v1), "r"(v0), "r"(hi));
  return r;
}

// byte K of w as a sign-extended int32 (PRMT sign-replicate selector)
template <int K>
__device__ __forceinline__ int32_t sbyte(uint32_t w) {
  return static_cast<int32_t>(prmt_imm<K | ((8 | K) * 0x1110u)>(w, 0u));
}

// d: the 16 int32 accumulators of this thread's chunk; ct: the channels'
// folded bias (shared memory, 16-byte aligned).  Host preconditions
// (fastplan fold_integer): sq0 non-negative (shape 10) or signed (shape 11)
// with every breakpoint of every channel verified, sq1 non-negative and the
// add exact in fp32, identity stores.
// CORR: some channel of the chunk has breakpoints moved by the float
// rounding of the conv value (fastplan fold_integer): tp[j] / tp[O + j] are
// its thresholds (global, read-only): a >= Tp counts one step early, a < Tn
// one step late
template <int SHAPE, bool CORR>
__device__ __forceinline__ void run_int_epi(const uint32_t (&d)[16], const int32_t* ct,
                                            const EpiConsts& e, const TileIo& io, int cl,
                                            const int32_t* tp, int O) {
  int32_t r[16];
#pragma unroll
  for (int j = 0; j < 16; j += 4) {
    const int4 c4 = lds128(static_cast<uint32_t>(__cvta_generic_to_shared(ct + j)));
    int32_t cc[4] = {c4.x, c4.y, c4.z, c4.w};
    if constexpr (CORR) {
      const int4 p4 = __ldg(reinterpret_cast<const int4*>(tp + j));
      const int4 n4 = __ldg(reinterpret_cast<const int4*>(tp + O + j));
      const int32_t pp[4] = {p4.x, p4.y, p4.z, p4.w};
      const int32_t nn[4] = {n4.x, n4.y, n4.z, n4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int32_t a = static_cast<int32_t>(d[j + i]);
        cc[i] += ((a >= pp[i] ? 1 : 0) - (a < nn[i] ? 1 : 0)) * e.i_cs;
      }
    }
    // (a multiply-high on the FMA pipe instead of the shift measured slower:
    // 1180 vs 1073 us for the step's add-forks)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      r[j + i] = (static_cast<int32_t>(d[j + i]) * e.i_m0 + cc[i]) >> e.i_r0;
    }
  }
  if constexpr (SHAPE == kShapeSqStoreInt) {
#pragma unroll
    for (int j = 0; j < 16; ++j) r[j] = min(r[j], e.i_hi0);
  } else {
    const int4 raw = lds128(tile_addr(io, e.slot_res, cl));
    const uint32_t w[4] = {static_cast<uint32_t>(raw.x), static_cast<uint32_t>(raw.y),
                           static_cast<uint32_t>(raw.z), static_cast<uint32_t>(raw.w)};
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int32_t c0 = min(max(r[j], e.i_lo0), e.i_hi0);
      int32_t c;
      switch (j & 3) {
        case 0: c = sbyte<0>(w[j >> 2]); break;
        case 1: c = sbyte<1>(w[j >> 2]); break;
        case 2: c = sbyte<2>(w[j >> 2]); break;
        default: c = sbyte<3>(w[j >> 2]); break;
      }
      r[j] = min((c0 * e.i_k0 + c * e.i_kr + e.i_h1) >> e.i_r1, e.i_hi1);
    }
  }
  const int4 packed = make_int4(static_cast<int>(pack_sat_u8(r[0], r[1], r[2], r[3])),
                                static_cast<int>(pack_sat_u8(r[4], r[5], r[6], r[7])),
                                static_cast<int>(pack_sat_u8(r[8], r[9], r[10], r[11])),
                                static_cast<int>(pack_sat_u8(r[12], r[13], r[14], r[15])));
  sts128(tile_addr(io, e.slot_out[0], cl), packed);
  if (SHAPE == kShapeAddForkInt && e.slot_out[1] >= 0) sts128(tile_addr(io, e.slot_out[1], cl), packed);
}

// DEPTH: number of PUSH slots the program may use (host-checked)
template <int W, int DEPTH>
__device__ __forceinline__ void run_prog(float (&v)[W], int64_t m, int n0, int nvalid,
                                         const StageTables& t, const TileIo* io = nullptr,
                                         int cl = 0) {
  float s0[W];
  float s1[DEPTH > 1 ? W : 1];
  float s2[DEPTH > 2 ? W : 1];
  int sp = 0;
  const int n_code = t.n_code;
#pragma unroll 1
  for (int pc = 0; pc < n_code; ++pc) {
    const ProgInstr ins = t.code[pc];
    switch (ins.op) {
      case kPSq:
        sq_values<W>(v, t.sq[ins.a]);
        break;
      case kPSqStore8: {
        float q[W];
        sq_codes<W>(v, q, t.sq[ins.a]);
        store_codes<W>(t.buf[ins.b], m, n0, nvalid, q, io, cl);
        break;
      }
      case kPRelu:
#pragma unroll
        for (int j = 0; j < W; ++j) v[j] = (v[j] < 0.0f) ? 0.0f : v[j];
        break;
      case kPClip: {
        const float2 c = t.clip[ins.a];
#pragma unroll
        for (int j = 0; j < W; ++j) v[j] = clampf_ref(v[j], c.x, c.y);
        break;
      }
      case kPAdd: {
        float o[W];
        load_values<W>(t.buf[ins.b], m, n0, nvalid, o, io, cl);
#pragma unroll
        for (int j = 0; j < W; ++j) v[j] = __fadd_rn(v[j], o[j]);
        break;
      }
      case kPStoreF32: {
        const ProgBuf& b = t.buf[ins.b];
        float* dst = static_cast<float*>(b.ptr) + buf_off(b, m, n0);
#pragma unroll
        for (int j = 0; j < W; ++j) {
          if (j < nvalid) dst[j] = v[j];
        }
        break;
      }
      case kPPush:
        if (DEPTH <= 1 || sp == 0) {
#pragma unroll
          for (int j = 0; j < W; ++j) s0[j] = v[j];
        } else if (DEPTH <= 2 || sp == 1) {
#pragma unroll
          for (int j = 0; j < W; ++j) s1[DEPTH > 1 ? j : 0] = v[j];
        } else {
#pragma unroll
          for (int j = 0; j < W; ++j) s2[DEPTH > 2 ? j : 0] = v[j];
        }
        ++sp;
        break;
      case kPPop:
        --sp;
        if (DEPTH <= 1 || sp == 0) {
#pragma unroll
          for (int j = 0; j < W; ++j) v[j] = s0[j];
        } else if (DEPTH <= 2 || sp == 1) {
#pragma unroll
          for (int j = 0; j < W; ++j) v[j] = s1[DEPTH > 1 ? j : 0];
        } else {
#pragma unroll
          for (int j = 0; j < W; ++j) v[j] = s2[DEPTH > 2 ? j : 0];
        }
        break;
      default:
        break;
    }
  }
}

// Integer epilogue of a realized conv/dense output element (IntEpi, fused.h):
// exact int64 zero-point correction + bias, ONE clamp to the accumulator
// dtype (or a trap at the lowest flat index), then the optional fused
// requantize (reference interpreter.cpp:25-37, :238-264, :464-482).  Shared
// by the tcgen05 kernel and the CUDA-core backend.
__device__ __forceinline__ int32_t int_epi_value(const IntEpi& ie, int64_t acc, int o,
                                                 int64_t flat) {
  int64_t v = acc;
  if (ie.wsum) v -= ie.zp0 * static_cast<int64_t>(__ldg(ie.wsum + o));
  if (ie.bias) v += __ldg(ie.bias + o);
  if (v < ie.acc_min || v > ie.acc_max) {
    if (ie.trap) atomicMin(ie.trap, static_cast<unsigned long long>(flat));
    v = v < ie.acc_min ? ie.acc_min : ie.acc_max;
  }
  for (int k = 0; k < ie.n_post; ++k) {
    const IntEpi::Post& pp = ie.post[k];
    if (pp.kind == kPostRelu) {
      v = v > pp.out_zp ? v : pp.out_zp;  // relu int: max(x, zero_point)
      continue;
    }
    if (pp.kind == kPostAdd) {
      v += __ldg(pp.other + flat);  // host-proven inside the add's accumulator range
      continue;
    }
    // requantize: fixed_point_rescale, round half away from zero
    const int64_t p = (v - pp.in_zp) * pp.mult;
    int64_t q = p;
    if (pp.shift > 0) {
      const int64_t nudge = int64_t{1} << (pp.shift - 1);
      q = p >= 0 ? (p + nudge) >> pp.shift : -((-p + nudge) >> pp.shift);
    }
    q += pp.out_zp;
    v = q < pp.q_min ? pp.q_min : (q > pp.q_max ? pp.q_max : q);
  }
  return static_cast<int32_t>(v);
}

}  // namespace quantc::kern
