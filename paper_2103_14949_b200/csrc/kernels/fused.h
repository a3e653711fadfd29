// fused.h — the fused int8 dataflow (engine v2): per-element epilogue
// programs and stage kernels.  Shared by host (fastplan.cpp) and device.
//
// A "program" is the chain of elementwise operators hanging off one
// producing operator (conv/dense GEMM, max-pool, GAP, graph input), applied
// per element in registers: the consumer-edge simulated_quantize nodes, relu
// / clip, a residual add whose other operand is already materialised, and
// identity reshapes (flatten).  Fan-out is expressed with PUSH/POP.  Values
// leave the program as int8 codes (sq outputs feeding MAC/pool/add
// consumers; NHWC rows) or fp32 (boundary values, graph outputs).
//
// Each stage gets a compact StageTables block (its instructions plus only the
// sq parameters / buffers / clip bounds it references, re-indexed locally);
// kernels stage it in shared memory once.
//
// Exactness: the fused engine only runs when every simulated_quantize of
// the graph has a power-of-two scale (engine mode auto) — then
// round(v/s) = roundf(v*2^-j), (q-zp)*s = q*2^j and the accumulator clamp
// compares are exact in fp32 with host-rounded bounds (see FSq), so every
// value equals the reference's double-precision result bit for bit.
#pragma once

#include <cstdint>

#include <vector_types.h>

namespace quantc::kern {

enum ProgOpKind : uint8_t {
  kPEnd = 0,
  kPSq = 1,        // v = sq(v, sq[a])
  kPSqStore8 = 2,  // v = sq(v, sq[a]); buf[b][m,n] = int8(q - zp)
  kPRelu = 3,
  kPClip = 4,      // v = clamp(v, clip[a].x, clip[a].y)
  kPAdd = 5,       // v = v + value(buf[b][m,n])
  kPStoreF32 = 6,  // buf[b][m,n] = v
  kPPush = 7,
  kPPop = 8,
};

struct ProgInstr {
  uint8_t op;
  uint8_t pad0;
  uint16_t a;
  uint32_t b;
};

// Simulated quantize in fp32 (pow2 scale).  Semantics of reference
// simulate.cpp:64-78:
//   v' = has_acc ? clamp((double)v, lo, hi) : v
//   passthrough -> (float)v'
//   q = clamp(round(v'/s) + zp, qmin, qmax);  out = (float)((q - zp) * s)
// lo_up = smallest float >= lo, hi_dn = largest float <= hi, so
// (double)v < lo  <=>  v < lo_up.  A clamped v' (possibly not a float) maps to
// the host-computed codes q_lo / q_hi and floats lo_rn / hi_rn.
struct FSq {
  float lo_up, hi_dn;   // clamp tests
  float lo_rn, hi_rn;   // (float)lo, (float)hi  (passthrough results)
  float q_lo, q_hi;     // code of a clamped value
  float inv_s, s;       // 2^-j, 2^j
  float qmin, qmax, zp;
  int32_t has_acc;
  int32_t passthrough;
  int32_t pad_[3];
};

// A materialised value: element (m, n) lives at
//   base + (m / hw) * ld + (m % hw) * cs + n
// (hw = 1, cs = 0 for plain NHWC rows; hw = H*W, cs = C for a flattened
// [N, H*W*C] dense operand).  kind 0: int8 codes with value (code)*scale;
// kind 1: fp32.
struct ProgBuf {
  void* ptr;
  int64_t ld;
  int32_t hw;
  int32_t cs;
  int32_t kind;
  float scale;
  // GEMM stages: >= 0 routes this buffer through shared-memory tile slot
  // `slot` (TMA store for outputs, TMA-prefetched tile for an add operand)
  int32_t slot;
  int32_t pad_;
};

// shared-memory tile slot geometry of the tcgen05 epilogue: 128 rows x BN
// bytes, stored as BN/S column blocks of S-byte swizzled rows (S = 128 for
// BN >= 128, 64 for BN = 64) — the TMA SWIZZLE_S layout.
#ifdef __CUDACC__
#define QC_HD __host__ __device__
#else
#define QC_HD
#endif
QC_HD inline int slot_swizzle(int bn) { return bn >= 128 ? 128 : 64; }

constexpr int kMaxCode = 48;
constexpr int kMaxSq = 12;
constexpr int kMaxBuf = 8;
constexpr int kMaxClip = 4;

struct StageTables {
  int32_t n_code, n_sq, n_buf, n_clip;
  ProgInstr code[kMaxCode];
  FSq sq[kMaxSq];
  ProgBuf buf[kMaxBuf];
  float2 clip[kMaxClip];
};

// ---- straight-line shape epilogues: host-folded constants -----------------------
// The shape kernels (fused.cuh kShape*) evaluate their sq chain without any
// conversion-pipe instruction.  Codes are carried as floats in one of two
// domains:
//   r-domain: the signed integer code r as a float;
//   T-domain: M + r with M = 1.5*2^23 (bits 0x4B400000 + r), used when r is
//             known >= 0 — its low byte is the int8 code.
// Rounding (reference std::round, half away from zero) of x clamped to
// [qmin - 1/2, qmax + 1/2] (nearest floats inside):
//   T-domain: RZ(RZ(x + 1/2) + M)             (x >= -1/2)
//   r-domain: copysign(RZ(RZ(|x| + 1/2) + M) - M, x)
// RZ(x + 1/2) keeps floor(x + 1/2) exact (integers are representable), and
// RZ(t + M) truncates the fraction on the unit grid of [2^23, 2^24).
constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23

// kEpiNoClamp (with kEpiExact): the host proved k * [qmin_in, qmax_in] lies
// inside [qmin, qmax], so the output-domain clamp is the identity
enum : int32_t { kEpiNonneg = 1, kEpiExact = 2, kEpiNoClamp = 4 };

struct EpiSq {
  float k;    // x = fma(R_in, k, off): input scale ratio s_in / s (sq0: s_x*s_w / s)
  float off;  // domain offset of the input (see fastplan make_epi)
  float lo, hi;   // clamp of x: rounding bounds, or (exact) the output-domain bounds
  int32_t flags;  // kEpiNonneg: output in T-domain; kEpiExact: x already integral
  int32_t pad_;
};

struct EpiConsts {
  EpiSq q[4];       // program-order sq ops of the shape
  float inv0;       // 1 / s of sq0 (bias table and the wide-accumulator path)
  float ka, ka_off; // residual code c (biased magic float C = 2^23 + c + 128):
                    // c * s_res / s_1 = fma(C, ka, ka_off)
  int32_t slot_out[2];
  int32_t slot_res;
  int32_t pad_;
  // shape 5: the fp32 value v = fma(R, f32_s, f32_off) of the last sq, stored
  // to plain rows f32_ptr[m * f32_ld + n]
  float f32_s, f32_off;
  float* f32_ptr;
  int64_t f32_ld;
  int32_t f32_cols;  // shape 9: valid output columns (O)
  int32_t pad2_;
  // shapes 6/7 (saturating rounding, fastplan fold_saturating): sq i's
  // input arrives pre-scaled by 1/P_i (P_i = 2^p: the code range is
  // [-P_i, P_i - 1] or [0, P_i - 1]) so add.rz.sat clamps the low side on the
  // FMA pipe; sat_top caps the high side (one min instead of a clamp pair)
  float sat_half[2];  // 0.5 / P_i
  float sat_p[2];     // P_i
  float sat_top[2];   // highest code (r-domain) or M + highest code (T-domain)
  // integer shapes 10/11 (fastplan fold_integer): the whole chain on the
  // int32 accumulator, no float conversion.
  //   r0 = clamp((acc * i_m0 + ctab[n]) >> i_r0, i_lo0, i_hi0)        (sq0)
  //   y  = clamp((r0 * i_k0 + c * i_kr + i_h1) >> i_r1, 0, i_hi1)     (add + sq1, shape 11)
  // ctab[n] is the channel's bias folded into sq0's grid; the host verified
  // every code breakpoint of every channel against the reference arithmetic.
  // Table layout (int32): C[O], Tp[O], Tn[O], then one bit per 16-channel
  // chunk (ceil(O/512) words) marking chunks with a channel whose breakpoints
  // the fp32 rounding of the conv value moved by one: there
  //   r0 = clamp((acc*i_m0 + C[n] + (acc >= Tp[n]) - (acc < Tn[n])) >> i_r0, ..)
  const int32_t* ctab;
  int32_t i_m0, i_r0, i_lo0, i_hi0;
  int32_t i_k0, i_kr, i_h1, i_r1, i_hi1;
  int32_t i_cs;          // one breakpoint correction in the (scaled) C domain
  int32_t i_mh0, i_mh1;  // 2^(32 - i_r0), 2^(32 - i_r1) (multiply-high form; unused)
};

// Straight-line epilogues for the program shapes that dominate CNN graphs
// (identified on the host after optimise_tables; operand indices are read
// from the stage table).  SHAPE 0 is the generic interpreter below.
//   1: SQ_STORE8
//   2: SQ, SQ_STORE8                          (conv -> sq [-> relu] -> sq -> codes)
//   3: SQ, ADD, SQ, PUSH, SQ_STORE8, POP, SQ_STORE8   (residual block end)
//   4: SQ, ADD, SQ, SQ_STORE8
//   5: SQ, ADD, SQ, STORE_F32                  (residual end -> fp32 for a pool)
// and two flag-specialised forms of the most common constant profiles (host
// checks the folded constants, fastplan make_epi / specialise):
//   6: shape 2 with sq0 non-negative rounding and an identity store (k = 1,
//      exact, no clamp): the T-domain code of sq0 is the stored byte
//   7: shape 3 with sq0 signed rounding, sq1 non-negative rounding and both
//      fork stores identities: one packed code, stored to both slots
//   9: SQ, STORE_F32 (a classifier's dense -> fp32 scores; any O, the last
//      chunk's columns past O are masked)
//   8: integer conv/dense of a realized graph (IntEpi): exact int64 epilogue,
//      accumulator-dtype clamp / trap, optional fused requantize, int32 NCHW out
//  10: shape 6 on the integer accumulator (EpiConsts i_*): sq0 as one
//      multiply-add, one shift and a saturating byte pack
//  11: shape 7 on the integer accumulator: sq0, the residual add and sq1 as
//      exact integer arithmetic on codes (every scale is a power of two)
enum : int { kShapeGeneric = 0, kShapeStore = 1, kShapeSqStore = 2, kShapeAddFork = 3,
             kShapeAdd = 4, kShapeAddF32 = 5, kShapeSqStoreId = 6, kShapeAddForkId = 7,
             kShapeInt = 8, kShapeSqF32 = 9, kShapeSqStoreInt = 10, kShapeAddForkInt = 11,
             kShapeSqStoreAcc = 12, kShapeStoreAcc = 13 };
//  12: shape 2 whose sq0 carries a live accumulator clamp (e.g. the
//      arm_vmlal_like int16 sums): x0 outside the host-scaled bounds q[3].lo /
//      q[3].hi takes the saturation codes q[3].k / q[3].off
QC_HD constexpr bool shape_is_int_fold(int s) {
  return s == kShapeSqStoreInt || s == kShapeAddForkInt;
}

// Integer epilogue (reference interpreter.cpp:238-309 then :464-482):
//   v = acc - zp0 * wsum[o] + bias[o]          (acc = sum_k x'*w', w' = w - zp1)
//   v outside [acc_min, acc_max] -> trap (lowest flat index) or saturate
//   requantize (optional): q = clamp(rescale(v - in_zp) + out_zp, q_min, q_max)
//   y[((img*O + o)*OH + oh)*OW + ow] = v or q   (int32, NCHW like Tensor)
constexpr int kMaxIntPosts = 5;  // e.g. requantize, add, requantize, relu, requantize (parameter block <= 4 KB)
struct IntEpi {
  int32_t* y;
  const int32_t* bias;  // may be null
  const int32_t* wsum;  // sum_k w'[o][k]; may be null when zp0 == 0
  unsigned long long* trap;  // may be null (saturate)
  int64_t zp0, acc_min, acc_max;
  // fused elementwise chain after the accumulator clamp (sole-consumer
  // requantize / relu nodes, reference interpreter.cpp:326-336, :464-482)
  struct Post {
    int16_t kind;   // kPostRequantize, kPostRelu or kPostAdd
    int16_t shift;  // requantize
    int32_t mult;   // requantize (RequantParams::multiplier is int32)
    int32_t in_zp, out_zp, q_min, q_max;  // requantize; relu: out_zp = zero point
    const int32_t* other;  // add: the other operand (same flat indexing as y)
  };
  Post post[kMaxIntPosts];
  int32_t n_post;
  // optional side output: the final values' low bytes as NHWC codes
  // [M][codes_ld] (channels >= O zero) — the next integer conv's packed
  // input, so it skips its pack pass
  uint8_t* codes;
  int32_t codes_ld;
  // 1: every requantize post is multiplier 2^30 with shift >= 30 and every
  // add operand's dtype is <= 16 bits — chunks whose values are < 2^30 run
  // the chain in int32 (kShapeInt epilogue)
  int32_t fast32;
  int32_t OHW;  // output pixels per image (1 for dense)
  int32_t a_unsigned;  // A codes are uint8 (tcgen05 unsigned A)
};
enum : int32_t { kPostRequantize = 1, kPostRelu = 2, kPostAdd = 3 };

// kernels receive the stage's table block in global memory
struct ProgArgs {
  const StageTables* tables;
  int32_t depth;  // PUSH depth of the program
  int32_t shape;  // straight-line epilogue shape (fused.cuh kShape*), 0 = interpreter
};

}  // namespace quantc::kern
