// kernels.h — host launchers of the sm_100a kernels (internal C++ interface
// used by the engine; the public C-ABI over them is include/quantc_cuda.h).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace quantc::kern {

// Simulated-quantize parameters resolved on the host once per node
// (reference simulate.cpp:64-78 with compute_scale/quant_bounds hoisted).
struct SqParams {
  double lo, hi;       // accumulator clamp bounds (valid if has_acc)
  double s;            // scale threshold / 2^(bit-sign)
  double inv_s;        // RN(1/s), fast-path reciprocal
  double qmin, qmax;   // code bounds (as doubles, like the reference clamp)
  double zp;           // zero point as double
  int32_t has_acc;
  int32_t passthrough;
  int32_t exact_div;   // 1 when inv_s is not finite: always divide
  int32_t pad_;
};

// ---- simulated quantize (simquant.cu) ------------------------------------
void sim_quant(const float* x, float* y, int64_t n, const SqParams& p, cudaStream_t s);
// also emit integer codes (q - zp) as int8 in NHWC order for a tcgen05 GEMM:
// x is NCHW [N,C,H,W] (H=W=1 for dense rows); codes [N,H,W,Cpad] with zero
// padding for channels >= C.
void sim_quant_codes_nhwc(const float* x, float* y, int8_t* codes, int N, int C, int H, int W,
                          int Cpad, const SqParams& p, cudaStream_t s);

// ---- statistics (stats.cu) -------------------------------------------------
// d_minmax: 2 uint64 order keys per slot (min key, max key), pre-initialised.
void minmax_init(unsigned long long* keys, int n_slots, cudaStream_t s);
void minmax_accumulate(const float* x, int64_t n, unsigned long long* keys2, cudaStream_t s);
void minmax_decode(const unsigned long long* keys, double* out, int n_slots, cudaStream_t s);
// histogram of |x| against absmax (reference calibration.cpp:28-33,97-105);
// counts are uint64 accumulated (multiplier applied per element count).
void histogram_accumulate(const float* x, int64_t n, double absmax, int bins,
                          unsigned long long* counts, unsigned long long multiplier,
                          cudaStream_t s);

// ---- KL sweep (kl.cu) --------------------------------------------------------
// counts: [n_edges][bins] int64; outputs best index i (bins units) and its KL.
void kl_sweep(const int64_t* counts, int n_edges, int bins, int target_bit, int* best_i,
              double* best_kl, cudaStream_t s);

// ---- exact fp32 conv/dense with sequential FP64 accumulation (conv_f64.cu) --
struct ConvShape {
  int N, C, H, W, O, KH, KW, OH, OW, sh, sw, ph, pw;
  // groups (0 or 1: a dense conv).  C and O are the totals; the weight is
  // [O][C/G][KH][KW] and output channel o reads input channels
  // [(o / (O/G)) * C/G, ... + C/G).  Op-set extension.
  int G;
};
__host__ __device__ inline int conv_groups(const ConvShape& cs) { return cs.G > 1 ? cs.G : 1; }
void conv2d_f64acc(const float* x, const float* w, const float* bias, float* y,
                   const ConvShape& cs, cudaStream_t s);

// ---- elementwise / pooling / reductions (eltwise.cu) -------------------------
void add_f32(const float* a, int64_t na, const float* b, int64_t nb, float* y, int64_t n,
             cudaStream_t s);  // na/nb: operand extents (broadcast by modulo)
void relu_f32(const float* x, float* y, int64_t n, cudaStream_t s);
void clip_f32(const float* x, float* y, int64_t n, float lo, float hi, cudaStream_t s);
void maxpool_f32(const float* x, float* y, int N, int C, int H, int W, int OH, int OW, int kh,
                 int kw, int sh, int sw, int ph, int pw, cudaStream_t s);
// op-set extension: avg_pool2d (double sum of x * fl32(1/(kh*kw)), padded taps
// skipped, count_include_pad divisor) and one input of a channel concat
void avgpool_f32(const float* x, float* y, int N, int C, int H, int W, int OH, int OW, int kh,
                 int kw, int sh, int sw, int ph, int pw, cudaStream_t s);
void concat_words(const void* x, void* y, int N, int64_t inner, int64_t outer, int64_t off,
                  cudaStream_t s);
void gap_f32(const float* x, float* y, int NC, int HW, cudaStream_t s);
void argmax_rows(const float* x, int rows, int64_t cols, int64_t* out, cudaStream_t s);
// grouped candidate evaluation: argmax of `groups` (<= 4) row blocks in one
// launch, and counts[g] += #{i : a[g*n + i] == b[i]}
void argmax_rows_multi(const float* const* xs, int64_t* const* outs, int groups, int rows,
                       int64_t cols, cudaStream_t s);
void count_equal_multi(const int64_t* a, const int64_t* b, int n, int groups,
                       unsigned long long* counts, cudaStream_t s);
void count_equal(const int64_t* a, const int64_t* b, int n, unsigned long long* count,
                 cudaStream_t s);

// ---- integer regime (intops.cu) ------------------------------------------------
// int32 storage (reference tensor.hpp:15-17); exact int64 accumulation.
// trap_flat: when non-null, overflowing elements atomicMin their flat index there.
void conv2d_int(const int32_t* x, const int32_t* w, const int32_t* bias, int32_t* y,
                const ConvShape& cs, int64_t zp0, int64_t zp1, int64_t acc_min, int64_t acc_max,
                unsigned long long* trap_flat, cudaStream_t s);
int64_t conv2d_int_value_at(const int32_t* x, const int32_t* w, const int32_t* bias,
                            const ConvShape& cs, int64_t zp0, int64_t zp1, int64_t flat,
                            cudaStream_t s);
void add_int(const int32_t* a, int64_t na, const int32_t* b, int64_t nb, int32_t* y, int64_t n,
             int64_t acc_min, int64_t acc_max, unsigned long long* trap_flat, cudaStream_t s);
void relu_int(const int32_t* x, int32_t* y, int64_t n, int32_t zp, cudaStream_t s);
void clip_int(const int32_t* x, int32_t* y, int64_t n, int32_t lo, int32_t hi, cudaStream_t s);
void maxpool_int(const int32_t* x, int32_t* y, int N, int C, int H, int W, int OH, int OW,
                 int kh, int kw, int sh, int sw, int ph, int pw, cudaStream_t s);
void quantize_f32_int(const float* x, int32_t* y, int64_t n, double scale, int64_t zp,
                      int64_t qmin, int64_t qmax, cudaStream_t s);
void dequantize_int_f32(const int32_t* x, float* y, int64_t n, double scale, int64_t zp,
                        cudaStream_t s);
void requantize_int(const int32_t* x, int32_t* y, int64_t n, int64_t mult, int shift,
                    int64_t in_zp, int64_t out_zp, int64_t qmin, int64_t qmax, cudaStream_t s);

// ---- tcgen05 int8 GEMM (gemm_tcgen05.cu) -----------------------------------------
// C[M,N] (int32 accumulators, consumed by the epilogue) = A[M,K] * B[N,K]^T,
// A/B int8 K-major, K a multiple of 128 (zero padded).  Epilogue: y (NCHW
// float, M rows = (img, oh, ow), N = channels) = float(acc * scale + bias[n]).
struct GemmEpilogue {
  float* y;          // output, NCHW
  const float* bias; // may be null
  double scale;      // s_x * s_w
  int OHW;           // pixels per image (OH*OW); 1 for dense
};
bool gemm_s8_tcgen05_available();
void gemm_s8_tcgen05(const int8_t* A, const int8_t* B, int M, int N, int K,
                     const GemmEpilogue& ep, cudaStream_t s);
// im2col of NHWC int8 codes into [M, Kpad] rows (k order = (kh, kw, c))
void im2col_s8(const int8_t* x, int8_t* out, int N, int H, int W, int Cpad, int KH, int KW,
               int OH, int OW, int sh, int sw, int ph, int pw, int Kpad, cudaStream_t s);
// weights [O][C][KH][KW] float (already sim-quantized) -> codes [O][Kpad] in
// (kh, kw, c) order with the same code convention.
void weights_to_codes(const float* w, int8_t* codes, int O, int C, int KH, int KW, int Cpad,
                      int Kpad, const SqParams& p, cudaStream_t s);

// ---- engine v2: fused int8 dataflow (conv_tc.cu, stages.cu) ------------------
}  // namespace quantc::kern
#include "fused.h"
namespace quantc::kern {

// problems of one layer a grouped tcgen05 launch can carry (TcConvSpec.groups)
constexpr int kMaxGroups = 4;

struct TcConvSpec {
  const int8_t* x;   // A source: NHWC codes (gather) or code rows (direct)
  const int8_t* w;   // B: weight codes [O][Kpad]
  int64_t M;         // output rows (pixels / samples)
  int O;             // output channels
  int Kpad;          // multiple of 128
  int gather;        // 1: implicit im2col gather, 0: direct TMA rows
  int Ktrue, lda;    // direct: valid K bytes per row, row stride
  int Nimg, H, W, C, ld, KH, KW, sh, sw, ph, pw, OH, OW;  // gather geometry
  int ldk;           // weight K stride of one tap (0: ld); 128 for 64-channel 2-D band convs
  const float* bias;
  double scale;      // s_x * s_w
  ProgArgs prog;
  // smem-staged epilogue I/O (ProgBuf::slot): code outputs stored by TMA
  // (slots 0..n_out-1) and one TMA-prefetched add operand (slot n_out)
  int n_out;
  void* out_ptr[2];
  int out_cols[2];
  int64_t out_ld[2];
  const void* res_ptr;
  int res_cols;
  int64_t res_ld;
  // 1: the add operand is prefetched into output slot 0 itself (no slot of
  // its own: each epilogue thread reads its residual bytes, then overwrites
  // them with its output codes); the store warp drains a set's stores before
  // it prefetches the next residual into it
  int res_alias;
  double acc_bound;  // host bound on |sum_k a*b| (K * max|qa| * max|qb|)
  // device bound on |sum_k a*b|: max_o sum_k |w_code[o][k]| (weight_l1_max),
  // times the input codes' max |q|; <= 2^24 lets the epilogue convert with I2F
  const int* w_l1;
  int x_absmax;
  EpiConsts epi;     // shape kernels (prog.shape != 0): host-folded constants
  IntEpi iepi;       // prog.shape == kShapeInt: integer epilogue
  // groups > 1: further problems of the same layer in the same launch (shape
  // kernels; same geometry, shape and output layout, their own operands and
  // constants), group g's tiles after group g-1's in the schedule.  Entry
  // [g-1] of the arrays below is group g.
  int groups;
  const int8_t* xg[kMaxGroups - 1];
  const int8_t* wg[kMaxGroups - 1];
  const int* w_l1g[kMaxGroups - 1];
  int x_absmaxg[kMaxGroups - 1];
  double scaleg[kMaxGroups - 1];
  void* out_ptrg[kMaxGroups - 1][2];
  const void* res_ptrg[kMaxGroups - 1];
  EpiConsts epig[kMaxGroups - 1];
};
void tc_conv(const TcConvSpec& spec, cudaStream_t s);

// CUDA-core integer conv/dense backend (conv_simt.cu): int16 codes or the
// int16-accumulator signature; dp4a / 16-bit products, fused IntEpi epilogue
struct SimtConvSpec {
  const uint32_t* x;  // [N][HP][WP][Cw] words (pack_words)
  const uint32_t* w;  // [KH*KW*Cw][O] words (pack_weight_words)
  int N, HP, WP, Cw, O, KH, KW, sh, sw, OH, OW;
  bool i16, u8;
  IntEpi ie;
};
void conv_int_simt(const SimtConvSpec& spec, cudaStream_t s);
// int32 NCHW values -> NHWC words (4 x 8-bit or 2 x 16-bit channels), the
// ph/pw border filled with `fill`
void pack_words(const int32_t* x, uint32_t* out, int N, int C, int H, int W, int ph, int pw,
                int Cw, bool i16, int32_t fill, cudaStream_t s);
// OIHW int32 weights -> words [taps*Cw][O] of w - zp1, wsum[o] += sum w';
// *bad != 0 when some w - zp1 leaves the 8/16-bit range
void pack_weight_words(const int32_t* w, uint32_t* out, int32_t* wsum, int* bad, int O, int C,
                       int taps, int Cw, bool i16, int64_t zp1, cudaStream_t s);
int tc_conv_bn(int O);  // output-channel tile the kernel uses for O channels

// weight codes [O][Kpad], k = tap*ldk + c, from OIHW float weights (taps =
// KH*KW; a flattened dense is the taps = H*W case), fp32 sq (pow2 scale)
void weight_codes_v2(const float* w, int8_t* codes, int O, int C, int taps, int ldk, int Kpad,
                     const FSq& p, cudaStream_t s);
// graph input NCHW fp32 [N, C, H, W] -> space-to-depth int8 codes
// [N, ceil(H/2), ceil(W/2), 16], channel ((h%2)*2 + w%2)*C + c (C <= 4)
void stage_input_s2d(const float* x, int N, int C, int H, int W, const FSq& p, int8_t* out,
                     cudaStream_t s);
// the same images under up to four bindings (grouped evaluation): one read,
// one space-to-depth code image per binding
void stage_input_s2d_multi(const float* x, int N, int C, int H, int W, const FSq* ps,
                           int8_t* const* outs, int groups, cudaStream_t s);
// weight codes [O][Kpad] of the space-to-depth form of a stride-2 KHxKW conv
// (KH2 x KW2 taps of 16 channels; original tap = 2*ka + dy - dh, 2*kb + dx - dw)
void weight_codes_s2d(const float* w, int8_t* codes, int O, int C, int KH, int KW, int KH2,
                      int KW2, int dh, int dw, int Kpad, const FSq& p, cudaStream_t s);
// out = max over rows of sum_k |codes[o][k]| (out zeroed by the caller)
void weight_l1_max(const int8_t* codes, int O, int Kpad, int* out, cudaStream_t s);
// realized-graph integer path: int32 NCHW values (int8 / uint8 range) -> 8-bit
// NHWC rows [N][H+2ph][W+2pw][ld] (channels >= C zero, the ph/pw border
// `fill`); dense: H = W = 1
void pack_i32_nhwc(const int32_t* x, uint8_t* out, int N, int C, int H, int W, int ph, int pw,
                   int ld, int32_t fill, cudaStream_t s);
// int32 OIHW weights -> int8 [O][Kpad] (k = tap*ld + c) of w - zp1, and
// wsum[o] = sum of those codes; *bad != 0 when some w - zp1 leaves int8
void pack_i32_weights(const int32_t* w, int8_t* codes, int32_t* wsum, int* bad, int O, int C,
                      int taps, int ld, int Kpad, int64_t zp1, cudaStream_t s);
// graph input NCHW fp32 -> program over (m = n*H*W + hw, c)
void stage_input(const float* x, int N, int C, int HW, const ProgArgs& prog, cudaStream_t s);
// max_pool2d over NHWC codes (value = code * scale) -> program
// average pool (zero padding counted) of fp32 NHWC rows with the stage
// program (fused engine; the exact engine's double arithmetic, wk = fl32(1/(kh*kw)))
struct DwFast;
void stage_avgpool_f32(const float* x, int ld, int N, int C, int H, int W, int OH, int OW, int kh,
                       int kw, int sh, int sw, int ph, int pw, double wk, const ProgArgs& prog,
                       const DwFast& fast, cudaStream_t s);
// depthwise conv (groups == C == O) of int8 codes with the stage program
// (fused engine; weights as tap quads [ceil(taps/4)][ldw] from dw_weight_quads)
// n > 0: the stage program is [passthrough accumulator sq fa (n == 2),]
// sq_store8 fs -> buf, run without the table interpreter
struct DwFast {
  int32_t n;
  int32_t pad_;
  FSq fa, fs;
  ProgBuf buf;
};
void stage_dw_conv(const int8_t* x, int ld, int N, int C, int H, int W, int KH, int KW, int sh,
                   int sw, int ph, int pw, int OH, int OW, const int32_t* wquads, int ldw,
                   const float* bias, float scale, const ProgArgs& prog, const DwFast& fast,
                   cudaStream_t s);
void dw_weight_quads(const int8_t* codes, int taps, int ldw, int32_t* quads, cudaStream_t s);
void stage_maxpool(const int8_t* x, int ld, float scale, int N, int C, int H, int W, int OH,
                   int OW, int kh, int kw, int sh, int sw, int ph, int pw, const ProgArgs& prog,
                   cudaStream_t s);
// global_avg_pool2d over NHWC values (fp32 rows, ld) -> program over (n, c)
void stage_gap(const float* x, int64_t ld, int N, int C, int HW, const ProgArgs& prog,
               cudaStream_t s);
// dense im2col rows of NHWC codes for tiny-channel convs: out[m][k] with
// k = (kh*KW + kw)*C + c for k < Ktrue, 0 up to Kpad
void pack_im2col(const int8_t* x, int8_t* out, int N, int H, int W, int C, int ld, int KH, int KW,
                 int sh, int sw, int ph, int pw, int OH, int OW, int Ktrue, int Kpad,
                 cudaStream_t s);
// max-pool whose program is only code stores (<= 2, e.g. a fork to two
// convs): per store the host-folded EpiSq of code -> code and a plain NHWC
// destination (fused.h EpiSq)
struct PoolStores {
  EpiSq q[2];
  int8_t* out[2];
  int64_t ld[2];
  int n_out;
};
void stage_maxpool_stores(const int8_t* x, int ld, int N, int C, int H, int W, int OH, int OW,
                          int kh, int kw, int sh, int sw, int ph, int pw, const PoolStores& e,
                          cudaStream_t s);
// generic elementwise stage over an (M, C) space: v = value(src) -> program
void stage_ew(const ProgBuf& src, int64_t M, int C, const ProgArgs& prog, cudaStream_t s);

}  // namespace quantc::kern
