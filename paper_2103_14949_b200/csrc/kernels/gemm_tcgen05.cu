// gemm_tcgen05.cu — int8 x int8 -> int32 GEMM on the 5th-generation tensor
// cores (tcgen05.mma kind::i8), operands staged by TMA, accumulators in TMEM,
// with the conv/dense epilogue of the simulated-quantized graph fused in.
//
// Role of this kernel (SURVEY.md §2 K4, §7 "Fast int8 path vs parity"):
// a conv2d/dense whose data and weight inputs are simulated_quantize outputs
// computes  sum_k x_k*w_k  =  s_x*s_w * sum_k q_x,k*q_w,k  when x = q_x*s_x and
// w = q_w*s_w are exact (power-of-two thresholds).  Every partial sum of the
// reference's sequential double accumulation (interpreter.cpp:222-233) is then
// an exact multiple of s_x*s_w below 2^53, so the int32 tensor-core sum scaled
// by s_x*s_w IS the reference's double accumulator, bit for bit; the epilogue
// adds the bias in double and rounds to float exactly like the reference.
//
// Structure (one 128 x BN output tile per CTA, 128 threads):
//   warp 0 / lane 0 : TMA producer, S-stage ring of {A 128x128B, B BNx128B}
//                     tiles (SWIZZLE_128B, K-major), mbarrier full/empty;
//   warp 1 / lane 0 : MMA issuer, 4 x tcgen05.mma (K=32 each) per stage,
//                     tcgen05.commit -> empty[s]; final commit -> done;
//   warps 0-3       : epilogue, tcgen05.ld 32x32b (warp w owns TMEM lanes
//                     32w..32w+31 = output rows), y = float(acc*s + bias).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <mutex>
#include <stdexcept>

#include "common.cuh"

namespace quantc::kern {

namespace {

constexpr int BM = 128;
constexpr int BK = 128;  // bytes of K per stage (int8 elements)
constexpr int UMMA_K = 32;
constexpr int STAGES = 4;
constexpr int THREADS = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row atoms of 128 B
// (SBO = 1024 B), sm100 descriptor version 1.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);           // start address
  d |= static_cast<uint64_t>(1) << 16;                          // LBO (unused for SW128 K-major)
  d |= static_cast<uint64_t>((1024 >> 4) & 0x3FFF) << 32;       // SBO
  d |= static_cast<uint64_t>(1) << 46;                          // version = 1 (sm100)
  d |= static_cast<uint64_t>(2) << 61;                          // layout = SWIZZLE_128B
  return d;
}

// Instruction descriptor kind::i8: D s32, A s8, B s8, both K-major, M, N.
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
  return (2u << 4)                                 // c_format = S32
         | (1u << 7)                               // a_format = signed int8
         | (1u << 10)                              // b_format = signed int8
         | (static_cast<uint32_t>(n >> 3) << 17)   // N >> 3
         | (static_cast<uint32_t>(m >> 4) << 24);  // M >> 4
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

template <int BN>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_s8_kernel(const __grid_constant__ CUtensorMap map_a,
                   const __grid_constant__ CUtensorMap map_b, int M, int N, int K,
                   GemmEpilogue ep) {
  constexpr uint32_t A_BYTES = BM * BK;
  constexpr uint32_t B_BYTES = BN * BK;
  constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-align the carve-out (SW128 atoms)
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  const int nk = K / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---- TMA producer ----
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      if (kb >= STAGES) mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
      mbar_expect_tx(&full[s], A_BYTES + B_BYTES);
      tma_load_2d(&map_a, &full[s], sa + s * A_BYTES, kb * BK, m0);
      tma_load_2d(&map_b, &full[s], sb + s * B_BYTES, kb * BK, n0);
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer ----
    constexpr uint32_t idesc = idesc_i8(BM, BN);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&full[s], (kb / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a_base = smem_u32(sa + s * A_BYTES);
      const uint32_t b_base = smem_u32(sb + s * B_BYTES);
#pragma unroll
      for (int k = 0; k < BK / UMMA_K; ++k) {
        mma_i8(tmem, umma_desc_sw128(a_base + k * UMMA_K), umma_desc_sw128(b_base + k * UMMA_K),
               idesc, (kb | k) != 0 ? 1u : 0u);
      }
      umma_commit(&empty[s]);
    }
    umma_commit(done);
  }
  __syncwarp();

  // ---- epilogue: TMEM -> registers -> y (NCHW float) ----
  mbar_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = m0 + warp * 32 + lane;  // TMEM lane == tile row
  const bool row_ok = row < M;
  int64_t img = 0, pix = 0;
  if (row_ok) {
    img = row / ep.OHW;
    pix = row % ep.OHW;
  }
  const uint32_t lane_base = tmem + (static_cast<uint32_t>(warp * 32) << 16);
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 16) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(lane_base + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (row_ok) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int n = n0 + c0 + j;
        if (n < N) {
          double v = __dmul_rn(static_cast<double>(static_cast<int32_t>(r[j])), ep.scale);
          if (ep.bias) v = __dadd_rn(v, static_cast<double>(__ldg(ep.bias + n)));
          ep.y[(img * N + n) * ep.OHW + pix] = __double2float_rn(v);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS));
  }
}

// ---- im2col of NHWC codes -------------------------------------------------------
__global__ void im2col_kernel(const int8_t* __restrict__ x, int8_t* __restrict__ out, int N,
                              int H, int W, int Cpad, int KH, int KW, int OH, int OW, int sh,
                              int sw, int ph, int pw, int Kpad) {
  const int chunks_per_row = Kpad / 16;
  const int cchunks = Cpad / 16;
  const int64_t total = static_cast<int64_t>(N) * OH * OW * chunks_per_row;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int ch = static_cast<int>(i % chunks_per_row);
    const int64_t m = i / chunks_per_row;
    int4 v = make_int4(0, 0, 0, 0);
    const int tap = ch / cchunks;
    if (tap < KH * KW) {
      const int cc = ch - tap * cchunks;
      const int kh = tap / KW, kw = tap % KW;
      const int ow = static_cast<int>(m % OW);
      const int oh = static_cast<int>((m / OW) % OH);
      const int64_t n = m / (static_cast<int64_t>(OW) * OH);
      const int ih = oh * sh - ph + kh, iw = ow * sw - pw + kw;
      if (ih >= 0 && ih < H && iw >= 0 && iw < W) {
        v = *reinterpret_cast<const int4*>(x + ((n * H + ih) * W + iw) * Cpad + cc * 16);
      }
    }
    *reinterpret_cast<int4*>(out + m * Kpad + ch * 16) = v;
  }
}

__global__ void weights_codes_kernel(const float* __restrict__ w, int8_t* __restrict__ codes,
                                     int O, int C, int KH, int KW, int Cpad, int Kpad,
                                     SqParams p) {
  const int64_t total = static_cast<int64_t>(O) * Kpad;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(i % Kpad);
    const int o = static_cast<int>(i / Kpad);
    int8_t code = 0;
    const int tap = k / Cpad, c = k % Cpad;
    if (tap < KH * KW && c < C) {
      const int kh = tap / KW, kw = tap % KW;
      double v = static_cast<double>(w[((static_cast<int64_t>(o) * C + c) * KH + kh) * KW + kw]);
      if (p.has_acc) v = clampd(v, p.lo, p.hi);
      code = static_cast<int8_t>(static_cast<int>(__dsub_rn(sq_code(v, p), p.zp)));
    }
    codes[i] = code;
  }
}

// ---- host side --------------------------------------------------------------------
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
  static EncodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      return static_cast<EncodeTiled>(nullptr);
    }
    return reinterpret_cast<EncodeTiled>(p);
  }();
  return fn;
}

CUtensorMap make_map(const int8_t* base, int rows, int K, int box_rows) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(K)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed");
  return m;
}

template <int BN>
void launch_gemm(const int8_t* A, const int8_t* B, int M, int N, int K, const GemmEpilogue& ep,
                 cudaStream_t s) {
  const size_t smem = 1024 + STAGES * (BM * BK + BN * BK) + 256;
  static std::once_flag once;
  std::call_once(once, [&] {
    cudaFuncSetAttribute(gemm_s8_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
  });
  CUtensorMap ma = make_map(A, M, K, BM);
  CUtensorMap mb = make_map(B, N, K, BN);
  dim3 grid((M + BM - 1) / BM, (N + BN - 1) / BN);
  gemm_s8_kernel<BN><<<grid, THREADS, smem, s>>>(ma, mb, M, N, K, ep);
  QC_CUDA_CHECK_LAUNCH();
}

}  // namespace

bool gemm_s8_tcgen05_available() {
  static int ok = -1;
  if (ok < 0) {
    int dev = 0, major = 0, minor = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    ok = (major == 10 && minor == 0 && encode_fn() != nullptr) ? 1 : 0;
  }
  return ok == 1;
}

void gemm_s8_tcgen05(const int8_t* A, const int8_t* B, int M, int N, int K,
                     const GemmEpilogue& ep, cudaStream_t s) {
  if (K % BK != 0) throw std::runtime_error("gemm_s8_tcgen05: K must be a multiple of 128");
  if (M <= 0 || N <= 0) return;
  if (N <= 64) {
    launch_gemm<64>(A, B, M, N, K, ep, s);
  } else if (N <= 128 || (static_cast<int64_t>(M + BM - 1) / BM) * ((N + 255) / 256) < 148) {
    launch_gemm<128>(A, B, M, N, K, ep, s);
  } else {
    launch_gemm<256>(A, B, M, N, K, ep, s);
  }
}

void im2col_s8(const int8_t* x, int8_t* out, int N, int H, int W, int Cpad, int KH, int KW,
               int OH, int OW, int sh, int sw, int ph, int pw, int Kpad, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(N) * OH * OW * (Kpad / 16);
  if (total <= 0) return;
  im2col_kernel<<<grid_for(total, 256), 256, 0, s>>>(x, out, N, H, W, Cpad, KH, KW, OH, OW, sh,
                                                     sw, ph, pw, Kpad);
  QC_CUDA_CHECK_LAUNCH();
}

void weights_to_codes(const float* w, int8_t* codes, int O, int C, int KH, int KW, int Cpad,
                      int Kpad, const SqParams& p, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(O) * Kpad;
  if (total <= 0) return;
  weights_codes_kernel<<<grid_for(total, 256), 256, 0, s>>>(w, codes, O, C, KH, KW, Cpad, Kpad, p);
  QC_CUDA_CHECK_LAUNCH();
}

}  // namespace quantc::kern
