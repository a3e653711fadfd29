// Probe: can a tcgen05 K-major SWIZZLE_128B operand start at a row offset
// that is not a multiple of the 8-row (1024 B) swizzle atom?  A is a
// 256x128 B int8 tile written in the TMA SW128 image (16-byte chunk c of row r
// at r*128 + ((c ^ (r & 7)) * 16)); the MMA reads rows shift..shift+127 with
// the descriptor's base-offset field set per `mode`.  D is checked on the host.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t base_off) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (1ull << 16) | (static_cast<uint64_t>(1024 >> 4) << 32) |
         (1ull << 46) | (static_cast<uint64_t>(base_off & 7) << 49) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc(int m, int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}

__global__ void probe(const int8_t* A, const int8_t* B, int32_t* D, int shift, int mode) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = sm;               // 256 rows x 128 B
  uint8_t* sb = sm + 256 * 128;   // 64 rows x 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 256 * 8; i += blockDim.x) {
    const int r = i / 8, c = i % 8;
    *reinterpret_cast<int4*>(sa + r * 128 + ((c ^ (r & 7)) * 16)) = *reinterpret_cast<const int4*>(A + r * 128 + c * 16);
  }
  for (int i = threadIdx.x; i < 64 * 8; i += blockDim.x) {
    const int r = i / 8, c = i % 8;
    *reinterpret_cast<int4*>(sb + r * 128 + ((c ^ (r & 7)) * 16)) = *reinterpret_cast<const int4*>(B + r * 128 + c * 16);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t a_addr = su32(sa) + shift * 128;
    const uint32_t bo = mode == 0 ? 0u : ((a_addr >> 7) & 7);
    const uint64_t a0 = desc_sw128(a_addr, bo), b0 = desc_sw128(su32(sb), 0);
    for (int k = 0; k < 4; ++k) {
      const uint32_t acc = k ? 1u : 0u;
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(tmem), "l"(a0 + 2 * k), "l"(b0 + 2 * k), "r"(idesc(128, 64)), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int c0 = 0; c0 < 64; c0 += 16) {
    uint32_t d[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
                   "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
                 : "r"(tmem + (static_cast<uint32_t>(w * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 16; ++j) D[(w * 32 + lane) * 64 + c0 + j] = static_cast<int32_t>(d[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

int main() {
  std::vector<int8_t> A(256 * 128), B(64 * 128);
  srand(1);
  for (auto& v : A) v = static_cast<int8_t>(rand() % 7 - 3);
  for (auto& v : B) v = static_cast<int8_t>(rand() % 7 - 3);
  int8_t *dA, *dB;
  int32_t* dD;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dD, 128 * 64 * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int mode = 0; mode < 2; ++mode) {
    for (int shift : {0, 1, 2, 3, 5, 8, 9}) {
      probe<<<1, 128, 48 * 1024>>>(dA, dB, dD, shift, mode);
      std::vector<int32_t> D(128 * 64);
      cudaError_t e = cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
      int bad = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 64; ++n) {
          int32_t ref = 0;
          for (int k = 0; k < 128; ++k) ref += A[(m + shift) * 128 + k] * B[n * 128 + k];
          bad += ref != D[m * 64 + n];
        }
      printf("mode %d (base_offset %s) shift %d rows: %s (%d / 8192 wrong)\n", mode,
             mode ? "(addr>>7)&7" : "0", shift, bad ? "MISMATCH" : "ok", bad);
    }
  }
  return 0;
}
