// Prototype: one CTA computes D[128 x 16] = A[128 x 32] . B[16 x 32]^T with
// tcgen05.mma kind::tf32 (both operands K-major, SWIZZLE_NONE core-matrix
// layout in shared memory), the accumulator in TMEM, read back with
// tcgen05.ld.  Checks the smem / instruction descriptor encodings against a
// CPU reference (inputs are exact in tf32).  Foundation for a tensor-core
// version of the tiled step path (DESIGN.md NEXT-3).
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128, N = 16, K = 32;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major SWIZZLE_NONE: core matrix = 8 rows x 16 B contiguous; SBO = stride of
// 8-row groups, LBO = stride of 16 B K-chunks (both in bytes).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // version (Blackwell)
  return d;                  // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}

__global__ void __launch_bounds__(128) mma_test(const float* A, const float* B, float* D, int swap_lbo_sbo) {
  __shared__ __align__(1024) float sA[M * K];
  __shared__ __align__(1024) float sB[N * K];
  __shared__ __align__(8) unsigned long long bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  auto off = [](int r, int k) { return (r / 8) * 256 + (k / 4) * 32 + (r % 8) * 4 + (k % 4); };   // floats
  for (int i = tid; i < M * K; i += 128) sA[off(i / K, i % K)] = A[i];
  for (int i = tid; i < N * K; i += 128) sB[off(i / K, i % K)] = B[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tmem_base;
  // instruction descriptor: D f32, A/B tf32, K-major both, N>>3, M>>4
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  const uint32_t lbo = swap_lbo_sbo ? 1024 : 128, sbo = swap_lbo_sbo ? 128 : 1024;
  if (tid == 0) {
    for (int kk = 0; kk < K / 8; ++kk) {
      const uint64_t da = smem_desc(su32(sA) + kk * 256, lbo, sbo);
      const uint64_t db = smem_desc(su32(sB) + kk * 256, lbo, sbo);
      const uint32_t acc = kk > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"((uint64_t)su32(&bar)));
  }
  asm volatile(
      "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(
          su32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(tm + ((uint32_t)(32 * warp) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int j = 0; j < N; ++j) D[(32 * warp + lane) * N + j] = __uint_as_float(r[j]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}

int main() {
  std::vector<float> A(M * K), B(N * K), D(M * N);
  unsigned s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (float)((int)(s >> 22) - 512) / 64.f; };   // exact in tf32
  for (auto& x : A) x = rnd();
  for (auto& x : B) x = rnd();
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  for (int swap = 0; swap < 2; ++swap) {
    cudaMemset(dD, 0, D.size() * 4);
    mma_test<<<1, 128>>>(dA, dB, dD, swap);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)A[m * K + k] * B[n * K + k];
        maxerr = fmax(maxerr, fabs(ref - D[m * N + n]));
        maxref = fmax(maxref, fabs(ref));
      }
    printf("swap_lbo_sbo=%d err=%s  max|D-ref| = %.3g (max|ref| %.3g)  D[0]=%g D[17*16+3]=%g\n", swap,
           cudaGetErrorString(e), maxerr, maxref, D[0], D[17 * 16 + 3]);
  }
}
