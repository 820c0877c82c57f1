// Microbenchmark: gather K random 256 B rows into smem per CTA (148 CTAs x 384
// threads): per-row cp.async.bulk vs cp.async 16 B vs LDG.128+STS.  Reports the
// median per-CTA cycles (clock64 from first issue to data-ready + bar.sync).
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
template <int MODE, int W1>
__global__ void __launch_bounds__(384, 1) k(const float* C, const int* rows, int K, long long* out, float* sink, const float* Wg) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar;
  __shared__ int rs[512];
  float* X = reinterpret_cast<float*>(sm);
  const int tid = threadIdx.x;
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  for (int i = tid; i < K; i += blockDim.x) rs[i] = rows[blockIdx.x * K + i];
  __syncthreads();
  long long t0 = clock64();
  float* Wsm = reinterpret_cast<float*>(sm + 100 * 1024);
  if (W1 && tid == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(40960 + (MODE == 0 ? K * 256 : 0)) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 40960, [%2];"
                 ::"r"(su32(Wsm)), "l"(Wg), "r"(su32(&bar)) : "memory");
  }
  if (MODE == 0) {
    if (tid == 0 && !W1) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(K * 256) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int i = tid; i < K; i += blockDim.x)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];"
                   ::"r"(su32(X + i * 64)), "l"(C + (size_t)rs[i] * 64), "r"(su32(&bar)) : "memory");
  } else if (MODE == 1) {
    for (int it = tid; it < K * 16; it += blockDim.x) {
      const int i = it >> 4, q = it & 15;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(X + i * 64 + 4 * q)), "l"(C + (size_t)rs[i] * 64 + 4 * q) : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else {
    float4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int it = tid + j * 384;
      if (it < K * 16) v[j] = __ldcg(reinterpret_cast<const float4*>(C + (size_t)rs[it >> 4] * 64) + (it & 15));
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int it = tid + j * 384;
      if (it < K * 16) reinterpret_cast<float4*>(X)[it] = v[j];
    }
  }
  if (MODE == 0 || W1)
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(su32(&bar)) : "memory");
  __syncthreads();
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
  if (X[tid * 7 % (K * 64)] == 12345.f) sink[0] = 1.f;
}
int main() {
  const int V = 100000, d = 64, G = 148;
  float* C; int* rows; long long* out; float* sink; float* fl;
  cudaMalloc(&C, (size_t)V * d * 4); cudaMemset(C, 0, (size_t)V * d * 4);
  cudaMalloc(&rows, G * 512 * 4); cudaMalloc(&out, G * 8); cudaMalloc(&sink, 4);
  cudaMalloc(&fl, 512u << 20);
  std::vector<int> hr(G * 512);
  unsigned s = 1; for (auto& r : hr) { s = s * 1664525u + 1013904223u; r = (s >> 8) % V; }
  cudaMemcpy(rows, hr.data(), hr.size() * 4, cudaMemcpyHostToDevice);
  auto run = [&](auto kern, int K, const char* nm, bool flush) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    std::vector<long long> all;
    for (int rep = 0; rep < 6; ++rep) {
      if (flush) cudaMemset(fl, rep, 512u << 20);
      kern<<<G, 384, 160 * 1024>>>(C, rows, K, out, sink, C + 12345 * 64);
      cudaDeviceSynchronize();
      std::vector<long long> h(G); cudaMemcpy(h.data(), out, G * 8, cudaMemcpyDeviceToHost);
      if (rep >= 1) all.insert(all.end(), h.begin(), h.end());
    }
    std::sort(all.begin(), all.end());
    printf("%-10s K=%3d flush=%d  cycles med %6lld  p90 %6lld  max %6lld\n", nm, K, flush, all[all.size() / 2], all[all.size() * 9 / 10], all.back());
  };
  for (int K : {32, 168})
    for (bool f : {false, true}) {
      run(k<0, 0>, K, "bulk/row", f);
      run(k<1, 0>, K, "cp.async16", f);
      run(k<2, 0>, K, "ldg+sts", f);
      run(k<0, 1>, K, "bulk+W1", f);
      run(k<1, 1>, K, "cpa16+W1", f);
      run(k<2, 1>, K, "ldg+W1", f);
    }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
