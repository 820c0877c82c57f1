// Microbenchmark: achievable DRAM bandwidth for reading 1M rows of 256 B
// (256 MB) in (a) sequential and (b) random row order, with (1) lane-group
// float4 loads, U rows in flight per lane group, and (2) TMA bulk copies
// (cp.async.bulk, 256 B per row) into an smem ring.  L2 flushed before each run.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
template <int U>
__global__ void __launch_bounds__(1024, 1) rd_lg(const float4* __restrict__ Y, const int* __restrict__ perm, int n, float* sink) {
  const int lane = threadIdx.x & 15;
  const int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 4, ng = (gridDim.x * blockDim.x) >> 4;
  // contiguous share of the (permuted) row sequence per lane group
  const int per = (n + ng - 1) / ng, lo = g * per, hi = min(n, lo + per);
  float4 acc = make_float4(0, 0, 0, 0);
  for (int r0 = lo; r0 < hi; r0 += U) {
    float4 v[U];
    int row[U];
#pragma unroll
    for (int u = 0; u < U; ++u) row[u] = r0 + u < hi ? (perm ? __ldg(perm + r0 + u) : r0 + u) : -1;
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = row[u] >= 0 ? __ldcs(Y + (size_t)row[u] * 16 + lane) : make_float4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
  }
  if (acc.x == 1234.5f) sink[0] = acc.y + acc.z + acc.w;
}
// TMA: one CTA per SM, NB stages of R rows; thread 0 issues, all threads consume
template <int R, int NB>
__global__ void __launch_bounds__(256, 1) rd_tma(const float* __restrict__ Y, const int* __restrict__ perm, int n, float* sink) {
  extern __shared__ __align__(128) float buf[];   // [NB][R][64]
  __shared__ __align__(8) unsigned long long bar[NB];
  const int per = (n + gridDim.x - 1) / gridDim.x, lo = blockIdx.x * per, hi = min(n, lo + per);
  const int nst = (hi - lo + R - 1) / R;
  if (threadIdx.x == 0) {
    for (int b = 0; b < NB; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[b])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](int st) {   // warp 0: lanes issue the R row copies of stage st
    const int b = st % NB;
    const int r0 = lo + st * R, cnt = min(R, hi - r0);
    if (threadIdx.x == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[b])), "r"(cnt * 256) : "memory");
    __syncwarp();
    for (int i = threadIdx.x; i < cnt; i += 32) {
      const int row = perm ? __ldg(perm + r0 + i) : r0 + i;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];"
                   ::"r"(su32(buf + ((size_t)b * R + i) * 64)), "l"(Y + (size_t)row * 64), "r"(su32(&bar[b])) : "memory");
    }
  };
  if (threadIdx.x < 32)
    for (int st = 0; st < NB && st < nst; ++st) issue(st);
  float acc = 0.f;
  for (int st = 0; st < nst; ++st) {
    const int b = st % NB;
    const unsigned ph = (st / NB) & 1;
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(su32(&bar[b])), "r"(ph) : "memory");
    const int cnt = min(R, hi - (lo + st * R));
    for (int i = threadIdx.x; i < cnt * 64; i += blockDim.x) acc += buf[(size_t)b * R * 64 + i];
    __syncthreads();
    if (threadIdx.x < 32 && st + NB < nst) issue(st + NB);
  }
  if (acc == 1234.5f) sink[0] = acc;
}
int main() {
  const int n = 1 << 20;
  float* Y; int* perm; float* sink; char* fl;
  cudaMalloc(&Y, (size_t)n * 256); cudaMemset(Y, 0, (size_t)n * 256);
  cudaMalloc(&perm, n * 4); cudaMalloc(&sink, 4); cudaMalloc(&fl, 512u << 20);
  std::vector<int> h(n);
  for (int i = 0; i < n; ++i) h[i] = i;
  unsigned long long s = 88172645463325252ull;
  for (int i = n - 1; i > 0; --i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; std::swap(h[i], h[s % (i + 1)]); }
  cudaMemcpy(perm, h.data(), n * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](auto launch, const char* nm) {
    float best = 1e9;
    for (int rep = 0; rep < 6; ++rep) {
      cudaMemset(fl, rep, 512u << 20);
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep) best = std::min(best, ms);
    }
    printf("%-40s %7.1f us  %6.0f GB/s of rows\n", nm, best * 1e3, (double)n * 256 / (best * 1e-3) / 1e9);
  };
  for (int rnd = 0; rnd < 2; ++rnd) {
    const int* p = rnd ? perm : nullptr;
    const char* w = rnd ? "rand" : "seq ";
    char nm[80];
    snprintf(nm, 80, "%s lanegrp U=4  1024thr", w); run([&] { rd_lg<4><<<148, 1024>>>((const float4*)Y, p, n, sink); }, nm);
    snprintf(nm, 80, "%s lanegrp U=8  1024thr", w); run([&] { rd_lg<8><<<148, 1024>>>((const float4*)Y, p, n, sink); }, nm);
    snprintf(nm, 80, "%s lanegrp U=16 1024thr", w); run([&] { rd_lg<16><<<148, 1024>>>((const float4*)Y, p, n, sink); }, nm);
    snprintf(nm, 80, "%s lanegrp U=8  2x512thr", w); run([&] { rd_lg<8><<<296, 512>>>((const float4*)Y, p, n, sink); }, nm);
    cudaFuncSetAttribute(rd_tma<64, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 8 * 256);
    cudaFuncSetAttribute(rd_tma<32, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 16 * 256);
    cudaFuncSetAttribute(rd_tma<64, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 12 * 256);
    snprintf(nm, 80, "%s tma R=64 NB=8 (128 KB)", w); run([&] { rd_tma<64, 8><<<148, 256, 64 * 8 * 256>>>(Y, p, n, sink); }, nm);
    snprintf(nm, 80, "%s tma R=32 NB=16 (128 KB)", w); run([&] { rd_tma<32, 16><<<148, 256, 32 * 16 * 256>>>(Y, p, n, sink); }, nm);
    snprintf(nm, 80, "%s tma R=64 NB=12 (192 KB)", w); run([&] { rd_tma<64, 12><<<148, 256, 64 * 12 * 256>>>(Y, p, n, sink); }, nm);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
