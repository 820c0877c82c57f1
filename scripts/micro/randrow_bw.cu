// Microbenchmark: DRAM bandwidth of random 256 B row reads (the sorted-gather
// pattern of the deterministic scatter) vs sequential reads of the same bytes.
// 1M rows of 64 fp32 (256 MB), L2 flushed before every run.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
template <int UNROLL>
__global__ void rd(const float4* __restrict__ Y, const int* __restrict__ perm, int n, float* sink) {
  // 16 lanes per row (16 B each); each half-warp walks rows with UNROLL in flight
  const int lane = threadIdx.x & 15;
  const long long hw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 4;
  const long long nhw = ((long long)gridDim.x * blockDim.x) >> 4;
  float4 acc = make_float4(0, 0, 0, 0);
  for (long long r0 = hw * UNROLL; r0 < n; r0 += nhw * UNROLL) {
    float4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const long long r = r0 + u;
      const int row = r < n ? (perm ? __ldg(perm + r) : (int)r) : 0;
      v[u] = r < n ? __ldcs(Y + (size_t)row * 16 + lane) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
  }
  if (acc.x == 1234.5f) sink[0] = acc.y + acc.z + acc.w;
}
int main() {
  const int n = 1 << 20;
  float4* Y; int* perm; float* sink; char* fl;
  cudaMalloc(&Y, (size_t)n * 256); cudaMemset(Y, 0, (size_t)n * 256);
  cudaMalloc(&perm, n * 4); cudaMalloc(&sink, 4); cudaMalloc(&fl, 512u << 20);
  std::vector<int> h(n);
  for (int i = 0; i < n; ++i) h[i] = i;
  unsigned long long s = 88172645463325252ull;
  for (int i = n - 1; i > 0; --i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; std::swap(h[i], h[s % (i + 1)]); }
  cudaMemcpy(perm, h.data(), n * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](auto kern, const int* p, int blocks, int threads, const char* nm) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemset(fl, rep, 512u << 20);
      cudaEventRecord(a);
      kern<<<blocks, threads>>>(Y, p, n, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep) best = std::min(best, ms);
    }
    printf("%-34s %7.1f us  %6.0f GB/s (rows 256 MB + idx)\n", nm, best * 1e3, ((double)n * 256 + (p ? n * 4.0 : 0)) / (best * 1e-3) / 1e9);
  };
  for (int bpsm : {4, 8, 16}) {
    char nm[64];
    snprintf(nm, 64, "seq   unroll4  %2d blk/SM x256", bpsm);  run(rd<4>, nullptr, 148 * bpsm, 256, nm);
    snprintf(nm, 64, "rand  unroll4  %2d blk/SM x256", bpsm);  run(rd<4>, perm, 148 * bpsm, 256, nm);
    snprintf(nm, 64, "rand  unroll8  %2d blk/SM x256", bpsm);  run(rd<8>, perm, 148 * bpsm, 256, nm);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
