// Microbenchmark: W[I[e]] += Y[e] (1M x 64 fp32 into 100k rows) with
// (a) red.global.add.v4.f32 per 16 B, (b) one TMA bulk reduction
// (cp.reduce.async.bulk .add.f32, 256 B) per row.  Uniform and Zipf-like (10%
// of entries on row 0) indices; L2 flushed before each run.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void red_v4(const int* I, const float4* Y, float* W, int n) {
  const int lane = threadIdx.x & 15;
  const long long hw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 4, nhw = ((long long)gridDim.x * blockDim.x) >> 4;
  for (long long e = hw; e < n; e += nhw) {
    const float4 v = __ldcs(Y + e * 16 + lane);
    float* d = W + (size_t)__ldg(I + e) * 64 + 4 * lane;
    asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(d), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
  }
}
// CHUNK rows per stage, NBUF stages; warp 0 lane 0 drives TMA; lanes 0..CHUNK-1 issue reductions
template <int CHUNK, int NBUF>
__global__ void __launch_bounds__(32) bulk_red(const int* I, const float* Y, float* W, int n) {
  __shared__ __align__(128) float buf[NBUF][CHUNK * 64];
  __shared__ __align__(8) unsigned long long bar[NBUF];
  const int lane = threadIdx.x;
  const long long nchunks = (n + CHUNK - 1) / CHUNK;
  if (lane == 0) {
    for (int b = 0; b < NBUF; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[b])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  auto load = [&](long long c, int b) {
    if (lane == 0) {
      const int rows = (int)min((long long)CHUNK, n - c * CHUNK);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[b])), "r"(rows * 256) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su32(buf[b])), "l"(Y + c * CHUNK * 64), "r"(rows * 256), "r"(su32(&bar[b])) : "memory");
    }
  };
  unsigned phase[NBUF] = {};
  long long c = blockIdx.x;
  const long long step = gridDim.x;
  for (int b = 0; b < NBUF; ++b) if (c + b * step < nchunks) load(c + b * step, b);
  int b = 0;
  for (; c < nchunks; c += step) {
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(su32(&bar[b])), "r"(phase[b]) : "memory");
    phase[b] ^= 1;
    const int rows = (int)min((long long)CHUNK, n - c * CHUNK);
    for (int r = lane; r < rows; r += 32) {
      const int row = __ldg(I + c * CHUNK + r);
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 256;"
                   ::"l"(W + (size_t)row * 64), "r"(su32(buf[b] + r * 64)) : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // smem reusable
    __syncwarp();
    const long long cn = c + NBUF * step;
    if (cn < nchunks) load(cn, b);
    b = (b + 1) % NBUF;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
int main() {
  const int n = 1 << 20, V = 100000;
  float *Y, *W, *fl; int *Iu, *Iz;
  cudaMalloc(&Y, (size_t)n * 256); cudaMemset(Y, 0, (size_t)n * 256);
  cudaMalloc(&W, (size_t)V * 256); cudaMalloc(&Iu, n * 4); cudaMalloc(&Iz, n * 4); cudaMalloc(&fl, 512u << 20);
  std::vector<int> hu(n), hz(n);
  unsigned long long s = 88172645463325252ull;
  for (int i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; hu[i] = s % V; hz[i] = (s >> 20) % 10 == 0 ? 0 : s % V; }
  cudaMemcpy(Iu, hu.data(), n * 4, cudaMemcpyHostToDevice); cudaMemcpy(Iz, hz.data(), n * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](auto launch, const char* nm) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemset(fl, rep, 512u << 20);
      cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (rep) best = std::min(best, ms);
    }
    printf("%-36s %7.1f us  (%5.0f GB/s of Y)\n", nm, best * 1e3, (double)n * 256 / (best * 1e-3) / 1e9);
  };
  for (int* I : {Iu, Iz}) {
    const char* dist = I == Iu ? "uniform" : "10%-hot";
    char nm[64];
    snprintf(nm, 64, "red.v4        %s", dist); run([&] { red_v4<<<148 * 8, 256>>>(I, (const float4*)Y, W, n); }, nm);
    snprintf(nm, 64, "bulk 32x4 x8/SM %s", dist); run([&] { bulk_red<32, 4><<<148 * 8, 32>>>(I, Y, W, n); }, nm);
    snprintf(nm, 64, "bulk 32x4 x16/SM %s", dist); run([&] { bulk_red<32, 4><<<148 * 16, 32>>>(I, Y, W, n); }, nm);
    snprintf(nm, 64, "bulk 16x4 x24/SM %s", dist); run([&] { bulk_red<16, 4><<<148 * 24, 32>>>(I, Y, W, n); }, nm);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
