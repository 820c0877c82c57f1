// Microbenchmark: W[I[e]] += Y[e] (1M x 64 fp32 into 100k rows, L2 flushed)
// with Y streamed through a TMA bulk-copy ring in shared memory (one producer
// lane, mbarrier full/empty pairs, NC consumer warps issuing red.v4 from smem)
// against the register-staged stream of sc_atomic_hot (U float4 per lane in
// flight).  MODE 0 reads only (the read ceiling), MODE 1 scatters.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned long long* b, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned ph) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(smem_u32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}

template <int CH, int S, int NC, int MODE>
__global__ void __launch_bounds__((NC + 1) * 32, 1) tma_k(const int* __restrict__ I, const float* __restrict__ Y,
                                                           float* W, int n, float* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  float4* Ys = reinterpret_cast<float4*>(sm);                          // [S][CH][16]
  int* Is = reinterpret_cast<int*>(sm + (size_t)S * CH * 256);         // [S][CH]
  unsigned long long* full = reinterpret_cast<unsigned long long*>(sm + (size_t)S * CH * 260);
  unsigned long long* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int C = (n + CH - 1) / CH;
  const int c0 = (int)((long long)blockIdx.x * C / gridDim.x), c1 = (int)((long long)(blockIdx.x + 1) * C / gridDim.x);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NC); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == NC) {
    if (lane == 0) {
      for (int c = c0; c < c1; ++c) {
        const int k = c - c0, s = k % S;
        if (k >= S) mbar_wait(&empty[s], ((k / S) - 1) & 1);
        const int e0 = c * CH, cnt = min(CH, n - e0);
        const unsigned ib = (unsigned)((cnt * 4 + 15) & ~15);
        mbar_expect(&full[s], cnt * 256u + ib);
        bulk_g2s(Ys + (size_t)s * CH * 16, Y + (size_t)e0 * 64, cnt * 256u, &full[s]);
        bulk_g2s(Is + s * CH, I + e0, ib, &full[s]);
      }
    }
    return;
  }
  float acc = 0.f;
  for (int c = c0; c < c1; ++c) {
    const int k = c - c0, s = k % S;
    mbar_wait(&full[s], (k / S) & 1);
    const int cnt = min(CH, n - c * CH);
    for (int it = threadIdx.x; it < cnt * 16; it += NC * 32) {
      const int e = it >> 4, g = it & 15;
      const float4 v = Ys[(size_t)s * CH * 16 + it];
      if (MODE == 0) acc += v.x + v.y + v.z + v.w;
      else {
        float* d = W + (size_t)Is[s * CH + e] * 64 + 4 * g;
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(d), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                     : "memory");
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (MODE == 0 && acc == 12345.f) *sink = acc;
}

template <int U, int MODE>   // register-staged (sc_atomic_hot style): half-warp per row, U rows in flight
__global__ void __launch_bounds__(1024, 1) reg_k(const int* __restrict__ I, const float4* __restrict__ Y, float* W,
                                                 int n, float* sink) {
  const int lane = threadIdx.x & 15;
  const long long hw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 4;
  const long long nhw = ((long long)gridDim.x * blockDim.x) >> 4;
  float acc = 0.f;
  for (long long e0 = hw * U; e0 < n; e0 += nhw * U) {
    float4 v[U];
    int row[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long e = e0 + u;
      row[u] = e < n ? __ldg(I + e) : 0;
      v[u] = e < n ? __ldcs(Y + e * 16 + lane) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (e0 + u >= n) break;
      float* d = W + (size_t)row[u] * 64 + 4 * lane;
      if (MODE == 0) acc += v[u].x + v[u].y + v[u].z + v[u].w;
      else
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(d), "f"(v[u].x), "f"(v[u].y), "f"(v[u].z),
                     "f"(v[u].w)
                     : "memory");
    }
  }
  if (MODE == 0 && acc == 12345.f) *sink = acc;
}

int main() {
  const int n = 1000000, V = 100000;
  float *Y, *W, *fl, *sink;
  int *Iu;
  cudaMalloc(&Y, (size_t)n * 256 + 4096);
  cudaMemset(Y, 0, (size_t)n * 256);
  cudaMalloc(&W, (size_t)V * 256);
  cudaMalloc(&Iu, n * 4 + 4096);
  cudaMalloc(&fl, 512u << 20);
  cudaMalloc(&sink, 4);
  std::vector<int> hu(n);
  unsigned long long x = 88172645463325252ull;
  for (int i = 0; i < n; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; hu[i] = x % V; }
  cudaMemcpy(Iu, hu.data(), n * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](auto launch, const char* nm) {
    std::vector<float> t;
    for (int rep = 0; rep < 9; ++rep) {
      cudaMemset(fl, rep, 512u << 20);
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep) t.push_back(ms * 1e3f);
    }
    std::sort(t.begin(), t.end());
    printf("%-36s median %7.1f us  min %7.1f  (%5.0f GB/s of Y at median)  %s\n", nm, t[t.size() / 2], t[0],
           (double)n * 256 / (t[t.size() / 2] * 1e-6) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
#define TMA(CH, S, NC, MODE)                                                                                   \
  {                                                                                                            \
    auto kf = tma_k<CH, S, NC, MODE>;                                                                          \
    const int smem = S * CH * 260 + 16 * S + 128;                                                              \
    cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);                              \
    char nm[80];                                                                                               \
    snprintf(nm, 80, "tma CH%d S%d NC%d %s", CH, S, NC, MODE ? "red" : "read");                               \
    run([&] { kf<<<148, (NC + 1) * 32, smem>>>(Iu, Y, W, n, sink); }, nm);                                     \
  }
  run([&] { reg_k<4, 0><<<148, 1024>>>(Iu, (const float4*)Y, W, n, sink); }, "reg U4 1024t read");
  run([&] { reg_k<4, 1><<<148, 1024>>>(Iu, (const float4*)Y, W, n, sink); }, "reg U4 1024t red");
  TMA(64, 4, 16, 0) TMA(64, 8, 16, 0) TMA(32, 8, 16, 0) TMA(64, 12, 16, 0) TMA(128, 6, 16, 0)
  TMA(64, 4, 16, 1) TMA(64, 8, 16, 1) TMA(32, 8, 16, 1) TMA(64, 12, 16, 1) TMA(128, 6, 16, 1)
  TMA(64, 8, 8, 1) TMA(64, 8, 24, 1) TMA(32, 16, 16, 1) TMA(64, 8, 31, 1)
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
