// Microbenchmark: the dense reduce pattern of phase 2.  148 CTAs each write a
// 41 KB record, then (after a grid barrier, or in a second launch) each CTA
// reads an 18-quad column slice from all 148 records.  Reports per-CTA cycles of
// the read phase: same-launch (just written) vs next-launch.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
constexpr int G = 148, NT = 384, STRIDE = 10368;   // floats per record
__device__ unsigned long long g_arr;
__device__ void gbar() {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long old;
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;" : "=l"(old) : "l"(&g_arr) : "memory");
    unsigned long long target = (old / G + 1) * G, now = old + 1;
    while (now < target) asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(now) : "l"(&g_arr) : "memory");
  }
  __syncthreads();
}
__global__ void __launch_bounds__(NT, 1) k(float* rec, int write, int read, long long* out, float* sink) {
  const int tid = threadIdx.x;
  if (write) {
    float4* r = reinterpret_cast<float4*>(rec + (size_t)blockIdx.x * STRIDE);
    for (int i = tid; i < STRIDE / 4; i += NT) r[i] = make_float4(tid, 1, 2, 3);
  }
  if (write && read) gbar();
  if (!read) return;
  const int NQ = STRIDE / 4, q0 = blockIdx.x * NQ / G, q1 = (blockIdx.x + 1) * NQ / G, nq = q1 - q0;
  const int groups = min(NT / nq, 32), qi = tid % nq, g = tid / nq;
  long long t0 = clock64();
  float4 acc = make_float4(0, 0, 0, 0);
  if (g < groups) {
    for (int r0 = g; r0 < G; r0 += 8 * groups) {
      float4 v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int r = r0 + j * groups;
        v[j] = r < G ? __ldcg(reinterpret_cast<const float4*>(rec + (size_t)r * STRIDE) + q0 + qi) : make_float4(0, 0, 0, 0);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) { acc.x += v[j].x; acc.y += v[j].y; acc.z += v[j].z; acc.w += v[j].w; }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
  if (acc.x == 1234.5f) sink[0] = acc.y;
}
int main() {
  float* rec; long long* out; float* sink; float* fl;
  cudaMalloc(&rec, (size_t)G * STRIDE * 4); cudaMalloc(&out, G * 8); cudaMalloc(&sink, 4); cudaMalloc(&fl, 512u << 20);
  void* args[5];
  auto run = [&](int w, int r, const char* nm, bool flush) {
    std::vector<long long> all;
    for (int rep = 0; rep < 8; ++rep) {
      if (flush) cudaMemset(fl, rep, 512u << 20);
      if (!w) k<<<G, NT>>>(rec, 1, 0, out, sink);   // records written by the previous launch
      int ww = w, rr = r;
      args[0] = &rec; args[1] = &ww; args[2] = &rr; args[3] = &out; args[4] = &sink;
      cudaLaunchCooperativeKernel((void*)k, G, NT, args, 0, 0);
      cudaDeviceSynchronize();
      std::vector<long long> h(G); cudaMemcpy(h.data(), out, G * 8, cudaMemcpyDeviceToHost);
      if (rep >= 2) all.insert(all.end(), h.begin(), h.end());
    }
    std::sort(all.begin(), all.end());
    printf("%-28s flush=%d read cycles med %6lld p90 %6lld max %6lld\n", nm, flush, all[all.size() / 2], all[all.size() * 9 / 10], all.back());
  };
  run(1, 1, "write+barrier+read", false);
  run(0, 1, "read (written last launch)", false);
  run(1, 1, "write+barrier+read", true);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
