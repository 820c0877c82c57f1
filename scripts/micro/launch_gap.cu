// Microbenchmark: period of back-to-back launches of the step's shape (148 x
// 384, 200 KB dynamic smem, 1 CTA/SM) -- cooperative vs regular launch, for an
// empty kernel and for a kernel that spins ~20 us (the gap between steps).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(384, 1) spin_k(int* out, long long ns) {
  extern __shared__ int sm[];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  sm[threadIdx.x] = threadIdx.x;
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while ((long long)(t - t0) < ns);
  __syncthreads();
  if (threadIdx.x == 0 && sm[5] == 12345) out[blockIdx.x] = 1;
}
int main() {
  int* out; cudaMalloc(&out, 4096);
  cudaFuncSetAttribute(spin_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int smem = 200 * 1024, pdl = 0;
  auto launch = [&](int coop, long long ns) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148); cfg.blockDim = dim3(384); cfg.dynamicSmemBytes = smem; cfg.stream = s;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (coop) { at[na].id = cudaLaunchAttributeCooperative; at[na].val.cooperative = 1; ++na; }
    if (pdl) { at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[na].val.programmaticStreamSerializationAllowed = 1; ++na; }
    cfg.attrs = at; cfg.numAttrs = na;
    cudaLaunchKernelEx(&cfg, spin_k, out, ns);
  };
  for (int v = 0; v < 3; ++v)
  for (long long ns : {0ll, 20000ll})
    for (int coop : {1, 0}) {
      smem = v == 1 ? 8 * 1024 : 200 * 1024;
      pdl = v == 2;
      for (int w = 0; w < 20; ++w) launch(coop, ns);
      const int K = 200;
      cudaEventRecord(a, s);
      for (int k = 0; k < K; ++k) launch(coop, ns);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("%s smem %3d KB pdl %d ", v == 1 ? "" : "", smem / 1024, pdl);
      printf("%s spin %5lld ns: period %6.2f us per launch (gap %5.2f us)\n", coop ? "coop   " : "regular", ns,
             ms * 1e3f / K, ms * 1e3f / K - ns * 1e-3f);
    }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
