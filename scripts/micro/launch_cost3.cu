// Microbenchmark: event-bracketed launch cost after a 512 MB fill, for the
// step's shape (148 x 384, 1 CTA/SM): cooperative vs regular launch, with and
// without the 200 KB dynamic shared-memory carveout.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(384, 1) empty_k(int* out) {
  extern __shared__ int sm[];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x == 0 && sm[5] == 12345) out[blockIdx.x] = 1;
}
__global__ void fill_k(float4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = make_float4(1, 2, 3, 4);
}
int main() {
  int* out; float4* fl; cudaMalloc(&out, 4096); cudaMalloc(&fl, 512u << 20);
  cudaFuncSetAttribute(empty_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto launch = [&](int coop, int smem) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148); cfg.blockDim = dim3(384); cfg.dynamicSmemBytes = smem; cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1;
    cfg.attrs = at; cfg.numAttrs = coop ? 1 : 0;
    cudaLaunchKernelEx(&cfg, empty_k, out);
  };
  struct V { const char* name; int coop, smem, carve; };
  V vs[] = {{"coop 200KB", 1, 200 * 1024, -1}, {"regular 200KB", 0, 200 * 1024, -1},
            {"coop 8KB", 1, 8192, -1}, {"regular 8KB", 0, 8192, -1},
            {"regular 8KB carve100", 0, 8192, 100}, {"coop 200KB carve100", 1, 200 * 1024, 100}};
  for (auto& v : vs) {
    if (v.carve >= 0) cudaFuncSetAttribute(empty_k, cudaFuncAttributePreferredSharedMemoryCarveout, v.carve);
    for (int flush : {0, 1}) {
      std::vector<float> t;
      for (int rep = 0; rep < 60; ++rep) {
        if (flush) fill_k<<<148 * 4, 256, 0, s>>>(fl, (512u << 20) / 16);
        cudaEventRecord(a, s);
        launch(v.coop, v.smem);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep >= 5) t.push_back(ms * 1e3f);
      }
      std::sort(t.begin(), t.end());
      printf("%-22s flush=%d  median %6.2f us  min %6.2f\n", v.name, flush, t[t.size() / 2], t[0]);
    }
  }
  // event pair with the fill before it, two events in a row
  for (int flags : {0, 1}) {
    cudaEvent_t c, e2; cudaEventCreateWithFlags(&c, flags ? cudaEventBlockingSync : 0); cudaEventCreateWithFlags(&e2, flags ? cudaEventBlockingSync : 0);
    std::vector<float> t;
    for (int rep = 0; rep < 60; ++rep) {
      fill_k<<<148 * 4, 256, 0, s>>>(fl, (512u << 20) / 16);
      cudaEventRecord(c, s);
      cudaEventRecord(e2, s);
      cudaEventSynchronize(e2);
      float ms; cudaEventElapsedTime(&ms, c, e2);
      if (rep >= 5) t.push_back(ms * 1e3f);
    }
    std::sort(t.begin(), t.end());
    printf("event pair flags=%d after fill  median %6.2f us  min %6.2f\n", flags, t[t.size() / 2], t[0]);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
