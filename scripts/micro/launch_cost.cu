// Microbenchmark: event-timed cost of launching an (almost) empty kernel of the
// step's shape (148 CTAs x 384 threads) right after a 512 MB fill, for
// normal vs cooperative launch and small vs ~200 KB dynamic shared memory.
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
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int coop = 0; coop < 2; ++coop)
    for (int smem : {2048, 200 * 1024})
      for (int flush : {0, 1}) {
        std::vector<float> t;
        for (int rep = 0; rep < 30; ++rep) {
          if (flush) fill_k<<<148 * 4, 256>>>(fl, (512u << 20) / 16);
          cudaEventRecord(a);
          void* args[] = {(void*)&out};
          if (coop) cudaLaunchCooperativeKernel((void*)empty_k, 148, 384, args, smem, 0);
          else empty_k<<<148, 384, smem>>>(out);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms; cudaEventElapsedTime(&ms, a, b);
          if (rep >= 5) t.push_back(ms * 1e3f);
        }
        std::sort(t.begin(), t.end());
        printf("coop=%d smem=%6d flush=%d  median %6.2f us  min %6.2f\n", coop, smem, flush, t[t.size() / 2], t[0]);
      }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
