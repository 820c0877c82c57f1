// Microbenchmark: what an event-bracketed launch of the step's shape costs
// after a 512 MB fill -- one empty cooperative kernel, two back to back, the
// kernel with the programmatic-stream-serialisation attribute, and a graph.
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
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(empty_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto coop = [&](int pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148); cfg.blockDim = dim3(384); cfg.dynamicSmemBytes = smem; cfg.stream = s;
    cudaLaunchAttribute at[2]; int na = 0;
    at[na].id = cudaLaunchAttributeCooperative; at[na].val.cooperative = 1; ++na;
    if (pdl) { at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[na].val.programmaticStreamSerializationAllowed = 1; ++na; }
    cfg.attrs = at; cfg.numAttrs = na;
    cudaLaunchKernelEx(&cfg, empty_k, out);
  };
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal); coop(0); cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  const char* names[] = {"coop x1", "coop x2", "coop+pdl attr x1", "graph(coop) x1", "no kernel"};
  for (int v = 0; v < 5; ++v)
    for (int flush : {0, 1}) {
      std::vector<float> t;
      for (int rep = 0; rep < 40; ++rep) {
        if (flush) fill_k<<<148 * 4, 256, 0, s>>>(fl, (512u << 20) / 16);
        cudaEventRecord(a, s);
        if (v == 0) coop(0);
        if (v == 1) { coop(0); coop(0); }
        if (v == 2) coop(1);
        if (v == 3) cudaGraphLaunch(ge, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep >= 5) t.push_back(ms * 1e3f);
      }
      std::sort(t.begin(), t.end());
      printf("%-18s flush=%d  median %6.2f us  min %6.2f\n", names[v], flush, t[t.size() / 2], t[0]);
    }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
