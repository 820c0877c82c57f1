// Host cost of cudaPointerGetAttributes (the ABI's host/device pointer test).
#include <cstdio>
#include <chrono>
#include <cuda_runtime.h>
int main() {
  float *d, *h, *pg = new float[1024];
  cudaMalloc(&d, 1 << 20); cudaMallocHost(&h, 1 << 20);
  for (void* p : {(void*)d, (void*)(d + 1), (void*)h, (void*)pg}) {
    cudaPointerAttributes a;
    auto t0 = std::chrono::high_resolution_clock::now();
    for (int i = 0; i < 10000; ++i) { cudaPointerGetAttributes(&a, p); }
    auto t1 = std::chrono::high_resolution_clock::now();
    printf("%p type %d: %.3f us/call\n", p, (int)a.type, std::chrono::duration<double, std::micro>(t1 - t0).count() / 10000);
  }
}
