// nccl_lsa.cu -- resolve the load/store addresses of every rank's copy of an
// NCCL symmetric-memory window once, at setup (NCCL 2.28 device API,
// ncclGetLsaPointer), so the step kernels address peers with plain pointers
// and need no NCCL headers.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <string>

#include "nccl_shim.h"

namespace {
__global__ void lsa_pointers_kernel(ncclWindow_t w, int world, unsigned long long* out) {
  for (int r = threadIdx.x; r < world; r += blockDim.x) out[r] = (unsigned long long)ncclGetLsaPointer(w, 0, r);
}
}  // namespace

int nccl_lsa_pointers(void* win, int world, unsigned long long* out, std::string* err) {
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMalloc(&d, sizeof(unsigned long long) * world);
  if (e == cudaSuccess) {
    lsa_pointers_kernel<<<1, 64>>>(static_cast<ncclWindow_t>(win), world, d);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(out, d, sizeof(unsigned long long) * world, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) {
    if (err) *err = std::string("ncclGetLsaPointer: ") + cudaGetErrorString(e);
    return 1;
  }
  return 0;
}
