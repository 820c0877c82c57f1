// Microbenchmark: cycles of one stable block radix pass (o_pass<DB>, the DET
// owner scatter's ranking, scatter_det.cu) on 8192 keys per CTA, 148 CTAs x 1024.
#include "../../paper_1404_1521_b200/csrc/scatter_det.cu"
#include <cstdio>
namespace pg {
template <int DB>
__device__ int o_pass_m(const unsigned (&key)[8], const bool (&valid)[8], int shift, unsigned* out,
                        unsigned short* whist, int* dstart, int* ws) {
  constexpr int kBins = 1 << DB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  unsigned short* wh = whist + warp * kBins;
  for (int d = lane; d < kBins; d += 32) wh[d] = 0;
  __syncwarp();
  int lrank[8];
  unsigned dig[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    dig[j] = (key[j] >> shift) & (unsigned)(kBins - 1);
    const unsigned mm = __match_any_sync(0xffffffffu, valid[j] ? dig[j] : 0xffffffffu);
    const unsigned peers = valid[j] ? mm : 0u;
    const int before = valid[j] ? wh[dig[j]] : 0;
    __syncwarp();
    if (valid[j] && (peers & lt) == 0) wh[dig[j]] = (unsigned short)(before + __popc(peers));
    __syncwarp();
    lrank[j] = before + __popc(peers & lt);
  }
  __syncthreads();
  int run = 0;
  if (tid < kBins) {
    for (int w = 0; w < 32; ++w) {
      const int v = whist[w * kBins + tid];
      whist[w * kBins + tid] = (unsigned short)run;
      run += v;
    }
  }
  int total = 0;
  const int ex = block_excl_scan(run, ws, &total);
  if (tid < kBins) dstart[tid] = ex;
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (valid[j]) out[dstart[dig[j]] + wh[dig[j]] + lrank[j]] = key[j];
  __syncthreads();
  return total;
}
template <int DB, int M>
__global__ void __launch_bounds__(1024, 1) opass_k(unsigned long long* cyc, int reps, unsigned range) {
  extern __shared__ __align__(16) unsigned char dsm[];
  unsigned* out = reinterpret_cast<unsigned*>(dsm);
  unsigned short* wh = reinterpret_cast<unsigned short*>(dsm + 8192 * 4);
  int* ds = reinterpret_cast<int*>(dsm + 8192 * 4 + 32 * (1 << DB) * 2);
  __shared__ int ws[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned key[8];
  bool val[8];
  for (int j = 0; j < 8; ++j) {
    const int i = warp * 256 + j * 32 + lane;
    unsigned x = (unsigned)(i * 2654435761u) ^ (blockIdx.x * 97u);
    key[j] = ((x % range) << 13) | (unsigned)i;
    val[j] = i < 6757;
  }
  __syncthreads();
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) { if (M) o_pass_m<DB>(key, val, 13, out, wh, ds, ws); else o_pass<DB>(key, val, 13, out, wh, ds, ws); }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
  if (out[threadIdx.x] == 0xdeadbeef) cyc[0] = 0;
}
}  // namespace pg
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 160 * 8);
  unsigned long long h[160];
  auto run = [&](auto k, const char* nm, unsigned range) {
    const int smem = 8192 * 4 + 32 * 1024 * 2 + 1025 * 4;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<148, 1024, smem>>>(d, 4, range);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0, sm = 0;
    for (int i = 0; i < 148; ++i) { mx = h[i] > mx ? h[i] : mx; sm += h[i]; }
    printf("%-10s range %5u: mean %6llu cycles, max %6llu (%.2f us at 1.9 GHz)\n", nm, range, sm / 148, mx, mx / 1900.0);
  };
  run(pg::opass_k<10, 0>, "ballot10", 676);
  run(pg::opass_k<10, 1>, "match10", 676);
  run(pg::opass_k<9, 0>, "ballot9", 400);
  run(pg::opass_k<9, 1>, "match9", 400);
  run(pg::opass_k<5, 0>, "ballot5", 32);
  run(pg::opass_k<5, 1>, "match5", 32);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
