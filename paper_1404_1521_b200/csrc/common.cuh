// common.cuh -- device helpers shared by the sm_100a kernels of libpg.
// Nothing here is shared with oracle/ (the two implementations are independent).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace pg {

constexpr int kMaxSMs = 160;          // upper bound on gridDim for per-CTA tables
constexpr unsigned long long kNoBad = ~0ull;

// ---------------------------------------------------------------- memory-order helpers
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_acqrel_gpu(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;"
               : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// red.global.add.v4.f32 (sm_90+): one vector reduction per 16 B.  Flushes
// subnormals (SASS REDG.E.ADD.F32x4.FTZ.RN) -- see DESIGN.md.
__device__ __forceinline__ void red_add_v4(float* addr, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};"
               ::"l"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

__device__ __forceinline__ float4 ldcg4(const float* p) {
  return __ldcg(reinterpret_cast<const float4*>(p));
}

// ---------------------------------------------------------------- grid barrier
// Sense-reversing barrier for a cooperative (co-resident) grid.  State lives in
// device memory and survives across launches: `count` returns to 0 after every
// barrier and `gen` increases monotonically.
__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned* gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned my_gen = ld_acquire_gpu(gen);
    __threadfence();
    unsigned arrived = atom_add_acqrel_gpu(count, 1u);
    if (arrived == gridDim.x - 1) {
      *count = 0;
      __threadfence();
      st_release_gpu(gen, my_gen + 1);
    } else {
      while (ld_acquire_gpu(gen) == my_gen) __nanosleep(40);
    }
    __threadfence();
  }
  __syncthreads();
}

// ---------------------------------------------------------------- warp helpers
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide exclusive scan of one int per thread (blockDim.x <= 1024).
// `ws` must hold 32 ints.  Returns the exclusive prefix; *total gets the sum.
__device__ __forceinline__ int block_excl_scan(int v, int* ws, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = lane < nw ? ws[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    ws[lane] = t;  // inclusive prefix of warp totals
  }
  __syncthreads();
  int res = x - v + (w > 0 ? ws[w - 1] : 0);
  if (total) *total = ws[nw - 1];
  __syncthreads();
  return res;
}

}  // namespace pg
