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

// ---------------------------------------------------------------- nonlinearity
// act 0: hardtanh z = clamp(a, -1, 1) (north_star; reading G1), derivative 1
// strictly inside (-1, 1), 0 at and beyond |a| = 1 (G2); act 1: z = tanh(a),
// derivative 1 - z^2.
__device__ __forceinline__ float act_f(float a, int act) {
  return act ? tanhf(a) : fminf(fmaxf(a, -1.f), 1.f);
}
// gw * f'(a) given z = f(a); the hardtanh branch is a select (no multiply), so
// that path's bits are unchanged by the switch.
__device__ __forceinline__ float act_g(float gw, float a, float z, int act) {
  return act ? gw * (1.f - z * z) : (fabsf(a) < 1.f ? gw : 0.f);
}
// sigma = delta + delta' for the context rows, delta = gw f'(a), delta' =
// -gw f'(a').  For tanh, (1 - z^2) - (1 - z'^2) cancels in fp32 (z^2 is small
// next to 1, so the difference keeps ~1e-4 relative accuracy); the same value
// is formed as gw (z' - z)(z' + z).  Hardtanh keeps delta + delta'.
__device__ __forceinline__ float act_sigma(float gw, float z, float zc, float dl, float dlc, int act) {
  return act ? gw * ((zc - z) * (zc + z)) : dl + dlc;
}

// ---------------------------------------------------------------- bitonic sort
// Bitonic sort of n (power of two, >= 32) 64-bit keys in smem with the
// sub-steps of stride < 32 done in registers by warp shuffles: key i sits at
// lane i % 32 of group i / 32, warp w takes groups w, w + #warps, ...  Only the
// stride >= 32 sub-steps go through shared memory, so a 1024-key sort needs 21
// block barriers instead of 55.  Same network, same result as bitonic_sort.
__device__ __forceinline__ unsigned long long shfl_xor_u64(unsigned long long v, int m) {
  const unsigned lo = __shfl_xor_sync(0xffffffffu, (unsigned)v, m);
  const unsigned hi = __shfl_xor_sync(0xffffffffu, (unsigned)(v >> 32), m);
  return ((unsigned long long)hi << 32) | lo;
}
__device__ __forceinline__ void bitonic_sort_warp(unsigned long long* k, int n) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5, G = n >> 5;
  // sub-steps with stride in [1, top] of stage `size`, for every group of this warp
  auto warp_steps = [&](int size, int top) {
    for (int g = warp; g < G; g += NW) {
      const int i = g * 32 + lane;
      unsigned long long v = k[i];
      for (int stride = top; stride > 0; stride >>= 1) {
        const unsigned long long o = shfl_xor_u64(v, stride);
        const bool up = (i & size) == 0, lower = (lane & stride) == 0;
        const bool take_min = lower == up;
        v = take_min ? (o < v ? o : v) : (o > v ? o : v);
      }
      k[i] = v;
    }
  };
  for (int g = warp; g < G; g += NW) {   // stages of size 2..32 entirely in registers
    const int i = g * 32 + lane;
    unsigned long long v = k[i];
    for (int sz = 2; sz <= 32; sz <<= 1)
      for (int stride = sz >> 1; stride > 0; stride >>= 1) {
        const unsigned long long o = shfl_xor_u64(v, stride);
        const bool up = (i & sz) == 0, lower = (lane & stride) == 0;
        v = (lower == up) ? (o < v ? o : v) : (o > v ? o : v);
      }
    k[i] = v;
  }
  __syncthreads();
  for (int size = 64; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride >= 32; stride >>= 1) {
      for (int t = threadIdx.x; t < (n >> 1); t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const unsigned long long a = k[lo], b = k[hi];
        if ((a > b) == up) { k[lo] = b; k[hi] = a; }
      }
      __syncthreads();
    }
    warp_steps(size, 16);
    __syncthreads();
  }
}

// ---------------------------------------------------------------- grid barrier
// Barrier for a cooperative (co-resident) grid on a monotonic 64-bit arrival
// counter that is never reset: every instance adds exactly gridDim.x, so the
// arrival value `old` names the instance (old / G) and its release point
// ((old / G + 1) * G).  Waiters poll the counter itself -- one L2 round trip
// after the last arrival, no separate generation word.  All users of one
// counter must launch the same grid size (callers keep one counter per grid
// size).  Ordering: bar.sync makes the CTA's
// writes visible to thread 0; its acq_rel arrival RMW (cumulative) publishes
// them; the waiter's acquire load of the final count synchronises with every
// arrival, and bar.sync hands that on to the CTA.
__device__ __forceinline__ unsigned ld_relaxed_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Split form: grid_arrive publishes this CTA's prior writes and returns (in
// thread 0) the instance's release count; independent work can run before
// grid_wait blocks on it.
__device__ __forceinline__ unsigned long long grid_arrive(unsigned long long* arrivals) {
  __syncthreads();
  unsigned long long target = 0;
  if (threadIdx.x == 0) {
    unsigned long long old;
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;" : "=l"(old) : "l"(arrivals) : "memory");
    const unsigned long long G = gridDim.x;
    target = (old / G + 1) * G;
  }
  return target;
}
__device__ __forceinline__ void grid_wait(unsigned long long* arrivals, unsigned long long target) {
  if (threadIdx.x == 0) {
    unsigned long long now;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(now) : "l"(arrivals) : "memory");
    } while (now < target);
  }
  __syncthreads();
}
__device__ __forceinline__ void grid_barrier(unsigned long long* arrivals) {
  grid_wait(arrivals, grid_arrive(arrivals));
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
