// scatter.cu -- the paper's advanced-indexing update W[I[k], :] += Y[k, :]
// (the paper's CUDA kernel "each row is indexed in parallel,
// and for each row, each cell in the row is added in parallel")
// as two sm_100a pipelines behind pg_scatter_add:
//
// DET (bit-reproducible): stable LSD radix sort of (I[k], k) in 2 passes of
//   <= 11-bit digits (histogram kernel + one onesweep kernel per pass with
//   decoupled look-back), then a segmented reduction over fixed chunks of S
//   sorted entries: every segment sums its Y rows in k order; segments that
//   cross chunk boundaries leave per-chunk partials that a fix-up kernel
//   combines in chunk order with a fixed-shape tree.  One read-modify-write of
//   W per (row, chunk) -- in practice one per unique row.
// ATOMIC: validation pass, then red.global.add.v4.f32 per 16 B of each Y row
//   (FTZ), no ordering guarantee.
#include "common.cuh"
#include "scatter.cuh"

namespace pg {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;   // 4096 keys per tile
constexpr int kChunk = 256;                             // sorted entries per reduce chunk
constexpr unsigned kFlagA = 1u << 30, kFlagP = 2u << 30, kCountMask = (1u << 30) - 1;

// ------------------------------------------------------------------ histogram + validation
__global__ void __launch_bounds__(512) sc_hist(const int32_t* __restrict__ I, int64_t n, int64_t rows,
                                               int passes, int bits, int* __restrict__ hist,
                                               ScatterStatus* st) {
  extern __shared__ int sh[];
  const int bins = 1 << bits;
  for (int i = threadIdx.x; i < passes * bins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const int64_t e = base + threadIdx.x;
    const bool valid = e < n;
    int key = valid ? __ldg(I + e) : 0;
    if (valid && (key < 0 || (int64_t)key >= rows)) {
      atomicMin(&st->bad, ((unsigned long long)e << 32) | (unsigned)key);
      atomicOr(&st->flag, 1);
      key = 0;
    }
    for (int p = 0; p < passes; ++p) {
      const int dig = valid ? ((unsigned)key >> (p * bits)) & (bins - 1) : bins;
      const unsigned peers = __match_any_sync(0xffffffffu, dig);
      if (valid && lane == __ffs(peers) - 1) atomicAdd(&sh[p * bins + dig], __popc(peers));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * bins; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// ------------------------------------------------------------------ onesweep pass
// dynamic smem: whist[NW][bins] + tpref[bins] + ws[32]
__global__ void __launch_bounds__(kSortThreads) sc_onesweep(
    const int32_t* __restrict__ kin, const int32_t* __restrict__ vin, int32_t* __restrict__ kout,
    int32_t* __restrict__ vout, int64_t n, int shift, int bits, const int* __restrict__ hist,
    unsigned* lookback, unsigned* tile_ctr, const ScatterStatus* st) {
  extern __shared__ int sh[];
  __shared__ int s_tile;
  const int bins = 1 << bits, NW = kSortThreads / 32;
  int* whist = sh;                    // [NW][bins]
  int* tpref = sh + NW * bins;        // [bins]
  int* ws = tpref + bins;             // [32]
  if (*(volatile const int*)&st->flag) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = (int)atomicAdd(tile_ctr, 1u);
  for (int i = tid; i < NW * bins; i += kSortThreads) whist[i] = 0;
  __syncthreads();
  const int tile = s_tile;
  const int64_t base = (int64_t)tile * kSortTile + (int64_t)warp * 32 * kSortItems;
  const unsigned lt = (1u << lane) - 1u;
  int keys[kSortItems], vals[kSortItems], lrank[kSortItems];
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int64_t e = base + j * 32 + lane;
    const bool valid = e < n;
    keys[j] = valid ? __ldg(kin + e) : 0;
    vals[j] = valid ? (vin ? __ldg(vin + e) : (int)e) : 0;
  }
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int64_t e = base + j * 32 + lane;
    const bool valid = e < n;
    const int dig = valid ? ((unsigned)keys[j] >> shift) & (bins - 1) : bins;
    const unsigned peers = __match_any_sync(0xffffffffu, dig);
    const int before = valid ? whist[warp * bins + dig] : 0;
    __syncwarp();
    if (valid && lane == __ffs(peers) - 1) whist[warp * bins + dig] = before + __popc(peers);
    __syncwarp();
    lrank[j] = before + __popc(peers & lt);
  }
  __syncthreads();
  // global exclusive prefix of the digit histogram (each tile recomputes it)
  const int per = (bins + kSortThreads - 1) / kSortThreads;   // <= 8
  {
    int loc[8];
    int sum = 0;
    for (int k = 0; k < per; ++k) {
      const int dg = tid * per + k;
      loc[k] = dg < bins ? __ldg(hist + dg) : 0;
      sum += loc[k];
    }
    int tot;
    int ex = block_excl_scan(sum, ws, &tot);
    for (int k = 0; k < per; ++k) {
      const int dg = tid * per + k;
      if (dg < bins) tpref[dg] = ex;
      ex += loc[k];
    }
  }
  __syncthreads();
  // per digit: exclusive over warps, tile count, decoupled look-back
  for (int dg = tid; dg < bins; dg += kSortThreads) {
    int run = 0;
    for (int w = 0; w < NW; ++w) {
      const int t = whist[w * bins + dg];
      whist[w * bins + dg] = run;
      run += t;
    }
    unsigned* slot = lookback + (size_t)tile * bins + dg;
    if (tile == 0) {
      st_release_gpu(slot, kFlagP | (unsigned)run);
    } else {
      st_release_gpu(slot, kFlagA | (unsigned)run);
      unsigned excl = 0;
      int t = tile - 1;
      while (true) {
        const unsigned v = ld_acquire_gpu(lookback + (size_t)t * bins + dg);
        const unsigned f = v & ~kCountMask;
        if (f == 0) continue;            // predecessor not published yet
        excl += v & kCountMask;
        if (f == kFlagP) break;
        --t;
      }
      st_release_gpu(slot, kFlagP | (excl + (unsigned)run));
      tpref[dg] += (int)excl;
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int64_t e = base + j * 32 + lane;
    if (e < n) {
      const int dig = ((unsigned)keys[j] >> shift) & (bins - 1);
      const int pos = tpref[dig] + whist[warp * bins + dig] + lrank[j];
      kout[pos] = keys[j];
      vout[pos] = vals[j];
    }
  }
}

// ------------------------------------------------------------------ segmented reduction
// Warp per chunk of kChunk sorted entries.  VEC floats per lane per row step.
template <int VEC>
__device__ __forceinline__ void load_row(const float* __restrict__ src, int cols, int lane, float* v) {
  if (VEC == 4) {
    float4 t = __ldg(reinterpret_cast<const float4*>(src) + lane);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else if (VEC == 2) {
    float2 t = __ldg(reinterpret_cast<const float2*>(src) + lane);
    v[0] = t.x; v[1] = t.y;
  } else {
    v[0] = lane < cols ? __ldg(src + lane) : 0.f;
  }
}

template <int VEC>
__device__ __forceinline__ void store_rmw(float* dst, int cols, int lane, const float* acc) {
  if (VEC == 4) {
    float4* p = reinterpret_cast<float4*>(dst) + lane;
    float4 t = __ldcg(p);
    t.x += acc[0]; t.y += acc[1]; t.z += acc[2]; t.w += acc[3];
    *p = t;
  } else if (VEC == 2) {
    float2* p = reinterpret_cast<float2*>(dst) + lane;
    float2 t = __ldcg(p);
    t.x += acc[0]; t.y += acc[1];
    *p = t;
  } else if (lane < cols) {
    dst[lane] = __ldcg(dst + lane) + acc[0];
  }
}

template <int VEC>
__device__ __forceinline__ void store_plain(float* dst, int cols, int lane, const float* acc) {
  if (VEC == 4) {
    reinterpret_cast<float4*>(dst)[lane] = make_float4(acc[0], acc[1], acc[2], acc[3]);
  } else if (VEC == 2) {
    reinterpret_cast<float2*>(dst)[lane] = make_float2(acc[0], acc[1]);
  } else if (lane < cols) {
    dst[lane] = acc[0];
  }
}

// cols == 32*VEC for VEC in {2, 4}; VEC == 1 handles cols <= 32.
template <int VEC>
__global__ void __launch_bounds__(256) sc_reduce(const int32_t* __restrict__ skeys,
                                                 const int32_t* __restrict__ svals,
                                                 const float* __restrict__ Y, float* W, int cols,
                                                 int64_t n, float* carry, const ScatterStatus* st) {
  if (*(volatile const int*)&st->flag) return;
  const int lane = threadIdx.x & 31;
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int U = 8;   // rows in flight per warp
  for (int64_t c = gw; c < nchunks; c += nwarps) {
    const int64_t c0 = c * kChunk, c1 = min(n, c0 + kChunk);
    const bool first_cont = c0 > 0 && __ldg(skeys + c0) == __ldg(skeys + c0 - 1);
    const bool last_cont = c1 < n && __ldg(skeys + c1 - 1) == __ldg(skeys + c1);
    float acc[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[v] = 0.f;
    bool seg_started_before = first_cont;
    for (int64_t b0 = c0; b0 < c1; b0 += 32) {
      const int64_t e = b0 + lane;
      const int mykey = e < c1 ? __ldg(skeys + e) : -1;
      const int mypos = e < c1 ? __ldg(svals + e) : 0;
      const int nxt = (e + 1 < c1) ? __ldg(skeys + e + 1) : -2;   // -2: chunk end
      const int cnt = (int)(c1 - b0 < 32 ? c1 - b0 : 32);
      for (int j0 = 0; j0 < cnt; j0 += U) {
        float r[U][VEC];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = j0 + u;
          const int pos = __shfl_sync(0xffffffffu, mypos, j & 31);
          if (j < cnt) load_row<VEC>(Y + (size_t)pos * cols, cols, lane, r[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = j0 + u;
          const int key = __shfl_sync(0xffffffffu, mykey, j & 31);
          const int next = __shfl_sync(0xffffffffu, nxt, j & 31);
          if (j < cnt) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) acc[v] += r[u][v];
            if (next != key) {   // segment ends at this entry
              const bool at_chunk_end = (next == -2);
              const bool continues = at_chunk_end && last_cont;
              if (!seg_started_before && !continues) {
                store_rmw<VEC>(W + (size_t)key * cols, cols, lane, acc);
              } else if (seg_started_before) {
                store_plain<VEC>(carry + (size_t)(2 * c) * cols, cols, lane, acc);
              } else {
                store_plain<VEC>(carry + (size_t)(2 * c + 1) * cols, cols, lane, acc);
              }
#pragma unroll
              for (int v = 0; v < VEC; ++v) acc[v] = 0.f;
              seg_started_before = false;
            }
          }
        }
      }
    }
  }
}

// Chains of chunk partials for segments that cross chunk boundaries.
template <int VEC>
__global__ void __launch_bounds__(256) sc_fixup(const int32_t* __restrict__ skeys, float* W, int cols,
                                                int64_t n, const float* __restrict__ carry,
                                                const ScatterStatus* st) {
  if (*(volatile const int*)&st->flag) return;
  __shared__ float part[8][128];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const int64_t c0 = c * kChunk, c1 = min(n, c0 + kChunk);
    const int k0 = __ldg(skeys + c0);
    const bool first_cont = c0 > 0 && k0 == __ldg(skeys + c0 - 1);
    if (!first_cont) continue;
    const bool spans = __ldg(skeys + c1 - 1) == k0 && c1 < n && __ldg(skeys + c1) == k0;
    if (spans) continue;   // not the chain end
    // first occurrence of k0
    int64_t lo = 0, hi = c0;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (__ldg(skeys + mid) < k0) lo = mid + 1; else hi = mid;
    }
    const int64_t cs = lo / kChunk;   // chain start chunk
    // chain items: carry[2*cs+1], carry[2*(cs+1)], ..., carry[2*c]
    const int64_t len = c - cs + 1;
    float acc[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[v] = 0.f;
    for (int64_t i = warp; i < len; i += 8) {
      const int64_t slot = i == 0 ? 2 * cs + 1 : 2 * (cs + i);
      float r[VEC];
      load_row<VEC>(carry + (size_t)slot * cols, cols, lane, r);
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[v] += r[v];
    }
#pragma unroll
    for (int v = 0; v < VEC; ++v) part[warp][lane * VEC + v] = acc[v];
    __syncthreads();
    if (warp == 0) {
      float s[VEC];
#pragma unroll
      for (int v = 0; v < VEC; ++v) s[v] = part[0][lane * VEC + v];
      for (int w = 1; w < 8; ++w)
#pragma unroll
        for (int v = 0; v < VEC; ++v) s[v] += part[w][lane * VEC + v];
      store_rmw<VEC>(W + (size_t)k0 * cols, cols, lane, s);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ atomic path
__global__ void sc_validate(const int32_t* __restrict__ I, int64_t n, int64_t rows, ScatterStatus* st) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += stride) {
    const int key = __ldg(I + e);
    if (key < 0 || (int64_t)key >= rows) {
      atomicMin(&st->bad, ((unsigned long long)e << 32) | (unsigned)key);
      atomicOr(&st->flag, 1);
    }
  }
}

// Lane group of G = cols/4 lanes (<= 32) per entry; 32/G entries per warp step.
__global__ void __launch_bounds__(256) sc_atomic(const int32_t* __restrict__ I, const float* __restrict__ Y,
                                                 float* W, int cols, int64_t n, const ScatterStatus* st) {
  if (*(volatile const int*)&st->flag) return;
  const int lane = threadIdx.x & 31;
  const int q = cols >> 2;                 // quads per row
  const int G = q >= 32 ? 32 : q;          // lanes per entry
  const int per = 32 / G;                  // entries per warp step
  const int sub = lane / G, gl = lane % G;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t e0 = gw * per; e0 < n; e0 += nwarps * per) {
    const int64_t e = e0 + sub;
    if (sub < per && e < n) {
      const int row = __ldg(I + e);
      const float4* src = reinterpret_cast<const float4*>(Y + (size_t)e * cols);
      float* dst = W + (size_t)row * cols;
      for (int f = gl; f < q; f += G) red_add_v4(dst + 4 * f, __ldg(src + f));
    }
  }
}

__global__ void sc_atomic_scalar(const int32_t* __restrict__ I, const float* __restrict__ Y, float* W,
                                 int cols, int64_t n, const ScatterStatus* st) {
  if (*(volatile const int*)&st->flag) return;
  const int64_t total = n * cols;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
    const int64_t e = t / cols;
    const int f = (int)(t % cols);
    atomicAdd(W + (size_t)__ldg(I + e) * cols + f, __ldg(Y + t));
  }
}

// ------------------------------------------------------------------ host side
static int bits_for(int64_t rows) {
  int b = 1;
  while (b < 31 && ((int64_t)1 << b) < rows) ++b;
  return b;
}

ScatterPlan scatter_plan(int64_t rows, int cols, int64_t n, int num_sms) {
  ScatterPlan pl{};
  const int nb = bits_for(rows);
  pl.passes = (nb + 10) / 11;
  pl.bits = (nb + pl.passes - 1) / pl.passes;
  pl.bins = 1 << pl.bits;
  pl.ntiles = (n + kSortTile - 1) / kSortTile;
  pl.nchunks = (n + kChunk - 1) / kChunk;
  pl.num_sms = num_sms;
  // workspace layout (bytes)
  size_t o = 0;
  auto take = [&](size_t b) { size_t r = o; o += (b + 255) & ~size_t(255); return r; };
  pl.off_status = take(sizeof(ScatterStatus));
  pl.off_hist = take(sizeof(int) * pl.passes * pl.bins);
  pl.off_ctr = take(sizeof(unsigned) * 4);
  pl.off_lookback = take(sizeof(unsigned) * pl.passes * pl.ntiles * pl.bins);
  pl.zero_bytes = o;   // everything above is zeroed per call
  pl.off_ka = take(sizeof(int) * n);
  pl.off_va = take(sizeof(int) * n);
  pl.off_kb = take(sizeof(int) * n);
  pl.off_vb = take(sizeof(int) * n);
  pl.off_carry = take(sizeof(float) * 2 * pl.nchunks * cols);
  pl.total_bytes = o;
  return pl;
}

static int vec_for(int cols) {
  if (cols == 128) return 4;
  if (cols == 64) return 2;
  if (cols <= 32) return 1;
  return 0;
}

int scatter_supported(int cols, int mode) {
  if (mode == 0) return vec_for(cols) != 0;
  return 1;
}

cudaError_t scatter_launch(const ScatterPlan& pl, void* ws, float* W, int64_t rows, int cols,
                           const float* Y, const int32_t* I, int64_t n, int mode, cudaStream_t s,
                           int* launches) {
  unsigned char* b = static_cast<unsigned char*>(ws);
  ScatterStatus* st = reinterpret_cast<ScatterStatus*>(b + pl.off_status);
  cudaError_t e = cudaMemsetAsync(b, 0, pl.zero_bytes, s);
  if (e != cudaSuccess) return e;
  // bad starts at "none"
  e = cudaMemsetAsync(&st->bad, 0xff, sizeof(st->bad), s);
  if (e != cudaSuccess) return e;
  const int blocks = pl.num_sms * 4;
  if (mode == 1) {
    sc_validate<<<blocks, 256, 0, s>>>(I, n, rows, st);
    if ((cols & 3) == 0) sc_atomic<<<blocks * 2, 256, 0, s>>>(I, Y, W, cols, n, st);
    else sc_atomic_scalar<<<blocks * 2, 256, 0, s>>>(I, Y, W, cols, n, st);
    *launches += 2;
    return cudaGetLastError();
  }
  int* hist = reinterpret_cast<int*>(b + pl.off_hist);
  unsigned* ctr = reinterpret_cast<unsigned*>(b + pl.off_ctr);
  unsigned* lb = reinterpret_cast<unsigned*>(b + pl.off_lookback);
  int32_t* ka = reinterpret_cast<int32_t*>(b + pl.off_ka);
  int32_t* va = reinterpret_cast<int32_t*>(b + pl.off_va);
  int32_t* kb = reinterpret_cast<int32_t*>(b + pl.off_kb);
  int32_t* vb = reinterpret_cast<int32_t*>(b + pl.off_vb);
  float* carry = reinterpret_cast<float*>(b + pl.off_carry);
  sc_hist<<<blocks, 512, sizeof(int) * pl.passes * pl.bins, s>>>(I, n, rows, pl.passes, pl.bits, hist, st);
  *launches += 1;
  const size_t sm = sizeof(int) * (8 * pl.bins + pl.bins + 32);
  const int32_t* kin = I;
  const int32_t* vin = nullptr;
  for (int p = 0; p < pl.passes; ++p) {
    int32_t* ko = (p & 1) ? kb : ka;
    int32_t* vo = (p & 1) ? vb : va;
    sc_onesweep<<<(unsigned)pl.ntiles, kSortThreads, sm, s>>>(
        kin, vin, ko, vo, n, p * pl.bits, pl.bits, hist + p * pl.bins,
        lb + (size_t)p * pl.ntiles * pl.bins, ctr + p, st);
    *launches += 1;
    kin = ko;
    vin = vo;
  }
  const int vec = vec_for(cols);
  const int rblocks = (int)((pl.nchunks * 32 + 255) / 256);
  switch (vec) {
    case 4:
      sc_reduce<4><<<rblocks, 256, 0, s>>>(kin, vin, Y, W, cols, n, carry, st);
      sc_fixup<4><<<blocks, 256, 0, s>>>(kin, W, cols, n, carry, st);
      break;
    case 2:
      sc_reduce<2><<<rblocks, 256, 0, s>>>(kin, vin, Y, W, cols, n, carry, st);
      sc_fixup<2><<<blocks, 256, 0, s>>>(kin, W, cols, n, carry, st);
      break;
    default:
      sc_reduce<1><<<rblocks, 256, 0, s>>>(kin, vin, Y, W, cols, n, carry, st);
      sc_fixup<1><<<blocks, 256, 0, s>>>(kin, W, cols, n, carry, st);
      break;
  }
  *launches += 2;
  return cudaGetLastError();
}

cudaError_t scatter_prepare(int bins) {
  const size_t sm = sizeof(int) * (8 * bins + bins + 32);
  return cudaFuncSetAttribute(sc_onesweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
}

}  // namespace pg
