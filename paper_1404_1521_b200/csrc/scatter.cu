// scatter.cu -- the paper's advanced-indexing update W[I[k], :] += Y[k, :]
// (the paper's CUDA kernel "each row is indexed in parallel,
// and for each row, each cell in the row is added in parallel")
// as two sm_100a pipelines behind pg_scatter_add:
//
// DET (bit-reproducible), n <= P * 8192 (P = SM count): one cooperative launch
//   (sc_det_owner, scatter_det.cu): bucket sort by owner CTA, per-owner stable
//   sort by row, segmented reduction; Zipf head rows split by position.
// DET, larger n (or PG_SC_DET_SORT set): stable LSD radix sort of (I[k], k) in passes of
//   <= 10-bit digits -- per pass an upsweep (per-tile digit counts), a
//   two-launch scan of the digit-major count matrix and a downsweep (stable
//   in-tile ranks by warp ballots, staged in smem, coalesced write-out) --
//   then a segmented reduction over fixed chunks of kChunk sorted entries:
//   every segment sums its Y rows in k order (Y rows stream through a cp.async
//   ring); segments that cross chunk boundaries leave per-chunk partials that a
//   fix-up kernel combines in chunk order with a fixed-shape tree.  Every row
//   receives exactly ONE vector reduction of its fixed-order total, so the
//   result does not depend on timing.
// ATOMIC: one cooperative streaming pass (sc_atomic_hot): index check, grid
//   barrier, frequent rows summed in shared memory, everything else reaches W
//   by red.global.add.v4.f32 per 16 B (FTZ); no ordering
//   guarantee.
#include "common.cuh"
#include "scatter.cuh"
#include <cstdlib>

namespace pg {

constexpr int kSortThreads = 1024;
constexpr int kSortItems = 8;
constexpr int kSortTile = kSortThreads * kSortItems;   // 8192 keys per tile
constexpr int kMaxDigitBits = 10;
constexpr int kChunk = 256;                             // sorted entries per reduce chunk
constexpr int kScanBlocks = 128;
constexpr int kRing = 16;                               // Y rows staged per reduce warp
constexpr int kRWarps = 8;                              // warps per reduce block

// ------------------------------------------------------------------ radix sort
// Lanes of the warp whose `dig` (bits wide) equals this lane's, among `valid`
// lanes: one ballot per digit bit (match.any is microcoded and slow here).
__device__ __forceinline__ unsigned warp_match(unsigned dig, int bits, bool valid) {
  unsigned peers = __ballot_sync(0xffffffffu, valid);
  for (int b = 0; b < bits; ++b) {
    const bool bit = (dig >> b) & 1u;
    const unsigned bb = __ballot_sync(0xffffffffu, bit);
    peers &= bit ? bb : ~bb;
  }
  return peers;
}

// counts[d * ntiles + tile] = #keys of the tile with digit d (per-warp smem
// histograms, one aggregated atomic per distinct digit per warp step).  With
// rows > 0 (first pass) the indices are also validated.
__global__ void __launch_bounds__(kSortThreads) sc_upsweep(const int32_t* __restrict__ kin, int64_t n, int shift,
                                                           int bits, int64_t rows, int* __restrict__ counts,
                                                           ScatterStatus* st) {
  extern __shared__ int sh[];   // [NW][bins]
  const int bins = 1 << bits, NW = kSortThreads / 32;
  const int tile = blockIdx.x, ntiles = gridDim.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < NW * bins; i += kSortThreads) sh[i] = 0;
  __syncthreads();
  const int64_t base = (int64_t)tile * kSortTile + (int64_t)warp * 32 * kSortItems;
  const unsigned lt = (1u << lane) - 1u;
  int* wh = sh + warp * bins;
  int key[kSortItems];
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int64_t e = base + j * 32 + lane;
    key[j] = e < n ? __ldg(kin + e) : 0;
  }
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int64_t e = base + j * 32 + lane;
    const bool valid = e < n;
    int k = key[j];
    if (valid && rows > 0 && (k < 0 || (int64_t)k >= rows)) {
      atomicMax(&st->nbad, ~(((unsigned long long)e << 32) | (unsigned)k));
      atomicOr(&st->flag, 1);
      k = 0;
    }
    const unsigned dig = ((unsigned)k >> shift) & (bins - 1);
    const unsigned peers = warp_match(dig, bits, valid);
    if (valid && (peers & lt) == 0) atomicAdd(&wh[dig], __popc(peers));
  }
  __syncthreads();
  for (int d = threadIdx.x; d < bins; d += kSortThreads) {
    int c = 0;
    for (int w = 0; w < NW; ++w) c += sh[w * bins + d];
    counts[(size_t)d * ntiles + tile] = c;
  }
}

// Exclusive scan of the digit-major count matrix (m ints) in two launches:
// block b reduces segment [b*m/NB, (b+1)*m/NB) (coalesced), then rescans it
// with the sum of the earlier segments added.
__global__ void __launch_bounds__(256) sc_scan_reduce(const int* __restrict__ a, int m, int* __restrict__ bsum,
                                                      const ScatterStatus* st) {
  __shared__ int ws[32];
  if (*(volatile const int*)&st->flag) return;
  const int s0 = (int)((long long)blockIdx.x * m / gridDim.x);
  const int s1 = (int)((long long)(blockIdx.x + 1) * m / gridDim.x);
  int sum = 0;
#pragma unroll 4
  for (int i = s0 + threadIdx.x; i < s1; i += 256) sum += __ldg(a + i);
  int tot;
  block_excl_scan(sum, ws, &tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(256) sc_scan_apply(int* __restrict__ a, int m, const int* __restrict__ bsum,
                                                     const ScatterStatus* st) {
  __shared__ int ws[32];
  if (*(volatile const int*)&st->flag) return;
  const int s0 = (int)((long long)blockIdx.x * m / gridDim.x);
  const int s1 = (int)((long long)(blockIdx.x + 1) * m / gridDim.x);
  const int pre = (int)threadIdx.x < (int)blockIdx.x ? __ldg(bsum + threadIdx.x) : 0;
  int carry;
  block_excl_scan(pre, ws, &carry);   // sum of the earlier segments
  for (int r0 = s0; r0 < s1; r0 += 256 * 4) {
    int v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = r0 + threadIdx.x * 4 + k;
      v[k] = i < s1 ? a[i] : 0;
    }
    int rt;
    int ex = carry + block_excl_scan(v[0] + v[1] + v[2] + v[3], ws, &rt);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = r0 + threadIdx.x * 4 + k;
      if (i < s1) a[i] = ex;
      ex += v[k];
    }
    carry += rt;
  }
}

// Stable in-tile ranking by warp ballots, then the tile is staged in digit
// order in smem and written out with coalesced runs.
// dynamic smem: whist[NW][bins] + tpref[bins] + tstart[bins] + skey[tile] + sval[tile]
__global__ void __launch_bounds__(kSortThreads) sc_downsweep(
    const int32_t* __restrict__ kin, const int32_t* __restrict__ vin, int32_t* __restrict__ kout,
    int32_t* __restrict__ vout, int64_t n, int shift, int bits, const int* __restrict__ offs,
    const ScatterStatus* st) {
  extern __shared__ int sh[];
  __shared__ int ws[32];
  const int bins = 1 << bits, NW = kSortThreads / 32;
  int* whist = sh;
  int* tpref = whist + NW * bins;
  int* tstart = tpref + bins;
  int* skey = tstart + bins;
  int* sval = skey + kSortTile;
  if (*(volatile const int*)&st->flag) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile = blockIdx.x, ntiles = gridDim.x;
  for (int i = tid; i < NW * bins; i += kSortThreads) whist[i] = 0;
  for (int d = tid; d < bins; d += kSortThreads) tpref[d] = __ldg(offs + (size_t)d * ntiles + tile);
  __syncthreads();
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
    const unsigned dig = valid ? ((unsigned)keys[j] >> shift) & (bins - 1) : 0u;
    const unsigned peers = warp_match(dig, bits, valid);
    const int before = valid ? whist[warp * bins + dig] : 0;
    __syncwarp();
    if (valid && (peers & lt) == 0) whist[warp * bins + dig] = before + __popc(peers);
    __syncwarp();
    lrank[j] = before + __popc(peers & lt);
  }
  __syncthreads();
  // per digit: exclusive over warps (warp order == position order) and the tile
  // total; then the in-tile digit starts (exclusive over digits)
  const int per = (bins + kSortThreads - 1) / kSortThreads;   // <= 1 (bins <= 1024)
  int tot_d[4];
  int sum = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    tot_d[k] = 0;
    const int dg = tid * per + k;
    if (k < per && dg < bins) {
      int run = 0;
      for (int w = 0; w < NW; ++w) {
        const int t = whist[w * bins + dg];
        whist[w * bins + dg] = run;
        run += t;
      }
      tot_d[k] = run;
      sum += run;
    }
  }
  int all;
  int ex = block_excl_scan(sum, ws, &all);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int dg = tid * per + k;
    if (k < per && dg < bins) { tstart[dg] = ex; ex += tot_d[k]; }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int64_t e = base + j * 32 + lane;
    if (e < n) {
      const int dig = ((unsigned)keys[j] >> shift) & (bins - 1);
      const int loc = tstart[dig] + whist[warp * bins + dig] + lrank[j];
      skey[loc] = keys[j];
      sval[loc] = vals[j];
    }
  }
  __syncthreads();
  const int64_t rem = n - (int64_t)tile * kSortTile;
  const int cnt = (int)(rem < kSortTile ? rem : kSortTile);
#pragma unroll 4
  for (int i = tid; i < cnt; i += kSortThreads) {
    const int k = skey[i];
    const int dig = ((unsigned)k >> shift) & (bins - 1);
    const int pos = tpref[dig] + (i - tstart[dig]);
    kout[pos] = k;
    vout[pos] = sval[i];
  }
}

#ifdef PG_TRACE
__device__ unsigned long long g_sort_tr[160][16];
#define SORT_MARK(k)                                                                          \
  do {                                                                                        \
    if (threadIdx.x == 0) {                                                                   \
      unsigned long long t_;                                                                  \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                  \
      g_sort_tr[blockIdx.x][k] = t_;                                                          \
    }                                                                                         \
  } while (0)
#else
#define SORT_MARK(k) do {} while (0)
#endif

// All radix passes in ONE cooperative launch when the keys fit one tile per CTA
// (n <= gridDim.x * kSortTile).  Per pass: stable in-tile ranking (warp
// ballots, as sc_downsweep) with the keys held in registers, tile digit totals
// to global -> grid barrier -> CTA q scans the tile column of its digit slice
// (exclusive over tiles) and publishes the digit totals -> grid barrier ->
// every CTA forms its digit bases and scatters its staged tile with coalesced
// runs -> grid barrier before the next pass reads the output.  Pass 0 also
// checks the indices; a bad one stops every CTA after the first barrier.
// dynamic smem: as sc_downsweep.
__global__ void __launch_bounds__(kSortThreads) sc_sort_coop(
    const int32_t* __restrict__ I, int32_t* ka, int32_t* va, int32_t* kb, int32_t* vb, int64_t n,
    int passes, int bits, int64_t rows, int* cnt, int* tot, ScatterStatus* st) {
  extern __shared__ int sh[];
  __shared__ int ws[32];
  const int bins = 1 << bits;
  constexpr int NW = kSortThreads / 32;
  int* whist = sh;
  int* tpref = whist + NW * bins;
  int* tstart = tpref + bins;
  int* skey = tstart + bins;
  int* sval = skey + kSortTile;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile = blockIdx.x, ntiles = gridDim.x;
  const int64_t base = (int64_t)tile * kSortTile + (int64_t)warp * 32 * kSortItems;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t rem = n - (int64_t)tile * kSortTile;
  const int tcnt = (int)(rem < 0 ? 0 : (rem < kSortTile ? rem : kSortTile));
  SORT_MARK(0);
  for (int p = 0; p < passes; ++p) {
    const int shift = p * bits;
    const int32_t* kin = p == 0 ? I : ((p & 1) ? ka : kb);
    const int32_t* vin = p == 0 ? nullptr : ((p & 1) ? va : vb);
    int32_t* kout = (p & 1) ? kb : ka;
    int32_t* vout = (p & 1) ? vb : va;
    for (int i = tid; i < NW * bins; i += kSortThreads) whist[i] = 0;
    __syncthreads();
    int keys[kSortItems], vals[kSortItems], lrank[kSortItems];
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
      const int64_t e = base + j * 32 + lane;
      const bool valid = e < n;
      keys[j] = valid ? __ldcg(kin + e) : 0;
      vals[j] = valid ? (vin ? __ldcg(vin + e) : (int)e) : 0;
    }
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
      const int64_t e = base + j * 32 + lane;
      const bool valid = e < n;
      if (p == 0 && valid && (keys[j] < 0 || (int64_t)keys[j] >= rows)) {
        atomicMax(&st->nbad, ~(((unsigned long long)e << 32) | (unsigned)keys[j]));
        atomicOr(&st->flag, 1);
        keys[j] = 0;
      }
      const unsigned dig = valid ? ((unsigned)keys[j] >> shift) & (bins - 1) : 0u;
      const unsigned peers = warp_match(dig, bits, valid);
      const int before = valid ? whist[warp * bins + dig] : 0;
      __syncwarp();
      if (valid && (peers & lt) == 0) whist[warp * bins + dig] = before + __popc(peers);
      __syncwarp();
      lrank[j] = before + __popc(peers & lt);
    }
    __syncthreads();
    SORT_MARK(1 + 6 * p);
    // per digit: exclusive over warps (warp order == position order), tile total
    int tot_d = 0;
    if (tid < bins) {
      int h[NW];
#pragma unroll
      for (int w = 0; w < NW; ++w) h[w] = whist[w * bins + tid];
      int run = 0;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        whist[w * bins + tid] = run;
        run += h[w];
      }
      tot_d = run;
      cnt[(size_t)tid * ntiles + tile] = run;
    }
    {
      int all;
      const int ex = block_excl_scan(tot_d, ws, &all);
      if (tid < bins) tstart[tid] = ex;
    }
    SORT_MARK(2 + 6 * p);
    grid_barrier(&st->arrivals);
    SORT_MARK(3 + 6 * p);
    if (p == 0 && *(volatile const int*)&st->flag) return;   // every CTA sees the flag now
    // column scans: warp w of CTA q takes digits d = q*NW + w, + ntiles*NW, ...;
    // lane l holds tiles 5l .. 5l+4 (ntiles <= 160), all loads issued at once
    for (int d = tile * NW + warp; d < bins; d += ntiles * NW) {
      int* col = cnt + (size_t)d * ntiles;
      int v[5];
#pragma unroll
      for (int k = 0; k < 5; ++k) v[k] = 5 * lane + k < ntiles ? __ldcg(col + 5 * lane + k) : 0;
      const int mine = v[0] + v[1] + v[2] + v[3] + v[4];
      int x = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      int run = x - mine;
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        if (5 * lane + k < ntiles) col[5 * lane + k] = run;
        run += v[k];
      }
      if (lane == 31) tot[d] = x;
    }
    grid_barrier(&st->arrivals);
    SORT_MARK(4 + 6 * p);
    {   // digit bases (exclusive over digits of the totals) + this tile's column prefix
      const int v = tid < bins ? __ldcg(tot + tid) : 0;
      int all;
      const int ex = block_excl_scan(v, ws, &all);
      if (tid < bins) tpref[tid] = ex + __ldcg(cnt + (size_t)tid * ntiles + tile);
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
      const int64_t e = base + j * 32 + lane;
      if (e < n) {
        const int dig = ((unsigned)keys[j] >> shift) & (bins - 1);
        const int loc = tstart[dig] + whist[warp * bins + dig] + lrank[j];
        skey[loc] = keys[j];
        sval[loc] = vals[j];
      }
    }
    __syncthreads();
#pragma unroll 4
    for (int i = tid; i < tcnt; i += kSortThreads) {
      const int k = skey[i];
      const int dig = ((unsigned)k >> shift) & (bins - 1);
      const int pos = tpref[dig] + (i - tstart[dig]);
      kout[pos] = k;
      vout[pos] = sval[i];
    }
    SORT_MARK(5 + 6 * p);
    if (p + 1 < passes) grid_barrier(&st->arrivals);
    SORT_MARK(6 + 6 * p);
  }
}

// ------------------------------------------------------------------ segmented reduction
template <int VEC>
__device__ __forceinline__ void load_row(const float* __restrict__ src, int cols, int lane, float* v) {
  if (VEC == 4) {
    float4 t = __ldcg(reinterpret_cast<const float4*>(src) + lane);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else if (VEC == 2) {
    float2 t = __ldcg(reinterpret_cast<const float2*>(src) + lane);
    v[0] = t.x; v[1] = t.y;
  } else {
    v[0] = lane < cols ? __ldcg(src + lane) : 0.f;
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

// One vector reduction of a finished row sum onto W.  In DET mode every row
// receives exactly one such add per call (its fixed-order total), so
// W_old + total does not depend on timing; the vector red flushes subnormals.
template <int VEC>
__device__ __forceinline__ void red_row(float* dst, int cols, int lane, const float* acc) {
  if (VEC == 4) {
    red_add_v4(dst + 4 * lane, make_float4(acc[0], acc[1], acc[2], acc[3]));
  } else if (VEC == 2) {   // pair lanes: 16 lanes x 16 B vector reductions
    const float a0 = __shfl_down_sync(0xffffffffu, acc[0], 1);
    const float a1 = __shfl_down_sync(0xffffffffu, acc[1], 1);
    if ((lane & 1) == 0) red_add_v4(dst + 2 * lane, make_float4(acc[0], acc[1], a0, a1));
  } else if (lane < cols) {
    atomicAdd(dst + lane, acc[0]);
  }
}

// Warp per chunk of kChunk sorted entries.  The chunk's (key, pos) pairs are
// staged in smem; Y rows stream through a kRing-row cp.async ring (12 rows in
// flight while 4 are summed), in sorted (= k within a key) order.
// cols == 32*VEC for VEC in {2, 4}; VEC == 1 handles cols <= 32.
template <int VEC>
__global__ void __launch_bounds__(kRWarps * 32) sc_reduce(const int32_t* __restrict__ skeys,
                                                          const int32_t* __restrict__ svals,
                                                          const float* __restrict__ Y, float* W, int cols,
                                                          int64_t n, float* carry, int32_t* cfk, int32_t* clk,
                                                          const ScatterStatus* st) {
  if (*(volatile const int*)&st->flag) return;
  constexpr int RW = 32 * VEC;   // floats per staged row
  extern __shared__ __align__(16) float rsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* ring = rsm + (size_t)warp * (kRing * RW + 2 * kChunk);
  int* kk = reinterpret_cast<int*>(ring + kRing * RW);
  int* pp = kk + kChunk;
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  const int64_t gw = (int64_t)blockIdx.x * kRWarps + warp;
  const int64_t nwarps = (int64_t)gridDim.x * kRWarps;
  for (int64_t c = gw; c < nchunks; c += nwarps) {
    const int64_t c0 = c * kChunk;
    const int cnt = (int)(n - c0 < kChunk ? n - c0 : kChunk);
#pragma unroll 1
    for (int j = lane; j < cnt; j += 32) { kk[j] = __ldg(skeys + c0 + j); pp[j] = __ldg(svals + c0 + j); }
    const int kprev = c0 > 0 ? __ldg(skeys + c0 - 1) : -1;
    const int knext = c0 + cnt < n ? __ldg(skeys + c0 + cnt) : -2;
    __syncwarp();
    if (lane == 0) { cfk[c] = kk[0]; clk[c] = kk[cnt - 1]; }
    const bool first_cont = kk[0] == kprev;
    const bool last_cont = kk[cnt - 1] == knext;
    auto issue = [&](int g) {   // rows 4g .. 4g+3 into their ring slots
      const int r0 = 4 * g;
      if (VEC > 1) {   // 16 B per lane
#pragma unroll
        for (int t = lane; t < 4 * (RW / 4); t += 32) {
          const int rr = t / (RW / 4), q = t % (RW / 4);
          const int j = r0 + rr;
          if (j < cnt) {
            const unsigned sa = (unsigned)__cvta_generic_to_shared(ring + ((j % kRing) * RW) + 4 * q);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa),
                         "l"(Y + (size_t)pp[j] * cols + 4 * q) : "memory");
          }
        }
      } else {         // cols <= 32: 4 B per lane
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
          const int j = r0 + rr;
          if (j < cnt && lane < cols) {
            const unsigned sa = (unsigned)__cvta_generic_to_shared(ring + ((j % kRing) * RW) + lane);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa),
                         "l"(Y + (size_t)pp[j] * cols + lane) : "memory");
          }
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const int ngroups = (cnt + 3) / 4;
    issue(0);
    issue(1);
    issue(2);
    float acc[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[v] = 0.f;
    bool started_before = first_cont;
#pragma unroll 1
    for (int g = 0; g < ngroups; ++g) {
      asm volatile("cp.async.wait_group 2;" ::: "memory");
      __syncwarp();
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = 4 * g + u;
        if (j < cnt) {
          const float* r = ring + (j % kRing) * RW;
#pragma unroll
          for (int v = 0; v < VEC; ++v)
            if (VEC > 1 || lane < cols) acc[v] += r[VEC * lane + v];
          const int key = kk[j];
          const int next = j + 1 < cnt ? kk[j + 1] : -2;
          if (next != key) {   // segment ends at entry j
            const bool continues = next == -2 && last_cont;
            if (!started_before && !continues) red_row<VEC>(W + (size_t)key * cols, cols, lane, acc);
            else if (started_before) store_plain<VEC>(carry + (size_t)(2 * c) * cols, cols, lane, acc);
            else store_plain<VEC>(carry + (size_t)(2 * c + 1) * cols, cols, lane, acc);
#pragma unroll
            for (int v = 0; v < VEC; ++v) acc[v] = 0.f;
            started_before = false;
          }
        }
      }
      __syncwarp();   // the ring slots of group g are free again
      issue(g + 3);
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
  }
}

// Chains of chunk partials for segments that cross chunk boundaries.  Warp w
// of block b checks chunk c = 8b + w.  If c ends a chain (its first segment
// started earlier and ends inside c): a 2-chunk chain is summed by the warp
// (carry[2(c-1)+1] + carry[2c]); a longer chain (a hot row spanning whole
// chunks) is queued and summed by the whole block in chunk order with a fixed
// tree, after a binary search over the per-chunk last keys for its start.
template <int VEC>
__global__ void __launch_bounds__(256) sc_fixup(float* W, int cols, int64_t n, const float* __restrict__ carry,
                                                const int32_t* __restrict__ cfk, const int32_t* __restrict__ clk,
                                                const ScatterStatus* st) {
  if (*(volatile const int*)&st->flag) return;
  __shared__ float part[8][128];
  __shared__ long long lq[8];
  __shared__ int nl;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  if (threadIdx.x == 0) nl = 0;
  __syncthreads();
  const int64_t c = (int64_t)blockIdx.x * 8 + warp;
  if (c > 0 && c < nchunks) {
    const int k0 = __ldcg(cfk + c);
    const bool first_cont = k0 == __ldcg(clk + c - 1);
    const bool spans = __ldcg(clk + c) == k0 && c + 1 < nchunks && __ldcg(cfk + c + 1) == k0;
    if (first_cont && !spans) {
      if (__ldcg(cfk + c - 1) != k0) {   // chain = (c-1, c)
        float a[VEC], b2[VEC];
        load_row<VEC>(carry + (size_t)(2 * (c - 1) + 1) * cols, cols, lane, a);
        load_row<VEC>(carry + (size_t)(2 * c) * cols, cols, lane, b2);
#pragma unroll
        for (int v = 0; v < VEC; ++v) a[v] += b2[v];
        red_row<VEC>(W + (size_t)k0 * cols, cols, lane, a);
      } else if (lane == 0) {
        lq[atomicAdd(&nl, 1)] = c;
      }
    }
  }
  __syncthreads();
  const int nlong = nl;
  for (int qi = 0; qi < nlong; ++qi) {
    const int64_t ce = lq[qi];
    const int k0 = __ldcg(cfk + ce);
    // chain start: the chunk before the run of chunks whose first key is k0
    // (all chunks ce-1, ce-2, ... start with k0); 256 chunks per round trip
    __shared__ long long s_cs;
    if (threadIdx.x == 0) s_cs = -1;
    __syncthreads();
    for (int64_t top = ce - 1; ; top -= 256) {
      const int64_t ci = top - threadIdx.x;
      const bool brk = ci >= 0 && __ldcg(cfk + ci) != k0;   // chunk ci does not start with k0
      const int any = __syncthreads_or(brk);
      if (brk) atomicMax(&s_cs, (long long)ci);
      __syncthreads();
      if (any || top - 255 <= 0) break;
    }
    int64_t cs = s_cs < 0 ? 0 : s_cs;
    if (__ldcg(clk + cs) != k0) ++cs;   // k0 starts exactly at chunk cs+1's first entry
    // chain items: carry[2*cs+1], carry[2*(cs+1)], ..., carry[2*ce]; warp w
    // sums the contiguous part [len*w/8, len*(w+1)/8) in order, 8 loads in flight
    const int64_t len = ce - cs + 1;
    const int64_t i0 = len * warp / 8, i1 = len * (warp + 1) / 8;
    float acc[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[v] = 0.f;
    for (int64_t ib = i0; ib < i1; ib += 8) {
      float r[8][VEC];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int64_t i = ib + k;
        const int64_t slot = i == 0 ? 2 * cs + 1 : 2 * (cs + i);
        if (i < i1) load_row<VEC>(carry + (size_t)slot * cols, cols, lane, r[k]);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (ib + k < i1)
#pragma unroll
          for (int v = 0; v < VEC; ++v) acc[v] += r[k][v];
    }
#pragma unroll
    for (int v = 0; v < VEC; ++v) part[warp][lane * VEC + v] = acc[v];
    __syncthreads();
    if (warp == 0) {
      float sacc[VEC];
#pragma unroll
      for (int v = 0; v < VEC; ++v) sacc[v] = part[0][lane * VEC + v];
      for (int w = 1; w < 8; ++w)
#pragma unroll
        for (int v = 0; v < VEC; ++v) sacc[v] += part[w][lane * VEC + v];
      red_row<VEC>(W + (size_t)k0 * cols, cols, lane, sacc);
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
      atomicMax(&st->nbad, ~(((unsigned long long)e << 32) | (unsigned)key));
      atomicOr(&st->flag, 1);
    }
  }
}

// Cooperative ATOMIC scatter, hot-set form (cols % 4 == 0, cols <= 128).
// Plain per-16 B vector reductions stream at ~4.3 TB/s of Y on uniform
// indices, but the L2 serialises reductions to one line (~5 ns each), so a
// Zipf head row with 80k entries alone would take > 500 us
// (scripts/micro/red_stream.cu, bulk_reduce.cu).  So:
//  1. every CTA checks its grid-strided share of I (all loads issued at once)
//     and arrives at the grid barrier; while the barrier completes it
//     prefetches its share of W into L2 (when W is small next to the L2) and,
//     redundantly and identically, counts a fixed sample (128 evenly spread runs of 32 entries) of
//     kHotSample entries in an smem hash: rows seen >= kHotMin times
//     (relative frequency >~ 0.1 %) are ranked by (count desc, row asc) with a
//     bitonic sort, so every CTA derives the same ranking -- the first ha go to
//     tier A (a private smem accumulator per lane group), the next up to kHotB to
//     tier B (kHotRep replica rows each, in global memory);
//  2. barrier wait (a bad index anywhere means nothing is applied);
//  3. warps take batches of 32 consecutive entries, interleaved over the
//     grid: lane i loads I[b0 + i] and probes the hot set for it, then the
//     lane groups stream the batch's Y rows (evict-first loads, U rows in
//     flight per lane group; row and slot arrive by shuffles): a tier-A row
//     is added into its lane group's private accumulator (a plain
//     read-modify-write, no atomics), a tier-B row goes by red.global.add.v4.f32 to
//     one of its replica rows (by entry position: 1/kHotRep of the per-line
//     serialisation), every other row straight to W the same way;
//  4. tier A (summed over the copies in order) reaches W with one vector
//     reduction per 16 B per CTA; after a second grid barrier, CTA c folds the
//     replica rows of tier-B rows c, c + grid, ... into W and zeroes them for
//     the next call.
// Uniform indices thus stay one streaming pass, and a Zipf head row costs one
// reduction per CTA instead of one per entry.
constexpr int kHotSample = 4096;
constexpr int kHotSampleHash = 8192;   // a multiple of the block size (warp-uniform candidate loop)
constexpr int kHotHash = 1024;
#ifndef PG_AH_HB
#define PG_AH_HB 256
#endif
#ifndef PG_AH_REP
#define PG_AH_REP 16
#endif
#ifndef PG_AH_HA
#define PG_AH_HA 8
#endif
constexpr int kHotB = PG_AH_HB;
constexpr int kHotMin = 4;                          // sample count of a hot row
constexpr int kHotCand = 1024;   // power of two >= kHotSample / kHotMin: every row seen >= kHotMin times
static_assert((kHotCand & (kHotCand - 1)) == 0 && kHotCand >= kHotSample / kHotMin, "candidate array");
constexpr int kHotRep = PG_AH_REP;                         // replica rows per tier-B row
constexpr size_t kHotPrefetchMax = 48u << 20;
#ifndef PG_AH_WPF
#define PG_AH_WPF 2   // W into L2 before the stream: 0 none, 1 per-line prefetch, 2 bulk prefetch
#endif
#ifndef PG_AH_RANK
#define PG_AH_RANK 1
#endif
template <int kThreads, int U>
__global__ void __launch_bounds__(kThreads, 1) sc_atomic_hot(const int32_t* __restrict__ I,
                                                             const float* __restrict__ Y, float* W, int64_t rows,
                                                             int cols, int64_t n, int ha, int hb,
                                                             ScatterStatus* st, int par, float* rep) {
  constexpr int NW = kThreads / 32;
  extern __shared__ __align__(16) unsigned char ah_sm[];
  float* accA = reinterpret_cast<float*>(ah_sm);                                // [NW][ha][cols]
  int* skey = reinterpret_cast<int*>(ah_sm);   // [kHotSampleHash] (aliases the accumulators)
  int* scnt = skey + kHotSampleHash;           // [kHotSampleHash]
  unsigned long long* cand = reinterpret_cast<unsigned long long*>(scnt + kHotSampleHash);   // [kHotCand]
  __shared__ int hkey[kHotHash], hslot[kHotHash], hrow[32 + kHotB];
  __shared__ int ncand;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = cols >> 2;
  const int G = q >= 32 ? 32 : q, per = 32 / G, sub = lane / G, gl = lane % G;
  SORT_MARK(0);
  const int64_t ns = n < kHotSample ? n : kHotSample;
  // the sample: ns / 32 runs of 32 consecutive entries spread evenly over I
  // (one 128 B line per warp load: every CTA reads the same lines, so
  // per-entry strided sampling put 148 x 4096 sector requests on the L2)
  const int64_t nruns = (ns + 31) / 32;
  const int64_t rstride = n / (nruns > 0 ? nruns : 1);
  constexpr int kSPer = (kHotSample + kThreads - 1) / kThreads;
  int samp[kSPer];
#pragma unroll
  for (int j = 0; j < kSPer; ++j) {
    const int64_t i = (int64_t)j * kThreads + tid;
    samp[j] = i < ns ? __ldg(I + (n <= kHotSample ? i : (i >> 5) * rstride + (i & 31))) : -1;
  }
  {   // validation: this CTA's grid-strided share, 4 x int4 per thread per trip
    const int64_t n4 = ((uintptr_t)I & 15) == 0 ? n >> 2 : 0;
    const int4* I4 = reinterpret_cast<const int4*>(I);
    for (int64_t e0 = (int64_t)blockIdx.x * kThreads + tid; e0 < n4; e0 += 4 * (int64_t)gridDim.x * kThreads) {
      int4 v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t e = e0 + (int64_t)j * gridDim.x * kThreads;
        v[j] = e < n4 ? __ldg(I4 + e) : make_int4(0, 0, 0, 0);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t e = e0 + (int64_t)j * gridDim.x * kThreads;
        const int k4[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (e < n4 && (k4[c] < 0 || (int64_t)k4[c] >= rows)) {
            atomicMax(&st->hot[par].nbad, ~(((unsigned long long)(4 * e + c) << 32) | (unsigned)k4[c]));
            atomicOr(&st->hot[par].flag, 1);
          }
      }
    }
    for (int64_t e = 4 * n4 + (int64_t)blockIdx.x * kThreads + tid; e < n; e += (int64_t)gridDim.x * kThreads) {
      const int key = __ldg(I + e);
      if (key < 0 || (int64_t)key >= rows) {
        atomicMax(&st->hot[par].nbad, ~(((unsigned long long)e << 32) | (unsigned)key));
        atomicOr(&st->hot[par].flag, 1);
      }
    }
  }
  // Everything up to grid_wait is CTA-local: it overlaps the barrier.
  SORT_MARK(1);
  const unsigned long long target = grid_arrive(&st->hot_arrivals);
  // W's first touch by a reduction after a cold L2 is an L2 miss the atomic
  // unit waits on; when W is small next to the L2, pull it in while the
  // prologue runs (this CTA's 1/gridDim share).
  if ((size_t)rows * cols * sizeof(float) <= kHotPrefetchMax) {
    const int64_t bytes = (int64_t)rows * cols * (int64_t)sizeof(float);
    const char* wb = reinterpret_cast<const char*>(W);
#if PG_AH_WPF == 2
    // bulk prefetches (16 B granular), one piece per lane of warp 0: a
    // per-line prefetch loop put ~1350 instructions per SM into the LSU queue
    // ahead of the prologue's shared-memory work
    if (warp == 0) {
      const int64_t slice = ((bytes / gridDim.x) + 15) & ~15ll, piece = ((slice / 32) + 15) & ~15ll;
      const int64_t a = (int64_t)blockIdx.x * slice + lane * piece;
      int64_t e = a + piece;
      if (e > (int64_t)(blockIdx.x + 1) * slice) e = (int64_t)(blockIdx.x + 1) * slice;
      if (e > (bytes & ~15ll)) e = bytes & ~15ll;
      if (e > a) {
        unsigned long long pol;
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;"
                     ::"l"(wb + a), "r"((unsigned)(e - a)), "l"(pol) : "memory");
      }
    }
#elif PG_AH_WPF == 1
    const int64_t lines = bytes >> 7;
    for (int64_t l = (int64_t)blockIdx.x * kThreads + tid; l < lines; l += (int64_t)gridDim.x * kThreads)
      asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(wb + (l << 7)));
#endif
  }
  SORT_MARK(9);
  for (int i = tid; i < kHotSampleHash; i += kThreads) { skey[i] = -1; scnt[i] = 0; }
  for (int i = tid; i < kHotHash; i += kThreads) hkey[i] = -1;
  if (tid == 0) ncand = 0;
  __syncthreads();
  SORT_MARK(10);
#pragma unroll
  for (int j = 0; j < kSPer; ++j) {
    const int row = samp[j];
    if (row < 0 || (int64_t)row >= rows) continue;
    unsigned h = ((unsigned)row * 2654435761u) & (kHotSampleHash - 1);
    while (true) {
      const int prev = atomicCAS(&skey[h], -1, row);
      if (prev == -1 || prev == row) break;
      h = (h + 1) & (kHotSampleHash - 1);
    }
    atomicAdd(&scnt[h], 1);
  }
  __syncthreads();
  SORT_MARK(11);
  // candidates: rows seen >= kHotMin times (<= kHotSample / kHotMin = kHotCand
  // of them), ranked by (count desc, row asc) with a bitonic sort, so every
  // CTA derives the same ranking -- tier B's replica rows in global memory
  // must mean the same row in every CTA
  // (one shared-memory atomic per warp and pass: ~150 candidates taking a slot
  // one atomic each were ~1.5 us of serialised atomics on one word)
  for (int s2 = tid; s2 < kHotSampleHash; s2 += kThreads) {   // kHotSampleHash % kThreads == 0
    const int key = skey[s2], ct = scnt[s2];
    const bool take = key != -1 && ct >= kHotMin;
    const unsigned bal = __ballot_sync(0xffffffffu, take);
    int base = 0;
    if (lane == 0 && bal) base = atomicAdd(&ncand, __popc(bal));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (take) cand[base + __popc(bal & ((1u << lane) - 1u))] = ((unsigned long long)(kHotSample - ct) << 32) | (unsigned)key;
  }
  __syncthreads();
  const int nc = ncand;
  const int nh = nc < ha + hb ? nc : ha + hb;
#if PG_AH_RANK
  // rank of candidate a = number of smaller keys (keys are distinct: one per
  // row), counted against every candidate (broadcast smem reads) -- the order
  // a sort would give, without its barriers
  for (int a = tid; a < nc; a += kThreads) {
    const unsigned long long key = cand[a];
    int rk = 0;
#pragma unroll 8
    for (int b = 0; b < nc; ++b) rk += cand[b] < key;   // unrolled: 8 loads in flight
    if (rk < nh) {
      const int r = (int)(unsigned)(key & 0xffffffffull);
      hrow[rk] = r;
      unsigned h = ((unsigned)r * 2654435761u) & (kHotHash - 1);
      while (atomicCAS(&hkey[h], -1, r) != -1) h = (h + 1) & (kHotHash - 1);
      hslot[h] = rk;
    }
  }
  SORT_MARK(12);
#else
  int npow = 1;
  while (npow < nc) npow <<= 1;
  for (int i = nc + tid; i < npow; i += kThreads) cand[i] = ~0ull;
  __syncthreads();
  if (npow >= 32) {
    bitonic_sort_warp(cand, npow);   // strides < 32 in registers (common.cuh)
  } else {
    for (int size = 2; size <= npow; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int t = tid; t < npow / 2; t += kThreads) {
          const int lo2 = 2 * t - (t & (stride - 1)), hi2 = lo2 + stride;
          const bool up = (lo2 & size) == 0;
          const unsigned long long x = cand[lo2], y = cand[hi2];
          if ((x > y) == up) { cand[lo2] = y; cand[hi2] = x; }
        }
        __syncthreads();
      }
  }
  SORT_MARK(12);
  for (int a = tid; a < nh; a += kThreads) {
    const int r = (int)(unsigned)(cand[a] & 0xffffffffull);
    hrow[a] = r;
    unsigned h = ((unsigned)r * 2654435761u) & (kHotHash - 1);
    while (atomicCAS(&hkey[h], -1, r) != -1) h = (h + 1) & (kHotHash - 1);
    hslot[h] = a;
  }
#endif
  const int na = nh < ha ? nh : ha, nb = nh - na;
  __syncthreads();
  // tier A: [NW][na][q] private copies (dense for the rows actually taken)
  const int NC = NW * per;   // tier-A copies: one per lane group (no turn-taking)
  for (int t = tid; t < NC * na * q; t += kThreads)
    reinterpret_cast<float4*>(accA)[t] = make_float4(0.f, 0.f, 0.f, 0.f);
  float4* accw = reinterpret_cast<float4*>(accA) + (size_t)(warp * per + (sub < per ? sub : 0)) * na * q;
  const bool act = sub < per && gl < q;
  // Warp batches of 32 consecutive entries: lane i loads I[b0 + i] and probes
  // the hot set once for it; the lane groups then take the batch's entries
  // `per` at a time (U in flight), row and slot broadcast by shuffles.  Row and
  // entry offsets are 32-bit (the host guarantees rows*cols, n*cols < 2^31).
  auto probe = [&](int r) -> int {
    unsigned hh = ((unsigned)r * 2654435761u) & (kHotHash - 1);
    int k;
    while ((k = hkey[hh]) != -1 && k != r) hh = (hh + 1) & (kHotHash - 1);
    return k == r ? hslot[hh] : -1;
  };
  // batches interleaved over the grid: at any moment the SMs stream
  // neighbouring parts of Y
  const int64_t gstride = (int64_t)gridDim.x * NW * 32;
  int64_t b0 = ((int64_t)blockIdx.x * NW + warp) * 32;
  const int64_t hi_all = n;
  int rl = b0 + lane < hi_all ? __ldg(I + b0 + lane) : -1;   // in flight across the barrier wait
  SORT_MARK(2);
  grid_wait(&st->hot_arrivals, target);
  SORT_MARK(3);
  if (blockIdx.x == 0 && tid == 0) { st->hot[par ^ 1].flag = 0; st->hot[par ^ 1].nbad = 0ull; }
  if (*(volatile const int*)&st->hot[par].flag) return;
  for (; b0 < hi_all; b0 += gstride) {
    const int nb = hi_all - b0 < 32 ? (int)(hi_all - b0) : 32;
    const int sl = (nh > 0 && rl >= 0) ? probe(rl) : -1;
    const int64_t bn = b0 + gstride;
    const int rn = bn + lane < hi_all ? __ldg(I + bn + lane) : -1;   // next batch's rows
    const float4* Yb = reinterpret_cast<const float4*>(Y) + (size_t)b0 * q;
    for (int k0 = 0; k0 < nb; k0 += per * U) {
      float4 v[U];
      int row[U], slot[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + u * per + sub;
        row[u] = __shfl_sync(0xffffffffu, rl, k & 31);
        slot[u] = __shfl_sync(0xffffffffu, sl, k & 31);
        const bool ok = act && k < nb;
        if (!ok) row[u] = -1;
        v[u] = ok ? __ldcs(Yb + k * q + gl) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int sv = row[u] >= 0 ? slot[u] : -1;
        if (row[u] >= 0 && sv < 0) red_add_v4(W + (row[u] * cols + 4 * gl), v[u]);
        if (sv >= na)   // tier B: one of kHotRep replica rows, by entry position
          red_add_v4(rep + ((sv - na) * kHotRep + (k0 + u * per + sub) % kHotRep) * cols + 4 * gl, v[u]);
        if (sv >= 0 && sv < na) {   // this lane group's own copy: a plain read-modify-write
          float4* p = accw + sv * q + gl;
          float4 t = *p;
          t.x += v[u].x; t.y += v[u].y; t.z += v[u].z; t.w += v[u].w;
          *p = t;
        }
      }
    }
    rl = rn;
  }
  SORT_MARK(4);
  __syncthreads();
  SORT_MARK(5);
  for (int t = tid; t < na * q; t += kThreads) {
    const int r = t / q, f = t - r * q;
    const float4* a = reinterpret_cast<const float4*>(accA) + (size_t)r * q + f;
    float4 sm4 = a[0];
    for (int w = 1; w < NC; ++w) {
      const float4 b = a[(size_t)w * na * q];
      sm4.x += b.x; sm4.y += b.y; sm4.z += b.z; sm4.w += b.w;
    }
    red_add_v4(W + (size_t)hrow[r] * cols + 4 * f, sm4);
  }
  SORT_MARK(6);
  if (nb == 0) return;   // identical in every CTA (same sample, same ranking)
  // tier B: after every CTA's reductions have landed, the replica rows are
  // folded into W and cleared for the next call
  grid_barrier(&st->hot_arrivals);
  SORT_MARK(7);
  // items spread over every CTA (item t -> CTA t % grid): with t = CTA-major
  // the 4096 items of 256 tier-B rows at d = 64 landed on 4 CTAs (~7 us tail)
  for (int t = tid * gridDim.x + blockIdx.x; t < nb * q; t += gridDim.x * kThreads) {
    const int j = t / q, f = t - j * q;
    float4* r4 = reinterpret_cast<float4*>(rep + (size_t)j * kHotRep * cols) + f;
    float4 sm4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int r = 0; r < kHotRep; ++r) {
      const float4 b = __ldcg(r4 + (size_t)r * q);
      sm4.x += b.x; sm4.y += b.y; sm4.z += b.z; sm4.w += b.w;
    }
#pragma unroll
    for (int r = 0; r < kHotRep; ++r) __stcg(r4 + (size_t)r * q, make_float4(0.f, 0.f, 0.f, 0.f));
    red_add_v4(W + (size_t)hrow[na + j] * cols + 4 * f, sm4);
  }
  SORT_MARK(8);
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

// sc_atomic_hot: 1024 threads (32 warps: enough rows in flight to stream Y),
// 4 rows in flight per lane group; 512-thread variants measured 20-30 % slower.
// sc_atomic_hot launch shape: 1024 threads (32 warps, the most at 64 registers)
// with 4 rows in flight per lane group; measured slower: 1024 x 2 / x 8 rows,
// 768 x 8, 512 x 8 (history in DESIGN.md 7.2).
constexpr int kHotThreads = 1024;
static const void* const kHotFn = (const void*)sc_atomic_hot<kHotThreads, 4>;
constexpr size_t kHotSmemMax = 200 * 1024;
// tier-A rows (one copy per lane group) and tier-B rows for a row width.
static int hot_copies(int cols) {   // tier-A copies per CTA: one per lane group of cols/4 lanes
  const int q = cols / 4, G = q >= 32 ? 32 : q;
  return (kHotThreads / 32) * (32 / G);
}
static void hot_tiers(int cols, int* ha, int* hb) {
  const size_t row = sizeof(float) * cols;
  int a = (int)(kHotSmemMax / ((size_t)hot_copies(cols) * row));
  // at most 8 tier-A rows: the copies' shared memory shrinks the L1, which the
  // uniform case pays for (12 rows: 85.4 us, 8: 77.9 us L2-flushed) while the
  // Zipf case is no faster with more (88.1 us either way)
  *ha = a > PG_AH_HA ? PG_AH_HA : a;
  (void)a;
  *hb = kHotB;   // tier B lives in global replica rows (ScatterPlan::off_rep)
}
static size_t hot_smem(int ha, int cols) {
  const size_t acc = sizeof(float) * (size_t)hot_copies(cols) * ha * cols;
  const size_t samp = sizeof(int) * 2 * kHotSampleHash + sizeof(unsigned long long) * kHotCand;
  return acc > samp ? acc : samp;
}
static bool g_sort_coop_ok = false;   // sc_sort_coop fits 1 CTA/SM (scatter_prepare)
static int bits_for(int64_t rows) {
  int b = 1;
  while (b < 31 && ((int64_t)1 << b) < rows) ++b;
  return b;
}

ScatterPlan scatter_plan(int64_t rows, int cols, int64_t n, int num_sms) {
  ScatterPlan pl{};
  const int nb = bits_for(rows);
  pl.passes = (nb + kMaxDigitBits - 1) / kMaxDigitBits;
  pl.bits = (nb + pl.passes - 1) / pl.passes;
  pl.bins = 1 << pl.bits;
  pl.ntiles = (n + kSortTile - 1) / kSortTile;
  pl.nchunks = (n + kChunk - 1) / kChunk;
  pl.num_sms = num_sms;
  size_t o = 0;
  auto take = [&](size_t b) { size_t r = o; o += (b + 255) & ~size_t(255); return r; };
  pl.off_status = take(sizeof(ScatterStatus));
  pl.zero_bytes = o;   // only the status block is reset per call
  // ATOMIC tier-B replica rows: kept zero between calls by the kernel itself;
  // at a fixed offset (right after the status) for every plan
  pl.off_rep = take(sizeof(float) * kHotB * kHotRep * 128);
  pl.off_hist = take(sizeof(int) * pl.bins * pl.ntiles);   // digit-major tile counts
  pl.off_ctr = take(sizeof(int) * (kScanBlocks > 1024 ? kScanBlocks : 1024));   // scan partials / digit totals
  pl.off_lookback = take(16);
  pl.off_ka = take(sizeof(int) * n);
  pl.off_va = take(sizeof(int) * n);
  pl.off_kb = take(sizeof(int) * n);
  pl.off_vb = take(sizeof(int) * n);
  pl.off_carry = take(sizeof(float) * 2 * pl.nchunks * cols);
  pl.off_cfk = take(sizeof(int) * pl.nchunks);
  pl.off_clk = take(sizeof(int) * pl.nchunks);
  pl.det_owner = det_owner_ok(rows, cols, n, num_sms) && !getenv("PG_SC_DET_SORT");
  if (pl.det_owner) {
    pl.off_bucket = take(sizeof(int2) * n);
    pl.off_hcnt = take(sizeof(unsigned) * num_sms * num_sms);
    pl.off_hpart = take(sizeof(float) * det_owner_hpart_floats(num_sms, cols));
    pl.off_hmask = take(sizeof(int) * det_owner_hmask_ints(num_sms));
  }
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

static size_t reduce_smem(int vec) { return sizeof(float) * kRWarps * (kRing * 32 * vec + 2 * kChunk); }

static size_t downsweep_smem(int bins) {
  return sizeof(int) * ((kSortThreads / 32) * bins + 2 * bins + 2 * kSortTile);
}

cudaError_t scatter_launch(const ScatterPlan& pl, void* ws, float* W, int64_t rows, int cols,
                           const float* Y, const int32_t* I, int64_t n, int mode, cudaStream_t s,
                           int* launches, unsigned long long epoch, int* slot) {
  unsigned char* b = static_cast<unsigned char*>(ws);
  ScatterStatus* st = reinterpret_cast<ScatterStatus*>(b + pl.off_status);
  *slot = -1;
  cudaError_t e;
  if (mode == 1 && (cols & 3) == 0 && cols <= 128 && rows * cols < (1ll << 31) && n * cols < (1ll << 31)) {
    int ha, hb;
    hot_tiers(cols, &ha, &hb);
    const size_t smem = hot_smem(ha, cols);
    int par = (int)(epoch & 1);
    float* rep = reinterpret_cast<float*>(b + pl.off_rep);
    void* args[] = {(void*)&I, (void*)&Y, (void*)&W, (void*)&rows, (void*)&cols, (void*)&n,
                    (void*)&ha, (void*)&hb, (void*)&st, (void*)&par, (void*)&rep};
    *launches += 1;
    *slot = par;
    return cudaLaunchCooperativeKernel(kHotFn, pl.num_sms, kHotThreads, args, smem, s);
  }
  if (mode == 0 && pl.det_owner) {
    const int par = (int)(epoch & 1);
    *launches += 1;
    *slot = par;
    static const long long ypf_mb = getenv("PG_SC_YPF_MB") ? atoll(getenv("PG_SC_YPF_MB")) : 0;
    int64_t ypf = (int64_t)(ypf_mb << 20) >> 7;
    if (ypf > (n * cols * (int64_t)sizeof(float)) >> 7) ypf = (n * cols * (int64_t)sizeof(float)) >> 7;
    return det_owner_launch(I, Y, W, rows, cols, n, st, par, reinterpret_cast<int2*>(b + pl.off_bucket),
                            reinterpret_cast<unsigned*>(b + pl.off_hcnt), reinterpret_cast<float*>(b + pl.off_hpart),
                            reinterpret_cast<int*>(b + pl.off_hmask), pl.num_sms, ypf, s);
  }
  e = cudaMemsetAsync(b, 0, pl.zero_bytes, s);
  if (e != cudaSuccess) return e;
  const int blocks = pl.num_sms * 4;
  if (mode == 1) {
    sc_validate<<<blocks, 256, 0, s>>>(I, n, rows, st);
    if ((cols & 3) == 0) sc_atomic<<<blocks * 2, 256, 0, s>>>(I, Y, W, cols, n, st);
    else sc_atomic_scalar<<<blocks * 2, 256, 0, s>>>(I, Y, W, cols, n, st);
    *launches += 2;
    return cudaGetLastError();
  }
  int* counts = reinterpret_cast<int*>(b + pl.off_hist);
  int* bsum = reinterpret_cast<int*>(b + pl.off_ctr);
  int32_t* ka = reinterpret_cast<int32_t*>(b + pl.off_ka);
  int32_t* va = reinterpret_cast<int32_t*>(b + pl.off_va);
  int32_t* kb = reinterpret_cast<int32_t*>(b + pl.off_kb);
  int32_t* vb = reinterpret_cast<int32_t*>(b + pl.off_vb);
  float* carry = reinterpret_cast<float*>(b + pl.off_carry);
  int32_t* cfk = reinterpret_cast<int32_t*>(b + pl.off_cfk);
  int32_t* clk = reinterpret_cast<int32_t*>(b + pl.off_clk);
  const size_t smu = sizeof(int) * (kSortThreads / 32) * pl.bins;
  const size_t smd = downsweep_smem(pl.bins);
  const int m = (int)(pl.bins * pl.ntiles);
  const int32_t* kin = I;
  const int32_t* vin = nullptr;
  if (pl.ntiles <= pl.num_sms && pl.bins <= kSortThreads && g_sort_coop_ok) {
    int ntl = (int)pl.ntiles, passes = pl.passes, bits = pl.bits;
    int* tot = bsum;
    void* args[] = {(void*)&I, (void*)&ka, (void*)&va, (void*)&kb, (void*)&vb, (void*)&n, (void*)&passes,
                    (void*)&bits, (void*)&rows, (void*)&counts, (void*)&tot, (void*)&st};
    e = cudaLaunchCooperativeKernel((const void*)sc_sort_coop, ntl, kSortThreads, args, smd, s);
    if (e != cudaSuccess) return e;
    *launches += 1;
    kin = ((pl.passes - 1) & 1) ? kb : ka;   // the last pass's output
    vin = ((pl.passes - 1) & 1) ? vb : va;
  } else
  for (int p = 0; p < pl.passes; ++p) {
    int32_t* ko = (p & 1) ? kb : ka;
    int32_t* vo = (p & 1) ? vb : va;
    sc_upsweep<<<(unsigned)pl.ntiles, kSortThreads, smu, s>>>(kin, n, p * pl.bits, pl.bits, p == 0 ? rows : 0,
                                                               counts, st);
    sc_scan_reduce<<<kScanBlocks, 256, 0, s>>>(counts, m, bsum, st);
    sc_scan_apply<<<kScanBlocks, 256, 0, s>>>(counts, m, bsum, st);
    sc_downsweep<<<(unsigned)pl.ntiles, kSortThreads, smd, s>>>(kin, vin, ko, vo, n, p * pl.bits, pl.bits, counts,
                                                                 st);
    *launches += 4;
    kin = ko;
    vin = vo;
  }
  const int vec = vec_for(cols);
  const int rblocks = (int)((pl.nchunks + kRWarps - 1) / kRWarps);
  const int fblocks = (int)((pl.nchunks + 7) / 8);
  switch (vec) {
    case 4:
      sc_reduce<4><<<rblocks, kRWarps * 32, reduce_smem(4), s>>>(kin, vin, Y, W, cols, n, carry, cfk, clk, st);
      sc_fixup<4><<<fblocks, 256, 0, s>>>(W, cols, n, carry, cfk, clk, st);
      break;
    case 2:
      sc_reduce<2><<<rblocks, kRWarps * 32, reduce_smem(2), s>>>(kin, vin, Y, W, cols, n, carry, cfk, clk, st);
      sc_fixup<2><<<fblocks, 256, 0, s>>>(W, cols, n, carry, cfk, clk, st);
      break;
    default:
      sc_reduce<1><<<rblocks, kRWarps * 32, reduce_smem(1), s>>>(kin, vin, Y, W, cols, n, carry, cfk, clk, st);
      sc_fixup<1><<<fblocks, 256, 0, s>>>(W, cols, n, carry, cfk, clk, st);
      break;
  }
  *launches += 2;
  return cudaGetLastError();
}

cudaError_t scatter_prepare(int bins) {
  cudaError_t e = cudaFuncSetAttribute(sc_downsweep, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)downsweep_smem(bins));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(sc_sort_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)downsweep_smem(bins));
  if (e == cudaSuccess) {
    int b = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, sc_sort_coop, kSortThreads, downsweep_smem(bins));
    g_sort_coop_ok = e == cudaSuccess && b >= 1;
  }
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(sc_upsweep, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(sizeof(int) * (kSortThreads / 32) * bins));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(kHotFn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kHotSmemMax);
  if (e == cudaSuccess) e = det_owner_prepare();
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(sc_reduce<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)reduce_smem(4));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(sc_reduce<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)reduce_smem(2));
  return e;
}

}  // namespace pg

#ifdef PG_TRACE
extern "C" int pg_debug_sort_trace(unsigned long long* out) {   // [160][16] globaltimer stamps
  return (int)cudaMemcpyFromSymbol(out, pg::g_sort_tr, sizeof(pg::g_sort_tr));
}
#endif
