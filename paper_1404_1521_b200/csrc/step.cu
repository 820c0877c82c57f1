// step.cu -- the fused SGD-step kernels for sm_100a.
//
// One step = phase 1 (gather + forward + hinge + backward + CTA-local
// duplicate aggregation of the embedding-gradient rows) and phase 2 (fixed-
// order dense reduction + SGD update of W1/b1/w2, and the embedding
// scatter-add), separated by a grid-wide barrier inside ONE persistent
// cooperative kernel (or, PG_OPT_FUSED=0, by a kernel boundary).
//
// The method (north_star; PAPER.md:98-102 for the scatter; readings G1-G19 in
// DESIGN.md) per example k, centre c = floor(n/2):
//   a_ctx = sum_{p != c} W1_p^T x_p        (shared by both windows)
//   a  = b1 + a_ctx + W1_c^T x_c,  a' = b1 + a_ctx + W1_c^T x'_c
//   z = clamp(a,-1,1); s = w2.z + b2; m = 1 - s + s'; l = max(0, m)
//   g = -[m > 0]/B; delta = g w2 [|a|<1]; delta' = -g w2 [|a'|<1]; sigma = delta + delta'
//   dW1_p += x_p sigma^T (p != c); dW1_c += x_c delta^T + x'_c delta'^T
//   db1 += sigma; dw2 += g (z - z')
//   gradient rows: G_p = W1_p sigma (p != c), G_c = W1_c delta, G'_c = W1_c delta'
// The n+1 rows per example replace the oracle's 2n unmerged rows; in exact
// arithmetic their scatter is identical (reading G7).
//
// Latency structure (the step is latency-bound below B ~ 8k): every global
// round trip is issued for a whole chunk at once -- cp.async for the row
// gather, unrolled loads for W1, the dense partials and the owner lists.
#include <cstdlib>

#include "common.cuh"
#include "step.cuh"

namespace pg {

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// Optional phase timestamps for profiling (PG_OPT_TRACE; thread 0 of each CTA).
// Phase stamps for scripts/trace_step.py: compiled only into the instrumented
// library variant (PG_TRACE, libpg_trace.so) -- the production kernel carries
// no trace code (its instructions would cost instruction-cache space).
#ifdef PG_TRACE
__device__ __forceinline__ void trace_mark(const StepParams& p, int k) {
  if (threadIdx.x == 0 && p.trace != nullptr) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[blockIdx.x * 64 + k] = t;
  }
}
__device__ __forceinline__ void trace_clock(const StepParams& p, int k) {
  if (threadIdx.x == 0 && p.trace != nullptr) p.trace[blockIdx.x * 64 + k] = clock64();
}
#else
__device__ __forceinline__ void trace_mark(const StepParams&, int) {}
__device__ __forceinline__ void trace_clock(const StepParams&, int) {}
#endif

// ------------------------------------------------------------------ error reporting
__device__ __forceinline__ void report_bad(DevStatus* st, long long pos, int value) {
  unsigned long long packed = ((unsigned long long)pos << 32) | (unsigned)value;
  atomicMin(&st->bad, packed);
  atomicOr(&st->flags, 1);
}

// ------------------------------------------------------------------ CTA-local aggregation
// Gradient rows of one chunk: keys rows_s[i], values Gs[i][0..d), i < K in
// (example, slot) order.  Distinct rows are found with an smem hash and placed
// into owner buckets (owner CTA q = row % P) of list L with per-owner offsets
// off[q]; each distinct row's duplicates are summed in i order by the warp that
// owns its entry.  The order of entries INSIDE an owner bucket is irrelevant to
// the arithmetic: a row appears at most once per list, and phase 2 sums a
// row's partials in list order.
__device__ __forceinline__ unsigned hash_row(unsigned row) { return row * 2654435761u; }

// Reset the chunk's hash / bucket state (ordered before use by later barriers).
__device__ __forceinline__ void agg_reset(const StepParams& p, unsigned char* sm) {
  const Layout& lay = p.lay;
  int* hk = reinterpret_cast<int*>(sm + lay.ahk);
  int* hc = reinterpret_cast<int*>(sm + lay.ahc);
  int* ocnt = reinterpret_cast<int*>(sm + lay.ocnt);
  int* ocur = reinterpret_cast<int*>(sm + lay.ocur);
  int* misc = reinterpret_cast<int*>(sm + lay.misc);
  #pragma unroll 1
  for (int i = threadIdx.x; i < 2 * kMaxKeys; i += blockDim.x) { hk[i] = -1; hc[i] = 0; }
  int* ecur = reinterpret_cast<int*>(sm + lay.ecur);
  #pragma unroll 1
  for (int i = threadIdx.x; i < 256; i += blockDim.x) { ocnt[i] = 0; ocur[i] = 0; ecur[i] = 0; }
  if (threadIdx.x == 0) { misc[0] = 0; misc[1] = 0; }
  uint4* am = reinterpret_cast<uint4*>(sm + lay.amask);
  #pragma unroll 1
  for (int i = threadIdx.x; i < 2 * kMaxKeys * (kMaxKeys / 32) / 4; i += blockDim.x) am[i] = make_uint4(0u, 0u, 0u, 0u);
}

// Stable rank of item i inside its bucket: the number of the bucket's members
// below i, read off the bucket's membership bitmask (bit i set for member i;
// NWORDS 32-bit words, built with atomicOr, so the result does not depend on
// the order in which members were discovered).  O(NWORDS) per item.
template <int NWORDS>
__device__ __forceinline__ int mask_rank(const unsigned* mask, int i) {
  const int wi = i >> 5;
  int r = 0;
#pragma unroll
  for (int w4 = 0; w4 < NWORDS / 4; ++w4) {
    if (4 * w4 <= wi) {
      const uint4 m4 = reinterpret_cast<const uint4*>(mask)[w4];
      const unsigned mw[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int w = 4 * w4 + k;
        const unsigned keep = w < wi ? ~0u : (w == wi ? (1u << (i & 31)) - 1u : 0u);
        r += __popc(mw[k] & keep);
      }
    }
  }
  return r;
}

// Ordered sum of the rows src[pos[0..m)] (row stride d) for the features
// f0 + lane + 32k < d, k < 4: 4 independent chains (positions i == c mod 4)
// combined in a fixed order, so the result depends only on the ordered list.
__device__ __forceinline__ float4 ordered_rowsum(const float* src, const unsigned short* pos, int m, int d, int f0) {
  const int lane = threadIdx.x & 31;
  float a[4][4];
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int k = 0; k < 4; ++k) a[c][k] = 0.f;
  bool fk[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) fk[k] = f0 + lane + 32 * k < d;
#pragma unroll 1
  for (int i = 0; i < m; i += 4) {
    // branch-free: clamped positions, masked adds -> the 4 chains overlap
    const float* r[4];
    bool ok[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      ok[c] = i + c < m;
      r[c] = src + (size_t)pos[ok[c] ? i + c : i] * d + f0 + lane;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float v = fk[k] ? r[c][32 * k] : 0.f;
        a[c][k] += ok[c] ? v : 0.f;
      }
  }
  return make_float4((a[0][0] + a[1][0]) + (a[2][0] + a[3][0]), (a[0][1] + a[1][1]) + (a[2][1] + a[3][1]),
                     (a[0][2] + a[1][2]) + (a[2][2] + a[3][2]), (a[0][3] + a[1][3]) + (a[2][3] + a[3][3]));
}

// The same ordered sum for one float4 of the features (q = feature quad) --
// thread-granular, so many (row, quad) items run in parallel.  Identical
// association: chains c = i mod 4, combined (a0 + a1) + (a2 + a3).
__device__ __forceinline__ float4 ordered_quadsum(const float4* src, const unsigned short* pos, int m, int Q, int q) {
  float4 a[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) a[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  // 8 positions per trip (two per chain, in order) so long lists keep 8 loads in flight
#pragma unroll 1
  for (int i = 0; i < m; i += 8) {
    float4 v[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = src[(size_t)pos[i + c < m ? i + c : i] * Q + q];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const bool ok = i + c < m;
      float4& t = a[c & 3];
      t.x += ok ? v[c].x : 0.f;
      t.y += ok ? v[c].y : 0.f;
      t.z += ok ? v[c].z : 0.f;
      t.w += ok ? v[c].w : 0.f;
    }
  }
  return make_float4((a[0].x + a[1].x) + (a[2].x + a[3].x), (a[0].y + a[1].y) + (a[2].y + a[3].y),
                     (a[0].z + a[1].z) + (a[2].z + a[3].z), (a[0].w + a[1].w) + (a[2].w + a[3].w));
}

// Aggregation pass 1 (run as soon as the chunk's row ids are known): insert the
// K row ids into the smem hash (slot per position, multiplicity, membership
// bitmask), count each distinct row for its owner, and number the distinct rows
// u = 0..nU-1 (urow / uslot; the numbering order is arbitrary and only decides
// where a row is staged).  Ends with a barrier; returns nU.
__device__ int agg_insert(const StepParams& p, int K, const int* rows_s, unsigned char* sm) {
  const Layout& lay = p.lay;
  const int tid = threadIdx.x, NT = blockDim.x;
  int* hk = reinterpret_cast<int*>(sm + lay.ahk);
  int* hc = reinterpret_cast<int*>(sm + lay.ahc);
  int* hslot = reinterpret_cast<int*>(sm + lay.aslot);
  int* ocnt = reinterpret_cast<int*>(sm + lay.ocnt);
  int* misc = reinterpret_cast<int*>(sm + lay.misc);
  int* urow = reinterpret_cast<int*>(sm + lay.urow);
  int* uslot = reinterpret_cast<int*>(sm + lay.uslot);
  unsigned* amask = reinterpret_cast<unsigned*>(sm + lay.amask);
  const int P = p.P, HA = 2 * kMaxKeys;
  #pragma unroll 1
  for (int i = tid; i < K; i += NT) {
    const int row = rows_s[i];
    unsigned h = hash_row((unsigned)row) & (HA - 1);
    bool mine = false;
    while (true) {
      const int prev = atomicCAS(&hk[h], -1, row);
      if (prev == -1) { mine = true; break; }
      if (prev == row) break;
      h = (h + 1) & (HA - 1);
    }
    hslot[i] = (int)h;
    atomicAdd(&hc[h], 1);
    atomicOr(&amask[h * (kMaxKeys / 32) + (i >> 5)], 1u << (i & 31));
    if (mine) {
      atomicAdd(&ocnt[(unsigned)row % (unsigned)P], 1);
      const int u = atomicAdd(&misc[1], 1);
      urow[u] = row;
      uslot[u] = (int)h;
    }
  }
  __syncthreads();
  return misc[1];
}

__device__ void aggregate_chunk(const StepParams& p, int L, int K, const int* rows_s,
                                const float* Gs, unsigned char* sm) {
  const Layout& lay = p.lay;
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, warp = tid >> 5, NW = NT >> 5;
  int* hc = reinterpret_cast<int*>(sm + lay.ahc);
  int* hslot = reinterpret_cast<int*>(sm + lay.aslot);
  int* ocnt = reinterpret_cast<int*>(sm + lay.ocnt);
  int* ocur = reinterpret_cast<int*>(sm + lay.ocur);
  int* hj = reinterpret_cast<int*>(sm + lay.hj);
  int* misc = reinterpret_cast<int*>(sm + lay.misc);
  int* ws = reinterpret_cast<int*>(sm + lay.ws);
  const int* urow = reinterpret_cast<const int*>(sm + lay.urow);
  const int* uslot = reinterpret_cast<const int*>(sm + lay.uslot);
  unsigned* amask = reinterpret_cast<unsigned*>(sm + lay.amask);
  const int P = p.P, d = p.d;
  const int nUd = misc[1];   // distinct rows (agg_insert)
  const bool tr = (L % p.R) == 0;
  if (tr) trace_mark(p, 14);
  int32_t* off = p.list_off + (size_t)L * (P + 1);
  int nU;
  {
    const int v = tid < P ? ocnt[tid] : 0;
    const int ex = block_excl_scan(v, ws, &nU);
    if (tid <= P) off[tid] = tid < P ? ex : nU;
    if (tid < P) ocnt[tid] = ex;   // bucket base
  }
  __syncthreads();
  if (tr) trace_mark(p, 15);
  // pass 2: creators take a slot in their owner bucket
  int32_t* lrows = p.list_rows + (size_t)L * p.cap;
  int* ecnt = reinterpret_cast<int*>(sm + lay.ecnt);
  int* eoff = reinterpret_cast<int*>(sm + lay.eoff);
  int* ecur = reinterpret_cast<int*>(sm + lay.ecur);
  unsigned short* spos = reinterpret_cast<unsigned short*>(sm + lay.spos);
  #pragma unroll 1
  for (int u = tid; u < nUd; u += NT) {
    const int row = urow[u], h = uslot[u];
    const int q = (int)((unsigned)row % (unsigned)P);
    const int j = ocnt[q] + atomicAdd(&ocur[q], 1);
    hj[h] = j;
    lrows[j] = row;
    ecnt[j] = hc[h];
  }
  __syncthreads();
  {
    const int v = tid < nU ? ecnt[tid] : 0;
    int tot;
    const int ex = block_excl_scan(v, ws, &tot);
    if (tid <= nU) eoff[tid] = tid < nU ? ex : tot;
  }
  __syncthreads();
  if (tr) trace_mark(p, 16);
  // pass 3: positions grouped by entry, increasing within each entry
  #pragma unroll 1
  for (int i = tid; i < K; i += NT) {
    const int h = hslot[i];
    spos[eoff[hj[h]] + mask_rank<kMaxKeys / 32>(amask + h * (kMaxKeys / 32), i)] = (unsigned short)i;
  }
  __syncthreads();
  if (tr) trace_mark(p, 18);
  // pass 4: ordered sum of each entry's gradient rows, one thread per (entry, quad)
  float* lvals = p.list_vals + (size_t)L * p.cap * d;
  if ((d & 3) == 0) {
    const int Q = d >> 2;
    const float4* G4 = reinterpret_cast<const float4*>(Gs);
#pragma unroll 1
    for (int it = tid; it < nU * Q; it += NT) {
      const int j = it / Q, q = it - j * Q;
      reinterpret_cast<float4*>(lvals + (size_t)j * d)[q] = ordered_quadsum(G4, spos + eoff[j], ecnt[j], Q, q);
    }
  } else {
#pragma unroll 1
    for (int j = warp; j < nU; j += NW) {
      const int m = ecnt[j];
      const unsigned short* ps = spos + eoff[j];
      float* dst = lvals + (size_t)j * d;
#pragma unroll 1
      for (int f0 = 0; f0 < d; f0 += 128) {
        const float4 o4 = ordered_rowsum(Gs, ps, m, d, f0);
        const float out[4] = {o4.x, o4.y, o4.z, o4.w};
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          if (f0 + lane + 32 * kk < d) dst[f0 + lane + 32 * kk] = out[kk];
      }
    }
  }
  if (tr) trace_mark(p, 17);
  __syncthreads();
}

__device__ void write_empty_list(const StepParams& p, int L) {
  int32_t* off = p.list_off + (size_t)L * (p.P + 1);
  #pragma unroll 1
  for (int q = threadIdx.x; q <= p.P; q += blockDim.x) off[q] = 0;
}

// ------------------------------------------------------------------ FAST phase 1
// h == 32 (lane == hidden unit), d % 32 == 0, NW = (n+1)*d/32 warps; warp w owns
// the 32-feature block (slot = w / (d/32), blk = w % (d/32)) of the extended
// input [x_0 .. x_{n-1}, x'_c]; its W1 rows live in registers for the whole
// step (Wcol for the forward, Wrow for the gradient rows).

// Gather the chunk's K = cnt*(n+1) embedding rows.  The index loads are issued
// first (the aggregation reset overlaps them); the row ids go through the
// aggregation hash at once (agg_insert), and only the nU DISTINCT rows are
// copied, to X[u][0..d), with pu[position] = u.  Deduplicating matters under
// Zipf traffic: without it every CTA fetches the hot rows many times and the
// requests pile up on the L2 slices holding them.  16 B cp.async pieces over all
// threads (lower latency than one bulk copy per row; scripts/micro/gather_bench.cu).
// Out-of-range indices are reported and read row 0 (the step is skipped).
template <typename WLoad, typename WPost>
__device__ __forceinline__ void gather_rows(const StepParams& p, unsigned char* sm, long long e0, int cnt,
                                            float* X, int* rows_s, bool tr, WLoad&& wload, WPost&& wpost) {
  const int tid = threadIdx.x, NT = blockDim.x, n = p.n, d = p.d, K = cnt * (n + 1);
  int row = 0, s = 0;
  long long ex = 0;
  if (tid < K) {   // K <= blockDim.x (step_fast_ok)
    const int e = tid / (n + 1);
    s = tid - e * (n + 1);
    ex = e0 + e;
    row = s < n ? __ldg(p.idx + ex * n + s) : __ldg(p.corr + ex);
  }
  asm volatile("" ::: "memory");   // keep the index loads ahead of the caller's loads
  wload();   // caller's register loads, queued behind the index loads
  agg_reset(p, sm);
  if (tid < K) {
    const bool ok = row >= 0 && (long long)row < p.V;
    if (!ok) report_bad(p.st, s < n ? ex * n + s : (long long)p.B * n + ex, row);
    rows_s[tid] = ok ? row : 0;
  }
  __syncthreads();
  if (tr) trace_mark(p, 19);
  const int nU = agg_insert(p, K, rows_s, sm);
  const Layout& lay = p.lay;
  const int* urow = reinterpret_cast<const int*>(sm + lay.urow);
  const int Q = d >> 2;
  #pragma unroll 2
  for (int it = tid; it < nU * Q; it += NT) {
    const int u = it / Q, q = it - u * Q;
    cp_async16(X + (size_t)u * d + 4 * q, p.C + (size_t)urow[u] * d + 4 * q);
  }
  {   // position -> distinct index (slot -> u inverse of uslot)
    int* pu = reinterpret_cast<int*>(sm + lay.pu);
    int* hu = reinterpret_cast<int*>(sm + lay.hj);   // hash slot -> u (hj is rebuilt by the aggregation)
    const int* uslot = reinterpret_cast<const int*>(sm + lay.uslot);
    const int* hslot = reinterpret_cast<const int*>(sm + lay.aslot);
    if (tid < nU) hu[uslot[tid]] = tid;
    __syncthreads();
    if (tid < K) pu[tid] = hu[hslot[tid]];
  }
  wpost();   // caller's work that only needs its own loads, while the rows land
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  if (tr) trace_mark(p, 25);
}

__device__ void phase1_fast(const StepParams& p, unsigned char* sm) {
  const Layout& lay = p.lay;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NW = blockDim.x >> 5;
  const int d = p.d, n = p.n, T = p.T, DB = d >> 5, c = n >> 1;
  const int slot = warp / DB, blk = warp % DB;
  const int wslot = slot == n ? c : slot;
  const int wrow0 = wslot * d + blk * 32;
  const int sel = slot == n ? 2 : (slot == c ? 1 : 0);  // sigma / delta / delta'
  float* X = reinterpret_cast<float*>(sm + lay.xs);
  float* pg = reinterpret_cast<float*>(sm + lay.pg);
  float* sig = reinterpret_cast<float*>(sm + lay.sig);
  float* hinge_s = reinterpret_cast<float*>(sm + lay.hinge);
  int* rows_s = reinterpret_cast<int*>(sm + lay.rows);
  float* red = reinterpret_cast<float*>(sm + lay.red);
  const int* pu = reinterpret_cast<const int*>(sm + lay.pu);
  // this warp's 32 features of example e's slot row (rows are deduplicated: pu)
  auto xrow = [&](int e) -> const float* { return X + (size_t)pu[e * (n + 1) + slot] * d + blk * 32; };

  const long long lo = (long long)(((unsigned long long)blockIdx.x * (unsigned)p.B) / (unsigned)p.P);
  const long long hi = (long long)(((unsigned long long)(blockIdx.x + 1) * (unsigned)p.B) / (unsigned)p.P);
  auto chunk_cnt = [&](int r) -> int {
    const long long e0 = lo + (long long)r * T;
    return (int)(hi - e0 < T ? (hi - e0 > 0 ? hi - e0 : 0) : T);
  };
  const float b1 = __ldg(p.b1 + lane), w2 = __ldg(p.w2 + lane), b2 = __ldg(p.b2);
  float2 dacc[16];   // dW1 rows: dacc[j] = (dW1[wrow0+lane][2j], [2j+1]), FFMA2 pairs
#pragma unroll
  for (int u = 0; u < 16; ++u) dacc[u] = make_float2(0.f, 0.f);
  float acc_db1 = 0.f, acc_dw2 = 0.f, acc_hinge = 0.f;

  // ---- per-CTA dense partial record (after the last chunk's backward, before
  // its aggregation, so the stores drain while the aggregation runs)
  auto write_record = [&]() {
    float* rec = p.dense_part + (size_t)blockIdx.x * p.dense_stride;
    float* dsm = sig;   // [DB][32][33]: the corrupt-centre warps' dW1 rows
    if (slot == n) {
  #pragma unroll
      for (int u = 0; u < 16; ++u) {
        dsm[(blk * 32 + lane) * 33 + 2 * u] = dacc[u].x;
        dsm[(blk * 32 + lane) * 33 + 2 * u + 1] = dacc[u].y;
      }
    }
    red[warp * 32 + lane] = acc_db1;
    red[32 * 32 + warp * 32 + lane] = acc_dw2;
    if (lane == 0) hinge_s[warp] = acc_hinge;
    __syncthreads();
    if (slot < n) {
      if (slot == c) {
  #pragma unroll
        for (int u = 0; u < 16; ++u) {
          dacc[u].x += dsm[(blk * 32 + lane) * 33 + 2 * u];
          dacc[u].y += dsm[(blk * 32 + lane) * 33 + 2 * u + 1];
        }
      }
      float* tile = reinterpret_cast<float*>(sm + lay.wsm) + (size_t)warp * 32 * 33;   // W1 tile is dead now
  #pragma unroll
      for (int u = 0; u < 16; ++u) {
        tile[lane * 33 + 2 * u] = dacc[u].x;
        tile[lane * 33 + 2 * u + 1] = dacc[u].y;
      }
      __syncwarp();
      float4* dst = reinterpret_cast<float4*>(rec + (size_t)wrow0 * 32);
  #pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int t = 4 * (lane + 32 * k), rr = t >> 5, cc = t & 31;
        dst[lane + 32 * k] = make_float4(tile[rr * 33 + cc], tile[rr * 33 + cc + 1], tile[rr * 33 + cc + 2],
                                         tile[rr * 33 + cc + 3]);
      }
    }
    const int ndh = n * d * 32;
    if (tid < 32) {
      float a = 0.f, b = 0.f;
      #pragma unroll 1
      for (int w = 0; w < NW; ++w) { a += red[w * 32 + tid]; b += red[32 * 32 + w * 32 + tid]; }
      rec[ndh + tid] = a;
      rec[ndh + 32 + tid] = b;
    }
    if (tid == 32) {
      float hsum = 0.f;
      #pragma unroll 1
      for (int w = 0; w < NW; ++w) hsum += hinge_s[w];
      rec[ndh + 64] = hsum;
    }
    if (tid >= 64 && tid < 64 + (p.dense_stride - ndh - 65)) rec[ndh + 65 + (tid - 64)] = 0.f;
  };
  const int rlast = (int)((hi - lo - 1) / T);   // last non-empty chunk
#pragma unroll 1
  for (int r = 0; r < p.R; ++r) {
    const long long e0 = lo + (long long)r * T;
    const int cnt = chunk_cnt(r);
    const int L = blockIdx.x * p.R + r;
    if (cnt <= 0) { write_empty_list(p, L); continue; }
    // This warp's W1 block straight into registers (L2-resident after the first
    // CTA touches it), issued before the gather so its latency is hidden:
    // Wcol[k] = W1[wrow0+k][lane] (forward), Wrow[u] = W1[wrow0+lane][u] (backward).
    float2 Wcol[16], Wrow[16];   // (k, k+1) pairs for FFMA2
    float* wt = reinterpret_cast<float*>(sm + lay.wsm) + (size_t)warp * 32 * 33;
    gather_rows(
        p, sm, e0, cnt, X, rows_s, r == 0,
        [&]() {   // coalesced: one 128 B W1 row per load
          const float* wg = p.W1 + (size_t)wrow0 * 32;
#pragma unroll
          for (int j = 0; j < 16; ++j) Wcol[j] = make_float2(__ldg(wg + (2 * j) * 32 + lane), __ldg(wg + (2 * j + 1) * 32 + lane));
        },
        [&]() {   // Wrow = Wcol transposed across the warp, via a padded smem tile
#pragma unroll
          for (int j = 0; j < 16; ++j) { wt[(2 * j) * 33 + lane] = Wcol[j].x; wt[(2 * j + 1) * 33 + lane] = Wcol[j].y; }
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 16; ++j) Wrow[j] = make_float2(wt[lane * 33 + 2 * j], wt[lane * 33 + 2 * j + 1]);
        });
    if (r == 0) trace_mark(p, 1);
    // ---- forward partials: part[warp][e][u] = sum_k x[e][k] W1[wrow0+k][u]
    float* part = pg;
    for (int e = 0; e < cnt; e += 4) {
      // even / odd k in the two halves of an FFMA2 pair, folded at the end
      float2 A0 = make_float2(0.f, 0.f), A1 = A0, A2 = A0, A3 = A0;
      const float4* x0 = reinterpret_cast<const float4*>(xrow(e));
      const float4* x1 = reinterpret_cast<const float4*>(xrow(min(e + 1, cnt - 1)));
      const float4* x2 = reinterpret_cast<const float4*>(xrow(min(e + 2, cnt - 1)));
      const float4* x3 = reinterpret_cast<const float4*>(xrow(min(e + 3, cnt - 1)));
#pragma unroll
      for (int k4 = 0; k4 < 8; ++k4) {
        const float4 v0 = x0[k4], v1 = x1[k4], v2 = x2[k4], v3 = x3[k4];
        A0 = __ffma2_rn(make_float2(v0.x, v0.y), Wcol[2 * k4], A0);
        A1 = __ffma2_rn(make_float2(v1.x, v1.y), Wcol[2 * k4], A1);
        A2 = __ffma2_rn(make_float2(v2.x, v2.y), Wcol[2 * k4], A2);
        A3 = __ffma2_rn(make_float2(v3.x, v3.y), Wcol[2 * k4], A3);
        A0 = __ffma2_rn(make_float2(v0.z, v0.w), Wcol[2 * k4 + 1], A0);
        A1 = __ffma2_rn(make_float2(v1.z, v1.w), Wcol[2 * k4 + 1], A1);
        A2 = __ffma2_rn(make_float2(v2.z, v2.w), Wcol[2 * k4 + 1], A2);
        A3 = __ffma2_rn(make_float2(v3.z, v3.w), Wcol[2 * k4 + 1], A3);
      }
      const float a0 = A0.x + A0.y, a1 = A1.x + A1.y, a2 = A2.x + A2.y, a3 = A3.x + A3.y;
      part[(warp * T + e) * 32 + lane] = a0;
      if (e + 1 < cnt) part[(warp * T + e + 1) * 32 + lane] = a1;
      if (e + 2 < cnt) part[(warp * T + e + 2) * 32 + lane] = a2;
      if (e + 3 < cnt) part[(warp * T + e + 3) * 32 + lane] = a3;
    }
    __syncthreads();
    if (r == 0) trace_mark(p, 2);
    // ---- sigma stage: warp per example, lane = hidden unit; KS examples per
    // pass (e, e + NW, e + 2 NW) so a chunk of <= KS*NW examples takes one pass
    // and the shuffle-reduction chains overlap
    constexpr int KS = 3;
    #pragma unroll 1
    for (int e = warp; e < cnt; e += KS * NW) {
      bool has[KS];
#pragma unroll
      for (int k = 0; k < KS; ++k) has[k] = e + k * NW < cnt;
      // all (n+1)*DB <= 12 block partials in flight at once, then summed per
      // category in ascending block order (context | centre | corrupt centre)
      float v[KS][12];
#pragma unroll
      for (int k = 0; k < KS; ++k)
#pragma unroll
        for (int w = 0; w < 12; ++w) v[k][w] = (has[k] && w < NW) ? part[(w * T + e + k * NW) * 32 + lane] : 0.f;
      float actx[KS], acen[KS], acor[KS];
#pragma unroll
      for (int k = 0; k < KS; ++k) actx[k] = acen[k] = acor[k] = 0.f;
      if (r == 0 && e == 0) trace_mark(p, 27);
#pragma unroll
      for (int w = 0; w < 12; ++w) {   // branch-free: +0.0 into the other categories is exact
        const bool cor = w >= n * DB, cen = !cor && w >= c * DB && w < (c + 1) * DB, ctx = !cor && !cen;
#pragma unroll
        for (int k = 0; k < KS; ++k) {
          acor[k] += cor ? v[k][w] : 0.f;
          acen[k] += cen ? v[k][w] : 0.f;
          actx[k] += ctx ? v[k][w] : 0.f;
        }
      }
      float z[KS], zc[KS], a[KS], ac[KS], sp[KS], spc[KS];
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        const float base = b1 + actx[k];
        a[k] = base + acen[k];
        ac[k] = base + acor[k];
        z[k] = act_f(a[k], p.act);
        zc[k] = act_f(ac[k], p.act);
        sp[k] = w2 * z[k];
        spc[k] = w2 * zc[k];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int k = 0; k < KS; ++k) {
          sp[k] += __shfl_xor_sync(0xffffffffu, sp[k], o);
          spc[k] += __shfl_xor_sync(0xffffffffu, spc[k], o);
        }
      }
      if (r == 0 && e == 0) trace_mark(p, 28);
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        if (!has[k]) break;
        const int ee = e + k * NW;
        const float sv = sp[k] + b2, svc = spc[k] + b2;
        const float m = 1.f - sv + svc;
        const bool active = m > 0.f;
        const float g = active ? -p.inv_B : 0.f;
        const float dl = act_g(g * w2, a[k], z[k], p.act);
        const float dlc = act_g(-g * w2, ac[k], zc[k], p.act);
        const float sg = act_sigma(g * w2, z[k], zc[k], dl, dlc, p.act);
        sig[(0 * T + ee) * 32 + lane] = sg;
        sig[(1 * T + ee) * 32 + lane] = dl;
        sig[(2 * T + ee) * 32 + lane] = dlc;
        acc_db1 += sg;
        acc_dw2 += g * z[k] + (-g) * zc[k];
        if (lane == 0) acc_hinge += active ? m : 0.f;
      }
    }
    __syncthreads();
    if (r == 0) trace_mark(p, 3);
    // ---- backward: gradient rows G[e][slot][blk*32+lane] and dW1 rows,
    // two examples per pass for ILP on the shared-memory broadcasts
    float* Gs = pg;   // part is dead now
    const float* sv_base = sig + sel * T * 32;
    for (int e = 0; e < cnt; e += 2) {
      const bool two = e + 1 < cnt;
      const int e1 = two ? e + 1 : e;
      const float xl0 = xrow(e)[lane], xl1 = two ? xrow(e1)[lane] : 0.f;
      const float4* sv0 = reinterpret_cast<const float4*>(sv_base + e * 32);
      const float4* sv1 = reinterpret_cast<const float4*>(sv_base + e1 * 32);
      float2 G01 = make_float2(0.f, 0.f), G23 = G01, H01 = G01, H23 = G01;
      const float2 x0p = make_float2(xl0, xl0), x1p = make_float2(xl1, xl1);
#pragma unroll
      for (int u4 = 0; u4 < 8; ++u4) {
        const float4 v = sv0[u4], w = sv1[u4];
        const float2 vlo = make_float2(v.x, v.y), vhi = make_float2(v.z, v.w);
        const float2 wlo = make_float2(w.x, w.y), whi = make_float2(w.z, w.w);
        G01 = __ffma2_rn(Wrow[2 * u4], vlo, G01);
        G23 = __ffma2_rn(Wrow[2 * u4 + 1], vhi, G23);
        H01 = __ffma2_rn(Wrow[2 * u4], wlo, H01);
        H23 = __ffma2_rn(Wrow[2 * u4 + 1], whi, H23);
        dacc[2 * u4] = __ffma2_rn(wlo, x1p, __ffma2_rn(vlo, x0p, dacc[2 * u4]));
        dacc[2 * u4 + 1] = __ffma2_rn(whi, x1p, __ffma2_rn(vhi, x0p, dacc[2 * u4 + 1]));
      }
      const float g0 = G01.x, g1 = G01.y, g2 = G23.x, g3 = G23.y, h0 = H01.x, h1 = H01.y, h2 = H23.x, h3 = H23.y;
      Gs[(e * (n + 1) + slot) * d + blk * 32 + lane] = (g0 + g1) + (g2 + g3);
      if (two) Gs[(e1 * (n + 1) + slot) * d + blk * 32 + lane] = (h0 + h1) + (h2 + h3);
    }
    __syncthreads();
    if (r == 0) trace_mark(p, 4);
    if (r == rlast) write_record();
    aggregate_chunk(p, L, cnt * (n + 1), rows_s, Gs, sm);
    if (r == 0) trace_mark(p, 5);
  }
}

// ------------------------------------------------------------------ TILED phase 1
// d % 32 == 0, h % 32 == 0, 64 <= h <= 128 (the large config: d = h = 128):
// chunks of kTT = 16 examples (kTTSmall = 4 when no CTA has more: step_kernel<3>),
// 384 threads, every FMA an FFMA2 with one operand
// broadcast, W1 read from L2 once per chunk per product (no per-thread
// redundancy), all other operands from shared memory.
//   forward  : thread (slot s, hidden pair) accumulates 16 examples over d
//              (x from XT[s][j][0..15] as float4 broadcasts);
//   hinge    : warp per example, lanes over h;
//   G rows   : thread (slot s, feature j) accumulates 16 examples over h
//              (its W1 row, sigma/delta/delta' as [u][e] float4 broadcasts);
//   dW1      : thread (row, 32 hidden) accumulates over the 16 examples and
//              adds into this CTA's dense record (CTA-private, chunk order).
constexpr int kTT = 16;   // chunk size of the tiled path (kTTSmall when every CTA has <= 4 examples)
constexpr int kTTSmall = 4;
constexpr int kTTMid = 8;
template <int TT>
__device__ void phase1_tiled_t(const StepParams& p, unsigned char* sm) {
  constexpr bool kGemm = TT == kTTSmall;   // only the 4-example kernel carries the dW1-GEMM code
  constexpr int XTS = TT + 4;   // XT row stride (floats): TT examples + 4 pad, 16 B aligned
  const Layout& lay = p.lay;
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, warp = tid >> 5, NW = NT >> 5;
  const int d = p.d, n = p.n, h = p.h, E = n + 1, c = n >> 1, H2 = h >> 1;
  float* X = reinterpret_cast<float*>(sm + lay.xs);     // deduped rows [u][d]
  float* part = X;                                      // forward partials [E][T][h]
  float* Gs = X;                                        // gradient rows [T][E][d]
  float* XT = reinterpret_cast<float*>(sm + lay.xt);    // [E][d][T]
  float* SU = reinterpret_cast<float*>(sm + lay.sigu);  // [3][h][T]
  float* SE = reinterpret_cast<float*>(sm + lay.sige);  // [3][T][h]
  float* DW = reinterpret_cast<float*>(sm + lay.dwt);   // [T][h]
  float* hinge_s = reinterpret_cast<float*>(sm + lay.hinge);
  int* rows_s = reinterpret_cast<int*>(sm + lay.rows);
  const int* pu = reinterpret_cast<const int*>(sm + lay.pu);
  float* rec = p.dense_part + (size_t)blockIdx.x * p.dense_stride;
  const int ndh = n * d * h;
  const float b2 = __ldg(p.b2);
  const long long lo = (long long)(((unsigned long long)blockIdx.x * (unsigned)p.B) / (unsigned)p.P);
  const long long hi = (long long)(((unsigned long long)(blockIdx.x + 1) * (unsigned)p.B) / (unsigned)p.P);
  float db1_acc = 0.f, dw2_acc = 0.f, hinge_acc = 0.f;   // thread u < h: db1[u], dw2[u]; thread 0: hinge
#pragma unroll 1
  for (int r = 0; r < p.R; ++r) {
    const long long e0 = lo + (long long)r * TT;
    const int cnt = (int)(hi - e0 < TT ? (hi - e0 > 0 ? hi - e0 : 0) : TT);
    const int L = blockIdx.x * p.R + r;
    if (cnt <= 0) { write_empty_list(p, L); continue; }
    gather_rows(p, sm, e0, cnt, X, rows_s, r == 0, [] {}, [] {});
    // XT[s][j][e] = x of example e, slot s (slot n = corrupt centre); 0 past cnt.
    // Warp per (s, e), lanes over j: conflict-free row reads; the [j][e] rows are
    // XTS floats apart so the column writes are 4-way at worst.
#pragma unroll 1
    for (int se = warp; se < E * TT; se += NW) {
      const int sl = se / TT, e = se - sl * TT;
      const float* xr = X + (size_t)(e < cnt ? pu[e * E + sl] : 0) * d;
      for (int j = lane; j < d; j += 32) XT[((size_t)sl * d + j) * XTS + e] = e < cnt ? xr[j] : 0.f;
    }
    __syncthreads();
    if (r < 2) trace_mark(p, 1 + 32 * r);
    // ---- forward partials part[s][e][u]: thread (slot, hidden pair), 16 examples
#pragma unroll 1
    for (int it = tid; it < E * H2; it += NT) {
      const int sl = it / H2, pp = it - sl * H2, ws = sl == n ? c : sl;
      const float2* wc = reinterpret_cast<const float2*>(p.W1 + (size_t)ws * d * h) + pp;
      const float4* xt = reinterpret_cast<const float4*>(XT + (size_t)sl * d * XTS);
      float2 acc[TT];
#pragma unroll
      for (int e = 0; e < TT; ++e) acc[e] = make_float2(0.f, 0.f);
      // every CTA reads the same W1; rotating the start row per CTA spreads the
      // simultaneous requests over the L2 slices instead of all CTAs hitting
      // the same lines in lockstep
      const int rot = (int)((blockIdx.x * 37u) % (unsigned)d);
#pragma unroll 16
      for (int jj = 0; jj < d; ++jj) {
        const int j = jj + rot < d ? jj + rot : jj + rot - d;
        const float2 w = __ldg(wc + (size_t)j * H2);
#pragma unroll
        for (int q = 0; q < TT / 4; ++q) {
          const float4 x = xt[j * (XTS / 4) + q];
          acc[4 * q] = __ffma2_rn(w, make_float2(x.x, x.x), acc[4 * q]);
          acc[4 * q + 1] = __ffma2_rn(w, make_float2(x.y, x.y), acc[4 * q + 1]);
          acc[4 * q + 2] = __ffma2_rn(w, make_float2(x.z, x.z), acc[4 * q + 2]);
          acc[4 * q + 3] = __ffma2_rn(w, make_float2(x.w, x.w), acc[4 * q + 3]);
        }
      }
#pragma unroll
      for (int e = 0; e < TT; ++e) reinterpret_cast<float2*>(part + ((size_t)sl * TT + e) * h)[pp] = acc[e];
    }
    __syncthreads();
    if (r < 2) trace_mark(p, 2 + 32 * r);
    // ---- hinge, delta, delta', sigma: warp per example, lanes over h (<= 4 per lane)
#pragma unroll 1
    for (int e = warp; e < TT; e += NW) {
      float a[4], ac[4], w2v[4];
      float sp = 0.f, spc = 0.f;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int u = lane + 32 * k;
        a[k] = ac[k] = w2v[k] = 0.f;
        if (u < h) {
          float ctx = __ldg(p.b1 + u);
          for (int sl = 0; sl < n; ++sl)
            if (sl != c) ctx += part[((size_t)sl * TT + e) * h + u];
          a[k] = ctx + part[((size_t)c * TT + e) * h + u];
          ac[k] = ctx + part[((size_t)n * TT + e) * h + u];
          w2v[k] = __ldg(p.w2 + u);
          sp += w2v[k] * act_f(a[k], p.act);
          spc += w2v[k] * act_f(ac[k], p.act);
        }
      }
      sp = warp_sum(sp);
      spc = warp_sum(spc);
      const float m = 1.f - (sp + b2) + (spc + b2);
      const bool active = e < cnt && m > 0.f;
      const float g = active ? -p.inv_B : 0.f;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int u = lane + 32 * k;
        if (u < h) {
          const float z = act_f(a[k], p.act), zc = act_f(ac[k], p.act);
          const float dl = act_g(g * w2v[k], a[k], z, p.act);
          const float dlc = act_g(-g * w2v[k], ac[k], zc, p.act);
          const float sg = act_sigma(g * w2v[k], z, zc, dl, dlc, p.act);
          SU[((size_t)0 * h + u) * XTS + e] = sg;
          SU[((size_t)1 * h + u) * XTS + e] = dl;
          SU[((size_t)2 * h + u) * XTS + e] = dlc;
          SE[((size_t)0 * TT + e) * h + u] = sg;
          SE[((size_t)1 * TT + e) * h + u] = dl;
          SE[((size_t)2 * TT + e) * h + u] = dlc;
          DW[(size_t)e * h + u] = g * z + (-g) * zc;
        }
      }
      if (lane == 0) hinge_s[e] = active ? m : 0.f;
    }
    __syncthreads();
    if (r < 2) trace_mark(p, 3 + 32 * r);
    if (kGemm && p.dw1_gemm) {   // this chunk's inputs and deltas, example-major, for the phase-2 dW1 GEMM
#pragma unroll 1
      for (int t = tid; t < cnt * E * d; t += NT) {
        const int e = t / (E * d), rw = t - e * (E * d);
        p.xg[(size_t)(e0 + e) * E * d + rw] = XT[(size_t)rw * XTS + e];
      }
#pragma unroll 1
      for (int t = tid; t < cnt * 3 * h; t += NT) {
        const int e = t / (3 * h), rw = t - e * (3 * h);
        p.sg[(size_t)(e0 + e) * 3 * h + rw] = SU[(size_t)rw * XTS + e];
      }
    }
    if (tid < h) {   // db1 / dw2 in example order
      for (int e = 0; e < cnt; ++e) { db1_acc += SE[(size_t)e * h + tid]; dw2_acc += DW[(size_t)e * h + tid]; }
    }
    if (tid == 0)
      for (int e = 0; e < cnt; ++e) hinge_acc += hinge_s[e];
    // ---- gradient rows G[e][s][j] = sum_u W1[ws*d+j][u] * cls_s[e][u]: thread per
    // two rows (j, j + d/2) of one slot, lanes over consecutive j, so W1 is read
    // from its transposed mirror W1T[u][row] as coalesced 128 B lines and the
    // sigma/delta float4 broadcasts serve both rows
    {
      const int nd = n * d, D2 = d >> 1;
#pragma unroll 1
      for (int it = tid; it < E * D2; it += NT) {
        const int sl = it / D2, j = it - sl * D2, ws = sl == n ? c : sl;
        const int cls = sl == c ? 1 : (sl == n ? 2 : 0);
        const float* wt = p.W1T + (size_t)ws * d + j;   // rows j and j + D2, + u * nd
        const float4* su = reinterpret_cast<const float4*>(SU + (size_t)cls * h * XTS);
        float2 acc[2][TT / 2];
#pragma unroll
        for (int q = 0; q < TT / 2; ++q) acc[0][q] = acc[1][q] = make_float2(0.f, 0.f);
        const int rot = (int)((blockIdx.x * 37u) % (unsigned)h);   // as in the forward
#pragma unroll 16
        for (int uu = 0; uu < h; ++uu) {
          const int u = uu + rot < h ? uu + rot : uu + rot - h;
          const float w0 = __ldg(wt + (size_t)u * nd), w1 = __ldg(wt + (size_t)u * nd + D2);
#pragma unroll
          for (int q = 0; q < TT / 4; ++q) {
            const float4 sv = su[u * (XTS / 4) + q];
            const float2 lo = make_float2(sv.x, sv.y), hi = make_float2(sv.z, sv.w);
            acc[0][2 * q] = __ffma2_rn(lo, make_float2(w0, w0), acc[0][2 * q]);
            acc[0][2 * q + 1] = __ffma2_rn(hi, make_float2(w0, w0), acc[0][2 * q + 1]);
            acc[1][2 * q] = __ffma2_rn(lo, make_float2(w1, w1), acc[1][2 * q]);
            acc[1][2 * q + 1] = __ffma2_rn(hi, make_float2(w1, w1), acc[1][2 * q + 1]);
          }
        }
#pragma unroll
        for (int rr2 = 0; rr2 < 2; ++rr2)
#pragma unroll
          for (int q = 0; q < TT / 2; ++q) {
            Gs[((size_t)(2 * q) * E + sl) * d + j + rr2 * D2] = acc[rr2][q].x;
            Gs[((size_t)(2 * q + 1) * E + sl) * d + j + rr2 * D2] = acc[rr2][q].y;
          }
      }
    }
    if (r < 2) trace_mark(p, 27 + 32 * r);
    // ---- dW1 rows into this CTA's record (chunk order): warp per row, lane =
    // 4 hidden units; the class's 16 x 4 sigma/delta values sit in registers
    // across rows, x[e] of the row is a float4 broadcast, the record row is
    // read (later chunks) and written as one coalesced 512 B access, with LA
    // record rows of reads in flight.  Centre rows add x'_c * delta' (delta'
    // read from shared memory) before their single write.
    if (!(kGemm && p.dw1_gemm)) {
      const bool first = r == 0;
      const int u0 = 4 * lane;
      const bool has_u = u0 < h;
      const int nA = n * d;
      int cur_cls = -1;
      float2 sreg[TT][2];
      constexpr int LA = 4;   // record-row lookahead
      float4 pre[LA];
#pragma unroll
      for (int k = 0; k < LA; ++k) {
        const int rr = warp + k * NW;
        pre[k] = (rr < nA && has_u && !first) ? __ldcg(reinterpret_cast<const float4*>(rec + (size_t)rr * h) + lane)
                                              : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      int sl = warp / d, j = warp - (warp / d) * d;   // (slot, feature) of row rr, stepped without a division
#pragma unroll 1
      for (int rr = warp; rr < nA; rr += NW, j += NW) {
        while (j >= d) { j -= d; ++sl; }
        const int cls = sl == c ? 1 : 0;
        if (cls != cur_cls) {
          cur_cls = cls;
#pragma unroll
          for (int e = 0; e < TT; ++e) {
            const float4 v = has_u ? *reinterpret_cast<const float4*>(SE + ((size_t)cls * TT + e) * h + u0)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
            sreg[e][0] = make_float2(v.x, v.y);
            sreg[e][1] = make_float2(v.z, v.w);
          }
        }
        const float4* xt4 = reinterpret_cast<const float4*>(XT + ((size_t)sl * d + j) * XTS);
        float2 a0 = make_float2(0.f, 0.f), a1 = a0;
#pragma unroll
        for (int q = 0; q < TT / 4; ++q) {
          const float4 x = xt4[q];
          const float xe[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float2 xp = make_float2(xe[t], xe[t]);
            a0 = __ffma2_rn(sreg[4 * q + t][0], xp, a0);
            a1 = __ffma2_rn(sreg[4 * q + t][1], xp, a1);
          }
        }
        if (cls == 1 && has_u) {   // centre block: + x'_c * delta'
          const float4* xc4 = reinterpret_cast<const float4*>(XT + ((size_t)n * d + j) * XTS);
#pragma unroll
          for (int q = 0; q < TT / 4; ++q) {
            const float4 x = xc4[q];
            const float xe[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const float4 v = *reinterpret_cast<const float4*>(SE + ((size_t)2 * TT + 4 * q + t) * h + u0);
              const float2 xp = make_float2(xe[t], xe[t]);
              a0 = __ffma2_rn(make_float2(v.x, v.y), xp, a0);
              a1 = __ffma2_rn(make_float2(v.z, v.w), xp, a1);
            }
          }
        }
        const float4 prev = pre[0];
#pragma unroll
        for (int t = 0; t + 1 < LA; ++t) pre[t] = pre[t + 1];
        {
          const int rn = rr + LA * NW;
          pre[LA - 1] = (rn < nA && has_u && !first) ? __ldcg(reinterpret_cast<const float4*>(rec + (size_t)rn * h) + lane)
                                                     : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        if (has_u) {
          const float4 o = make_float4(a0.x, a0.y, a1.x, a1.y);
          reinterpret_cast<float4*>(rec + (size_t)rr * h)[lane] =
              first ? o : make_float4(prev.x + o.x, prev.y + o.y, prev.z + o.z, prev.w + o.w);
        }
      }
    }
    __syncthreads();
    if (r < 2) trace_mark(p, 4 + 32 * r);
    aggregate_chunk(p, L, cnt * E, rows_s, Gs, sm);
    if (r < 2) trace_mark(p, 5 + 32 * r);
  }
  if (tid < h) {
    rec[ndh + tid] = db1_acc;
    rec[ndh + h + tid] = dw2_acc;
  }
  if (tid == 0) rec[ndh + 2 * h] = hinge_acc;
  if (tid >= 32 && tid < 32 + (p.dense_stride - ndh - 2 * h - 1)) rec[ndh + 2 * h + 1 + (tid - 32)] = 0.f;
}

// ------------------------------------------------------------------ GENERIC phase 1
// Any (d, n, h) with h <= 128: plain per-thread loops, W1 read through L1.
__device__ void phase1_generic(const StepParams& p, unsigned char* sm) {
  const Layout& lay = p.lay;
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, warp = tid >> 5, NW = NT >> 5;
  const int d = p.d, n = p.n, h = p.h, T = p.T, c = n >> 1, E = (n + 1) * d;
  float* X = reinterpret_cast<float*>(sm + lay.xs);
  float* A = reinterpret_cast<float*>(sm + lay.A);
  float* Ac = reinterpret_cast<float*>(sm + lay.Ac);
  float* SIG = reinterpret_cast<float*>(sm + lay.SIG);
  float* DEL = reinterpret_cast<float*>(sm + lay.DEL);
  float* DELc = reinterpret_cast<float*>(sm + lay.DELc);
  float* gz = reinterpret_cast<float*>(sm + lay.gz);
  float* hinge_s = reinterpret_cast<float*>(sm + lay.hinge);
  int* rows_s = reinterpret_cast<int*>(sm + lay.rows);
  const float* W1 = p.W1;
  const float b2 = __ldg(p.b2);
  float* rec = p.dense_part + (size_t)blockIdx.x * p.dense_stride;
  const int ndh = n * d * h;
  float hinge_acc = 0.f;

  const long long lo = (long long)blockIdx.x * p.B / p.P;
  const long long hi = (long long)(blockIdx.x + 1) * p.B / p.P;
  bool first = true;
  for (int r = 0; r < p.R; ++r) {
    const long long e0 = lo + (long long)r * T;
    const int cnt = (int)(hi - e0 < T ? (hi - e0 > 0 ? hi - e0 : 0) : T);
    const int L = blockIdx.x * p.R + r;
    if (cnt <= 0) { write_empty_list(p, L); continue; }
    agg_reset(p, sm);
    for (int i = tid; i < cnt * (n + 1); i += NT) {
      const int e = i / (n + 1), s = i % (n + 1);
      const long long ex = e0 + e;
      int row = s < n ? __ldg(p.idx + ex * n + s) : __ldg(p.corr + ex);
      const bool ok = row >= 0 && (long long)row < p.V;
      if (!ok) report_bad(p.st, s < n ? ex * n + s : (long long)p.B * n + ex, row);
      rows_s[i] = ok ? row : -1;
    }
    __syncthreads();
    for (int i = tid; i < cnt * E; i += NT) {
      const int e = i / E, s = (i % E) / d, j = i % d;
      const int row = rows_s[e * (n + 1) + s];
      if (row >= 0) cp_async4(X + i, p.C + (size_t)row * d + j);
      else X[i] = 0.f;
    }
    cp_async_wait_all();
    __syncthreads();
    for (int i = tid; i < cnt * (n + 1); i += NT) if (rows_s[i] < 0) rows_s[i] = 0;
    // forward
    for (int i = tid; i < cnt * h; i += NT) {
      const int e = i / h, u = i % h;
      const float* x = X + (size_t)e * E;
      float actx = 0.f, acen = 0.f, acor = 0.f;
      for (int s = 0; s < n; ++s) {
        if (s == c) continue;
        for (int j = 0; j < d; ++j) actx = fmaf(x[s * d + j], __ldg(W1 + (size_t)(s * d + j) * h + u), actx);
      }
      for (int j = 0; j < d; ++j) {
        const float w = __ldg(W1 + (size_t)(c * d + j) * h + u);
        acen = fmaf(x[c * d + j], w, acen);
        acor = fmaf(x[n * d + j], w, acor);
      }
      const float base = __ldg(p.b1 + u) + actx;
      A[i] = base + acen;
      Ac[i] = base + acor;
    }
    __syncthreads();
    for (int e = warp; e < cnt; e += NW) {
      float sp = 0.f, spc = 0.f;
      for (int u = lane; u < h; u += 32) {
        const float w2 = __ldg(p.w2 + u);
        sp += w2 * act_f(A[e * h + u], p.act);
        spc += w2 * act_f(Ac[e * h + u], p.act);
      }
      const float s = warp_sum(sp) + b2, sc = warp_sum(spc) + b2;
      const float m = 1.f - s + sc;
      const bool active = m > 0.f;
      const float g = active ? -p.inv_B : 0.f;
      for (int u = lane; u < h; u += 32) {
        const float w2 = __ldg(p.w2 + u);
        const float dl = act_g(g * w2, A[e * h + u], act_f(A[e * h + u], p.act), p.act);
        const float dlc = act_g(-g * w2, Ac[e * h + u], act_f(Ac[e * h + u], p.act), p.act);
        DEL[e * h + u] = dl; DELc[e * h + u] = dlc;
        SIG[e * h + u] = act_sigma(g * w2, act_f(A[e * h + u], p.act), act_f(Ac[e * h + u], p.act), dl, dlc, p.act);
      }
      if (lane == 0) { gz[e] = g; hinge_s[e] = active ? m : 0.f; }
    }
    __syncthreads();
    for (int i = tid; i < ndh; i += NT) {
      const int row = i / h, u = i % h, s = row / d, j = row % d;
      float acc = 0.f;
      if (s == c) {
        for (int e = 0; e < cnt; ++e)
          acc = fmaf(X[e * E + n * d + j], DELc[e * h + u], fmaf(X[e * E + c * d + j], DEL[e * h + u], acc));
      } else {
        for (int e = 0; e < cnt; ++e) acc = fmaf(X[e * E + s * d + j], SIG[e * h + u], acc);
      }
      rec[i] = first ? acc : rec[i] + acc;
    }
    for (int u = tid; u < h; u += NT) {
      float db = 0.f, dw = 0.f;
      for (int e = 0; e < cnt; ++e) {
        db += SIG[e * h + u];
        const float z = act_f(A[e * h + u], p.act);
        const float zc = act_f(Ac[e * h + u], p.act);
        dw += gz[e] * z + (-gz[e]) * zc;
      }
      rec[ndh + u] = first ? db : rec[ndh + u] + db;
      rec[ndh + h + u] = first ? dw : rec[ndh + h + u] + dw;
    }
    if (tid == 0) for (int e = 0; e < cnt; ++e) hinge_acc += hinge_s[e];
    __syncthreads();
    float* Gs = X;   // G does not read X
    for (int i = tid; i < cnt * E; i += NT) {
      const int e = i / E, s = (i % E) / d, j = i % d;
      const float* vec = s == n ? DELc : (s == c ? DEL : SIG);
      const int ws = s == n ? c : s;
      const float* wr = W1 + (size_t)(ws * d + j) * h;
      float acc = 0.f;
      for (int u = 0; u < h; ++u) acc = fmaf(__ldg(wr + u), vec[e * h + u], acc);
      Gs[i] = acc;
    }
    __syncthreads();
    agg_insert(p, cnt * (n + 1), rows_s, sm);
    aggregate_chunk(p, L, cnt * (n + 1), rows_s, Gs, sm);
    first = false;
  }
  if (first) {
    for (int i = tid; i < p.dense_stride; i += NT) rec[i] = 0.f;
  } else if (tid == 0) {
    rec[ndh + 2 * h] = hinge_acc;
    for (int i = ndh + 2 * h + 1; i < p.dense_stride; ++i) rec[i] = 0.f;
  }
}

// ------------------------------------------------------------------ phase 2
// All of phase 2's global reads are issued before the flag / loss decision is
// consumed, so the bad-index / divergence gate costs no round trip:
//   trip 1: flags, hinge partials, dense partials (+ the params they update),
//           this owner's entry counts in every list;
//   trip 2: the owner's entries (row ids + gradient partials);
//   trip 3: the C rows to update.
// Only the final stores are gated on the decision.
__device__ __forceinline__ float* param_ptr(const StepParams& p, int i, int ndh) {
  if (i < ndh) return p.W1 + i;
  if (i < ndh + p.h) return p.b1 + (i - ndh);
  return p.w2 + (i - ndh - p.h);
}

struct DenseSlice {
  int q0, q1;
};

__device__ __forceinline__ DenseSlice dense_slice(const StepParams& p) {
  // with dw1_gemm the records carry only db1 | dw2 (dW1 is the phase-2 GEMM)
  const int Q0 = p.dw1_gemm ? (p.n * p.d * p.h) / 4 : 0;
  const int NQ = (p.dense_len + 3) / 4 - Q0, G = gridDim.x;
  return {Q0 + (int)((long long)blockIdx.x * NQ / G), Q0 + (int)((long long)(blockIdx.x + 1) * NQ / G)};
}

// dW1 as an output-tiled GEMM over the whole batch (p.dw1_gemm): CTA t takes
// tiles of kGRT dW1 rows (one slot) x kGCT hidden units and stages the tile's
// inputs xg and deltas sg (example-major) in shared memory in example chunks.
// Thread (4 rows x 8 units, split s of kGNS) sums its examples in order
// (register micro-tile: 3 LDS.128 per 32 FMA); the splits are combined in
// order, then W1 (and its transposed mirror) is updated.  16 x 32 tiles: the
// large config (640 x 128) is 160 tiles, two on 12 of the 148 CTAs; 32 x 32
// (80 tiles, one per CTA, 12 splits) measured slower (B = 512: 57.4 against
// 53.3 us) -- a tile's time is its staging plus twice the per-thread sums.
// dW1[slot p] = sum_e x_p sigma^T (context), x_c delta^T + x'_c delta'^T
// (centre) -- the same terms as the per-CTA records, one fixed association.
__device__ __forceinline__ unsigned smem_u32(const void* q) { return (unsigned)__cvta_generic_to_shared(q); }
// One 3-D tensor tile (TMA, cp.async.bulk.tensor) into shared memory, completing on `bar`.
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, unsigned long long* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(smem_u32(dst)), "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)) : "memory");
}

__device__ void dw1_gemm_tiles(const StepParams& p, unsigned char* sm, bool write) {
  constexpr int RT = kGRT, CT = kGCT, EC = kGEC, NS = kGNS;
  const int tid = threadIdx.x, NT = blockDim.x;
  const int d = p.d, n = p.n, h = p.h, B = p.B, c = n >> 1;
  const int rtiles = n * d / RT, ctiles = h / CT, ntiles = rtiles * ctiles;
  // operands staged by TMA (tensor maps over xg / sg, built on the host): one
  // box per operand and pass of EC examples, example-major -- [EC][RT] x rows
  // of the tile's slot (and of the corrupt centre for the centre slot),
  // [EC][CT] deltas; examples past B arrive as zeros.  A ring of kGBUF pass
  // buffers: a tile's first kGBUF passes are all issued at once (B <= 512
  // is one TMA round trip), later passes refill the buffer just consumed.
  constexpr int NB = kGBUF, BUF = 2 * EC * (RT + CT);    // floats per buffer
  unsigned char* base = sm + ((128u - (smem_u32(sm) & 127u)) & 127u);
  float* bufs = reinterpret_cast<float*>(base);          // [NB][xs0 | xs1 | ss0 | ss1]
  float* red = bufs;                                     // [NS][RT * CT], after a tile's last pass
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(bufs + NB * BUF);   // [NB]
  const unsigned char* tmx = reinterpret_cast<const unsigned char*>(p.tmap);
  const unsigned char* tms = tmx + 128;
  if (tid < NB) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + tid)) : "memory");
  if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  unsigned qn = 0;   // passes issued before this tile: pass q uses buffer q % NB, phase (q / NB) & 1
  constexpr int MT = kGMT, CB = CT / 8, KO = (RT * CT + 383) / 384;
  const int mt = tid % MT, split = tid / MT;             // micro-tile (rows 4 rt.., units 8 ct..)
  const int rt = mt / CB, ct = mt - rt * CB;
  const int npass = (B + EC - 1) / EC;
  #pragma unroll 1
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int tr = t / ctiles, tc = t - tr * ctiles;
    const int row0 = tr * RT, sl = row0 / d, j0 = row0 - sl * d, col0 = tc * CT;
    const bool centre = sl == c;
    const int cls = centre ? 1 : 0;
    auto issue = [&](unsigned q, int eb) {   // thread 0: the pass at example eb into buffer q % NB
      float* xb = bufs + (q % NB) * BUF;
      unsigned long long* br = bar + (q % NB);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic accesses before the async writes
      const unsigned bytes = (unsigned)((centre ? 2 : 1) * EC * (RT + CT) * sizeof(float));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(br)), "r"(bytes) : "memory");
      tma_load_3d(xb, tmx, br, j0, sl, eb);
      tma_load_3d(xb + 2 * EC * RT, tms, br, col0, cls, eb);
      if (centre) {
        tma_load_3d(xb + EC * RT, tmx, br, j0, n, eb);
        tma_load_3d(xb + 2 * EC * RT + EC * CT, tms, br, col0, 2, eb);
      }
    };
    __syncthreads();   // the ring is free (the previous tile's split sums are read)
    if (tid == 0)
      for (int k = 0; k < NB && k < npass; ++k) issue(qn + k, k * EC);
    // the tile's current W1 values, read now so the update at the end waits for nothing
    float wcur[KO];
    #pragma unroll
    for (int k = 0; k < KO; ++k) {
      const int o = tid + k * NT;
      wcur[k] = o < RT * CT ? __ldcg(p.W1 + (size_t)(row0 + o / CT) * h + col0 + (o % CT)) : 0.f;
    }
    float2 acc[4][4];   // (unit 2k, 2k+1) pairs: one FFMA2 per pair, the same per-unit rounding as FFMA
    #pragma unroll
    for (int i = 0; i < 4; ++i)
      #pragma unroll
      for (int k = 0; k < 4; ++k) acc[i][k] = make_float2(0.f, 0.f);
    #pragma unroll 1
    for (int ip = 0; ip < npass; ++ip) {
      const unsigned q = qn + ip;
      const int eb = ip * EC, ne = min(EC, B - eb);
      asm volatile(
          "{\n .reg .pred P1;\n WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra WAIT_%=;\n}\n"
          ::"r"(smem_u32(bar + (q % NB))), "r"((q / NB) & 1u) : "memory");
      if (t == blockIdx.x && ip < 2) trace_mark(p, 40 + 2 * ip);
      if (split < NS) {
        const float* xb = bufs + (q % NB) * BUF;
        const int per = (ne + NS - 1) / NS, e0 = split * per, e1 = min(ne, e0 + per);
        for (int k2 = 0; k2 < (centre ? 2 : 1); ++k2) {
          const float* xk = xb + k2 * EC * RT;
          const float* sk = xb + 2 * EC * RT + k2 * EC * CT;
          #pragma unroll 2
          for (int e = e0; e < e1; ++e) {
            const float4 x = *reinterpret_cast<const float4*>(xk + e * RT + 4 * rt);
            const float4 s0 = *reinterpret_cast<const float4*>(sk + e * CT + 8 * ct);
            const float4 s1 = *reinterpret_cast<const float4*>(sk + e * CT + 8 * ct + 4);
            const float xv[4] = {x.x, x.y, x.z, x.w};
            const float2 sv[4] = {make_float2(s0.x, s0.y), make_float2(s0.z, s0.w), make_float2(s1.x, s1.y),
                                  make_float2(s1.z, s1.w)};
            #pragma unroll
            for (int i = 0; i < 4; ++i)
              #pragma unroll
              for (int k = 0; k < 4; ++k) acc[i][k] = __ffma2_rn(make_float2(xv[i], xv[i]), sv[k], acc[i][k]);
          }
        }
      }
      if (ip + NB < npass) {   // refill the buffer just consumed
        __syncthreads();
        if (tid == 0) issue(q + NB, (ip + NB) * EC);
      }
    }
    qn += npass;
    __syncthreads();   // every pass is consumed: the split sums take the ring
    if (t == blockIdx.x) trace_mark(p, 46);
    if (split < NS) {
      #pragma unroll
      for (int i = 0; i < 4; ++i)
        #pragma unroll
        for (int k = 0; k < 4; ++k)
          *reinterpret_cast<float2*>(red + split * RT * CT + (4 * rt + i) * CT + 8 * ct + 2 * k) = acc[i][k];
    }
    __syncthreads();
    if (t == blockIdx.x) trace_mark(p, 47);
    #pragma unroll
    for (int k = 0; k < KO; ++k) {   // splits combined in order; o = row * CT + unit
      const int o = tid + k * NT;
      if (o >= RT * CT || !write) continue;
      float g = red[o];
      #pragma unroll 4
      for (int s2 = 1; s2 < NS; ++s2) g += red[s2 * RT * CT + o];
      const int row = row0 + o / CT, col = col0 + (o % CT);
      const float nw = wcur[k] - p.lr * g;
      p.W1[(size_t)row * h + col] = nw;
      if (p.W1T != nullptr) p.W1T[(size_t)col * (n * d) + row] = nw;
    }
  }
}

// Fixed-order reduction of quads [qb, qb+nq) over the P records: thread
// (quad qi, group g) sums records g, g+G, ... (4 loads in flight).
__device__ __forceinline__ float4 dense_partial(const StepParams& p, int qb, int nq, int groups) {
  const int qi = threadIdx.x % nq, g = threadIdx.x / nq;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (g >= groups) return acc;
  const float* base = p.dense_part + 4 * (qb + qi);
  #pragma unroll 1
  for (int r0 = g; r0 < p.P; r0 += 8 * groups) {   // 8 loads in flight, summed in record order
    float4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int r = r0 + k * groups;
      v[k] = r < p.P ? ldcg4(base + (size_t)r * p.dense_stride) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) { acc.x += v[k].x; acc.y += v[k].y; acc.z += v[k].z; acc.w += v[k].w; }
  }
  return acc;
}

__device__ __forceinline__ int dense_groups(int nq, int NT) {
  int g = NT / nq;
  return g > 32 ? 32 : g;
}

// Combine the groups (in order) and apply W1/b1/w2 -= lr * grad for one block.
__device__ __forceinline__ void dense_apply(const StepParams& p, unsigned char* sm, int qb, int nq, int groups, float4 acc,
                                         float4 cur4, bool write, float* sums_out = nullptr) {
  const float cur[4] = {cur4.x, cur4.y, cur4.z, cur4.w};
  const int tid = threadIdx.x, ndh = p.n * p.d * p.h, DL = p.dense_len;
  float4* dred = reinterpret_cast<float4*>(sm + p.lay.dred);
  const int qi = tid % nq, g = tid / nq;
  if (g < groups) dred[g * nq + qi] = acc;
  __syncthreads();
  if (tid < nq) {
    float4 s = dred[tid];
    #pragma unroll 1
    for (int gg = 1; gg < groups; ++gg) {
      const float4 v = dred[gg * nq + tid];
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    const float sv[4] = {s.x, s.y, s.z, s.w};
    const int base = 4 * (qb + tid);
    if (sums_out) {   // data-parallel record: this rank's summed dense gradient
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (base + k < DL) sums_out[base + k] = sv[k];
    } else if (write) {
      if ((ndh & 3) == 0 && (p.h & 3) == 0) {   // a quad never straddles W1 | b1 | w2
        float* q = param_ptr(p, base, ndh);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (base + k < DL) q[k] = cur[k] - p.lr * sv[k];
        if (p.W1T != nullptr && base < ndh) {   // tiled path: keep W1^T in step
          const int row = base / p.h, u = base - row * p.h, nd = p.n * p.d;
#pragma unroll
          for (int k = 0; k < 4; ++k) p.W1T[(size_t)(u + k) * nd + row] = cur[k] - p.lr * sv[k];
        }
      } else {
#pragma unroll 1
        for (int k = 0; k < 4; ++k)
          if (base + k < DL) *param_ptr(p, base + k, ndh) = cur[k] - p.lr * sv[k];
      }
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------------ phase 2: deterministic scatter
// Bitonic sort of n (power of two) 64-bit keys in smem.
__device__ void bitonic_sort(unsigned long long* k, int n) {
  #pragma unroll 1
  for (int size = 2; size <= n; size <<= 1) {
    #pragma unroll 1
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      #pragma unroll 1
      for (int t = threadIdx.x; t < (n >> 1); t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        unsigned long long a = k[lo], b = k[hi];
        if ((a > b) == up) { k[lo] = b; k[hi] = a; }
      }
      __syncthreads();
    }
  }
}

// One (segment, column) work item of the sorted fallback's window sums: the
// segment's entries [max(s0, sb0), min(s1, sb1)) of staged column `col`
// (units of VT: float or float4) summed in 4 chains by (e - s0) & 3, combined
// as (c0 + c1) + (c2 + c3); a finished segment parks its total in its first
// staged row, a window-crossing one hands its chains on through `carry`
// [2][4][d] floats (the same bytes for either VT).
__device__ __forceinline__ float vzero(float) { return 0.f; }
__device__ __forceinline__ float4 vzero(float4) { return make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ void vadd(float& a, float b) { a += b; }
__device__ __forceinline__ void vadd(float4& a, float4 b) { a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w; }
template <typename VT>
__device__ __forceinline__ void fb_segsum(float* stage, float* carry, int d, int sb0, int sb1, int s0, int s1,
                                          int col, int par) {
  constexpr int VW = sizeof(VT) / sizeof(float);
  const int rs = d / VW;   // row stride in VT units
  VT* st = reinterpret_cast<VT*>(stage);
  VT* cr = reinterpret_cast<VT*>(carry);
  const int a0 = max(s0, sb0), a1 = min(s1, sb1);
  VT c0 = vzero(VT()), c1 = c0, c2 = c0, c3 = c0;
  if (s0 < sb0) {
    c0 = cr[(par * 4 + 0) * rs + col]; c1 = cr[(par * 4 + 1) * rs + col];
    c2 = cr[(par * 4 + 2) * rs + col]; c3 = cr[(par * 4 + 3) * rs + col];
  }
  int ix = (a0 - sb0) * rs + col, e = a0;
  for (; e < a1 && ((e - s0) & 3); ++e, ix += rs) {
    const int k = (e - s0) & 3;
    if (k == 0) vadd(c0, st[ix]); else if (k == 1) vadd(c1, st[ix]); else if (k == 2) vadd(c2, st[ix]); else vadd(c3, st[ix]);
  }
  #pragma unroll 4
  for (; e + 3 < a1; e += 4, ix += 4 * rs) {
    vadd(c0, st[ix]); vadd(c1, st[ix + rs]); vadd(c2, st[ix + 2 * rs]); vadd(c3, st[ix + 3 * rs]);
  }
  for (; e < a1; ++e, ix += rs) {
    const int k = (e - s0) & 3;
    if (k == 0) vadd(c0, st[ix]); else if (k == 1) vadd(c1, st[ix]); else if (k == 2) vadd(c2, st[ix]); else vadd(c3, st[ix]);
  }
  if (s1 <= sb1) {
    vadd(c0, c1); vadd(c2, c3); vadd(c0, c2);
    st[(a0 - sb0) * rs + col] = c0;
  } else {
    cr[((par ^ 1) * 4 + 0) * rs + col] = c0; cr[((par ^ 1) * 4 + 1) * rs + col] = c1;
    cr[((par ^ 1) * 4 + 2) * rs + col] = c2; cr[((par ^ 1) * 4 + 3) * rs + col] = c3;
  }
}

// Sorted fallback for owners with more than MCAP entries (pathological index
// patterns): windows of whole lists, bitonic sort by (row, list), segment sums
// in list order with a carry across staged sub-batches.
// emit_rows == nullptr: C[row] += -lr * total; else the (row, total) pairs are
// written to emit_rows / emit_vals from index 0 on (a row whose entries
// straddle two key windows is emitted twice, its partials in order) and the
// number written is returned.
__device__ int scatter_det_sorted(const StepParams& p, unsigned char* sm, const Lists& ls,
                                  int32_t* emit_rows = nullptr, float* emit_vals = nullptr) {
  const Layout& lay = p.lay;
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, warp = tid >> 5, NW = NT >> 5;
  const int d = p.d, NL = ls.xstride ? p.world : p.NL;
  const int* lbase = reinterpret_cast<const int*>(sm + lay.lbase);
  const int* loff = reinterpret_cast<const int*>(sm + lay.loff);
  int emitted = 0;
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(sm + lay.keys);
  int* seg = reinterpret_cast<int*>(sm + lay.seg);
  float* stage = reinterpret_cast<float*>(sm + lay.stagefb);
  float* carry = reinterpret_cast<float*>(sm + lay.carry);
  int* ws = reinterpret_cast<int*>(sm + lay.ws2);
  const float nlr = -p.lr;
  int La = 0;
  while (La < NL) {
    int Lb = La;
    if (lbase[NL] - lbase[La] <= kCapK) Lb = NL;
    else while (Lb < NL && lbase[Lb + 1] - lbase[La] <= kCapK) ++Lb;
    const int base = lbase[La], Mw = lbase[Lb] - base;
    if (Mw > 0) {
      int npow = 1;
      while (npow < Mw) npow <<= 1;
      #pragma unroll 1
      for (int e = tid; e < npow; e += NT) {
        if (e < Mw) {
          int lo = La, hi = Lb - 1;
          while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (lbase[mid] <= base + e) lo = mid; else hi = mid - 1;
          }
          const int L = lo;
          const int rel = base + e - lbase[L];   // offset inside the owner bucket (< 256)
          // low word: the entry code, which grows with (list, offset) in both
          // layouts (per-CTA lists; ranked records), so sorting by the key
          // orders each row's entries by (list, offset)
          const unsigned li = ls.code(L, loff[L] + rel);
          const unsigned row = (unsigned)__ldcg(ls.row(li));
          keys[e] = ((unsigned long long)row << 32) | (unsigned long long)li;
        } else {
          keys[e] = ~0ull;
        }
      }
      __syncthreads();
      trace_mark(p, 40);
      if (npow >= 32) bitonic_sort_warp(keys, npow); else bitonic_sort(keys, npow);
      trace_mark(p, 41);
      int nseg_total = 0;
      #pragma unroll 1
      for (int e0 = 0; e0 < Mw; e0 += NT) {
        const int e = e0 + tid;
        int head = 0;
        if (e < Mw) head = (e == 0) || ((keys[e] >> 32) != (keys[e - 1] >> 32));
        int tot;
        int ex = block_excl_scan(head, ws, &tot);
        if (e < Mw && head) seg[nseg_total + ex] = e;
        nseg_total += tot;
      }
      if (tid == 0) seg[nseg_total] = Mw;
      __syncthreads();
      trace_mark(p, 42);
      int par = 0;   // carry double buffer: read carry[par], write carry[par ^ 1]
      #pragma unroll 1
      for (int sb0 = 0; sb0 < Mw; sb0 += lay.SB, par ^= 1) {
        const int sb1 = min(Mw, sb0 + lay.SB);
        if ((d & 3) == 0) {   // 16 B pieces, 8 loads in flight per thread
          const int Q = d >> 2, nq = (sb1 - sb0) * Q;
          float4* st4w = reinterpret_cast<float4*>(stage);
          #pragma unroll 1
          for (int t0 = tid; t0 < nq; t0 += 8 * NT) {
            float4 v[8];
            #pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int t = t0 + j * NT;
              if (t < nq) {
                const int e = sb0 + t / Q, f = t - (t / Q) * Q;
                v[j] = __ldcg(reinterpret_cast<const float4*>(ls.val((unsigned)keys[e], d)) + f);
              }
            }
            #pragma unroll
            for (int j = 0; j < 8; ++j)
              if (t0 + j * NT < nq) st4w[t0 + j * NT] = v[j];
          }
        } else {
          #pragma unroll 1
          for (int t = tid; t < (sb1 - sb0) * d; t += NT) {
            const int e = sb0 + t / d, f = t % d;
            stage[t] = __ldcg(ls.val((unsigned)keys[e], d) + f);
          }
        }
        __syncthreads();
        if (sb0 == 0) trace_mark(p, 44);
        if (sb0 / lay.SB < 4) trace_mark(p, 50 + 2 * (sb0 / lay.SB));
        int slo = 0, shi = nseg_total - 1;
        while (slo < shi) {
          int mid = (slo + shi + 1) >> 1;
          if (seg[mid] <= sb0) slo = mid; else shi = mid - 1;
        }
        int she = slo, hi2 = nseg_total;   // first segment starting at or after sb1
        while (she < hi2) {
          const int mid = (she + hi2) >> 1;
          if (seg[mid] < sb1) she = mid + 1; else hi2 = mid;
        }
        // window sums: short segments (<= kLongSeg entries here) by thread per
        // (segment, float4) -- few items for many small segments -- long
        // (hot) segments by thread per (segment, float column), d threads with
        // 4-way ILP each; fb_segsum fixes the chain order, so the result does
        // not depend on which form summed a segment
        const int nsw = she - slo;
        constexpr int kLongSeg = 64;
        int* longl = ws;   // <= SB / kLongSeg + 1 long segments per window
        if (tid == 0) ws[63] = 0;
        __syncthreads();
        for (int i = tid; i < nsw; i += NT) {
          const int s0 = seg[slo + i], s1 = seg[slo + i + 1];
          if (min(s1, sb1) - max(s0, sb0) > kLongSeg) longl[atomicAdd(&ws[63], 1)] = slo + i;
        }
        __syncthreads();
        const int nlong = ws[63];
        if ((d & 3) == 0) {
          const int Q = d >> 2;
          #pragma unroll 1
          for (int it = tid; it < nsw * Q; it += NT) {
            const int sidx = slo + it / Q, qf = it - (it / Q) * Q;
            const int s0 = seg[sidx], s1 = seg[sidx + 1];
            if (min(s1, sb1) - max(s0, sb0) > kLongSeg) continue;
            fb_segsum<float4>(stage, carry, d, sb0, sb1, s0, s1, qf, par);
          }
        } else {
          #pragma unroll 1
          for (int it = tid; it < nsw * d; it += NT) {
            const int sidx = slo + it / d, f = it - (it / d) * d;
            const int s0 = seg[sidx], s1 = seg[sidx + 1];
            if (min(s1, sb1) - max(s0, sb0) > kLongSeg) continue;
            fb_segsum<float>(stage, carry, d, sb0, sb1, s0, s1, f, par);
          }
        }
        #pragma unroll 1
        for (int it = tid; it < nlong * d; it += NT) {
          const int sidx = longl[it / d], f = it - (it / d) * d;
          fb_segsum<float>(stage, carry, d, sb0, sb1, seg[sidx], seg[sidx + 1], f, par);
        }
        __syncthreads();
        if (sb0 / lay.SB < 4) trace_mark(p, 51 + 2 * (sb0 / lay.SB));
        // C += -lr * total for the segments that end in this window, with
        // several row reads in flight per thread (not one dependent global
        // round trip per (segment, column)); or emit (row, total)
        {
          const int fin0 = (nsw > 0 && seg[she] > sb1) ? she - 1 : she;   // segments [slo, fin0) end here
          const int nfin = fin0 - slo;
          if (emit_rows) {
            #pragma unroll 1
            for (int t = tid; t < nfin * d; t += NT) {
              const int sidx = slo + t / d, f = t - (t / d) * d;
              const int a0 = max(seg[sidx], sb0);
              if (f == 0) emit_rows[emitted + sidx - slo] = (int)(keys[seg[sidx]] >> 32);
              emit_vals[(size_t)(emitted + sidx - slo) * d + f] = stage[(size_t)(a0 - sb0) * d + f];
            }
            emitted += nfin;
          } else {
          const bool v4 = (d & 3) == 0;
          const int W4 = v4 ? d >> 2 : d;
          #pragma unroll 1
          for (int t0 = tid; t0 < nfin * W4; t0 += 4 * NT) {
            float4 cur[4];
            float4* dst[4];
            float4 tot[4];
            #pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int t = t0 + j * NT;
              dst[j] = nullptr;
              if (t < nfin * W4) {
                const int sidx = slo + t / W4, f = t - (t / W4) * W4;
                const int a0 = max(seg[sidx], sb0);
                const unsigned row = (unsigned)(keys[seg[sidx]] >> 32);
                if (v4) {
                  dst[j] = reinterpret_cast<float4*>(p.C + (size_t)row * d) + f;
                  tot[j] = reinterpret_cast<const float4*>(stage + (size_t)(a0 - sb0) * d)[f];
                  cur[j] = __ldcg(dst[j]);
                } else {
                  dst[j] = reinterpret_cast<float4*>(p.C + (size_t)row * d + f);   // scalar slot
                  tot[j].x = stage[(size_t)(a0 - sb0) * d + f];
                  cur[j].x = __ldcg(p.C + (size_t)row * d + f);
                }
              }
            }
            #pragma unroll
            for (int j = 0; j < 4; ++j) {
              if (!dst[j]) continue;
              if (v4)
                *dst[j] = make_float4(cur[j].x + nlr * tot[j].x, cur[j].y + nlr * tot[j].y,
                                      cur[j].z + nlr * tot[j].z, cur[j].w + nlr * tot[j].w);
              else
                *reinterpret_cast<float*>(dst[j]) = cur[j].x + nlr * tot[j].x;
            }
          }
          }
        }
        __syncthreads();
        if (sb0 == 0) trace_mark(p, 45);
        if (sb0 / lay.SB < 4) trace_mark(p, 46 + sb0 / lay.SB);
      }
    }
    La = Lb;
  }
  trace_mark(p, 43);
  return emitted;
}

// Trip 1 of the owner merge: CTA q's entry count in every list, scanned into
// lbase (entry base per list) and loff (offset of q's bucket inside the list).
// Returns M, the owner's entry count; *base_q (if given) receives the sum of
// loff over the lists = the entries of owners < q, where owner q's merged rows
// start in a data-parallel record (so the record layout is deterministic).
__device__ int det_counts(const StepParams& p, unsigned char* sm, int pre_a, int pre_b, int* base_q = nullptr) {
  const Layout& lay = p.lay;
  const int tid = threadIdx.x, NT = blockDim.x, q = blockIdx.x, P = p.P, NL = p.NL;
  int* lbase = reinterpret_cast<int*>(sm + lay.lbase);
  int* loff = reinterpret_cast<int*>(sm + lay.loff);
  int* ws = reinterpret_cast<int*>(sm + lay.ws2);
  int running = 0, asum = 0;
  #pragma unroll 1
  for (int L0 = 0; L0 < NL; L0 += NT) {
    const int L = L0 + tid;
    int cnt = 0;
    if (L < NL) {
      int a = pre_a, b = pre_b;   // lists [0, NT) were loaded with the other trip-1 reads
      if (L0 > 0) {
        const int32_t* off = p.list_off + (size_t)L * (P + 1);
        a = __ldcg(off + q);
        b = __ldcg(off + q + 1);
      }
      loff[L] = a;
      asum += a;
      cnt = b - a;
    }
    int tot;
    const int ex = block_excl_scan(cnt, ws, &tot);
    if (L < NL) lbase[L] = running + ex;
    running += tot;
  }
  if (base_q) block_excl_scan(asum, ws, base_q);
  if (tid == 0) lbase[NL] = running;
  __syncthreads();
  return running;
}

// Phase-2 table resets: CTA-local, so they run between the grid-barrier arrive
// and wait (phase 1's shared memory is dead by then).  Needs a barrier before use.
__device__ void phase2_prep(const StepParams& p, unsigned char* sm) {
  const Layout& lay = p.lay;
  const int tid = threadIdx.x, NT = blockDim.x;
  int* hkey = reinterpret_cast<int*>(sm + lay.hkey);
  int* hfirst = reinterpret_cast<int*>(sm + lay.hfirst);
  #pragma unroll 1
  for (int i = tid; i < lay.HS; i += NT) { hkey[i] = -1; hfirst[i] = 0; }
  uint4* rmask = reinterpret_cast<uint4*>(sm + lay.rmask);
  #pragma unroll 1
  for (int i = tid; i < lay.MCAP * 4; i += NT) rmask[i] = make_uint4(0u, 0u, 0u, 0u);
  if (tid == 0) reinterpret_cast<int*>(sm + lay.rcur)[lay.MCAP] = 0;
}

// Issue half: entry sources, then trip 2 (row ids, then the gradient partials)
// as cp.async groups -- returns at once so the dense update runs while they are
// in flight.  NL lists described by lbase / loff (smem) and `ls`.
__device__ void det_issue(const StepParams& p, unsigned char* sm, int M, int NL, const Lists& ls) {
  const Layout& lay = p.lay;
  const int tid = threadIdx.x, NT = blockDim.x;
  const int d = p.d;
  const int* lbase = reinterpret_cast<const int*>(sm + lay.lbase);
  const int* loff = reinterpret_cast<const int*>(sm + lay.loff);
  unsigned* esrc = reinterpret_cast<unsigned*>(sm + lay.esrc);
  int* erow = reinterpret_cast<int*>(sm + lay.erow);
  float* stage = reinterpret_cast<float*>(sm + lay.stage);
  #pragma unroll 1
  for (int L = tid; L < NL; L += NT) {   // entries of list L: [lbase[L], lbase[L+1])
    const int b = lbase[L], cnt = lbase[L + 1] - b;
    #pragma unroll 1
    for (int j = 0; j < cnt; ++j) esrc[b + j] = ls.code(L, loff[L] + j);
  }
  __syncthreads();
  trace_mark(p, 20);
  #pragma unroll 1
  for (int e = tid; e < M; e += NT) cp_async4(erow + e, ls.row(esrc[e]));
  asm volatile("cp.async.commit_group;" ::: "memory");
  if ((d & 3) == 0) {
    const int Q = d >> 2;
    #pragma unroll 2
    for (int it = tid; it < M * Q; it += NT) {
      const int e = it / Q, q = it - e * Q;
      cp_async16(stage + (size_t)e * d + 4 * q, ls.val(esrc[e], d) + 4 * q);
    }
  } else {
    #pragma unroll 1
    for (int t = tid; t < M * d; t += NT) {
      const int e = t / d, f = t - e * d;
      cp_async4(stage + t, ls.val(esrc[e], d) + f);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// Deterministic owner merge (hash fast path, M <= MCAP): CTA q owns rows with
// row % P == q.  Its entries are staged in (list, position) order -- list
// order is the fixed summation order -- and each distinct row's partials are
// summed in that order, then C[row] += -lr * sum (one rounding), or, with
// emit_rows, the (row, sum) pairs are written to emit_rows / emit_vals
// [0, nrows) (a data-parallel record).  Runs after det_issue; returns nrows.
__device__ int det_merge(const StepParams& p, unsigned char* sm, int M, bool write, int32_t* emit_rows = nullptr,
                         float* emit_vals = nullptr) {
  const Layout& lay = p.lay;
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, warp = tid >> 5, NW = NT >> 5;
  const int d = p.d;
  int* ws = reinterpret_cast<int*>(sm + lay.ws2);
  int* esrc = reinterpret_cast<int*>(sm + lay.esrc);
  int* erow = reinterpret_cast<int*>(sm + lay.erow);
  int* heads = reinterpret_cast<int*>(sm + lay.heads);
  unsigned short* hlist = reinterpret_cast<unsigned short*>(sm + lay.hlist);
  int* hkey = reinterpret_cast<int*>(sm + lay.hkey);
  int* hfirst = reinterpret_cast<int*>(sm + lay.hfirst);
  float* stage = reinterpret_cast<float*>(sm + lay.stage);
  const int HS = lay.HS;
  const float nlr = -p.lr;
  unsigned* rmask = reinterpret_cast<unsigned*>(sm + lay.rmask);
  __shared__ int s_nseg;
  if (tid == 0) s_nseg = 0;
  asm volatile("cp.async.wait_group 1;" ::: "memory");   // row ids landed (partials may still fly)
  __syncthreads();
  trace_mark(p, 21);
  // ---- distinct rows: smem hash (row -> distinct index), multiplicity per row
  int* hcnt = hfirst;          // reused: per-slot multiplicity
  int* eslot = esrc;           // reused: entry -> hash slot (sources already issued)
  int* rcnt = reinterpret_cast<int*>(sm + lay.rcnt);
  int* roff = reinterpret_cast<int*>(sm + lay.roff);
  int* rcur = reinterpret_cast<int*>(sm + lay.rcur);
  int* rrow = heads;           // distinct index -> row
  int* hrid = reinterpret_cast<int*>(sm + lay.misc2);
  int my_r[2] = {-1, -1}, my_hs[2] = {0, 0};
  #pragma unroll 1
  for (int e = tid, k = 0; e < M; e += NT, ++k) {
    const int key = erow[e];
    unsigned hsl = hash_row((unsigned)key) & (HS - 1);
    bool mine = false;
    while (true) {
      const int prev = atomicCAS(&hkey[hsl], -1, key);
      if (prev == -1) { mine = true; break; }
      if (prev == key) break;
      hsl = (hsl + 1) & (HS - 1);
    }
    eslot[e] = (int)hsl;
    atomicAdd(&hcnt[hsl], 1);
    if (mine && k < 2) {
      const int r = atomicAdd(&rcur[lay.MCAP], 1);
      hrid[hsl] = r;
      rrow[r] = key;
      if (k == 0) { my_r[0] = r; my_hs[0] = (int)hsl; }
      else { my_r[1] = r; my_hs[1] = (int)hsl; }
    }
  }
  __syncthreads();
  trace_mark(p, 22);
  const int nrows = rcur[lay.MCAP];
  // trip 3, issued now: the current C rows, staged behind the M partials while
  // they fit (rows beyond the stage capacity are read directly when applied)
  const int Q = d >> 2;
  const bool quad = (d & 3) == 0;
  const int ccap = (quad && !emit_rows) ? min(nrows, lay.MCAP - M) : 0;
  #pragma unroll 2
  for (int it = tid; it < ccap * Q; it += NT) {
    const int ri = it / Q, q = it - ri * Q;
    cp_async16(stage + (size_t)(M + ri) * d + 4 * q, p.C + (size_t)rrow[ri] * d + 4 * q);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  if (my_r[0] >= 0) rcnt[my_r[0]] = hcnt[my_hs[0]];
  if (my_r[1] >= 0) rcnt[my_r[1]] = hcnt[my_hs[1]];
  #pragma unroll 1
  for (int e = tid; e < M; e += NT) {   // entry -> distinct row; row membership mask
    const int r = hrid[eslot[e]];
    eslot[e] = r;
    atomicOr(&rmask[r * 16 + (e >> 5)], 1u << (e & 31));
  }
  __syncthreads();
  {
    int running = 0;
    #pragma unroll 1
    for (int r0 = 0; r0 < nrows; r0 += NT) {
      const int r = r0 + tid;
      const int v = r < nrows ? rcnt[r] : 0;
      int tot;
      const int ex = block_excl_scan(v, ws, &tot);
      if (r < nrows) { roff[r] = running + ex; rcur[r] = 0; }
      running += tot;
    }
  }
  __syncthreads();
  trace_mark(p, 23);
  // entries grouped by row, in list order within each row
  #pragma unroll 1
  for (int e = tid; e < M; e += NT) {
    const int r = eslot[e];
    hlist[roff[r] + mask_rank<16>(rmask + r * 16, e)] = (unsigned short)e;
  }
  // long rows (more than kLongRow partials: the Zipf head rows this CTA owns) are
  // summed in kLongRow-entry segments by separate threads, then the segments are
  // added in order -- a fixed association that depends only on the row's count.
  // lpart holds the worst case (Layout::NSEG), so EVERY long row splits; the
  // atomicAdd only decides where a row's segments are stored, not the sums.
  constexpr int kLongRow = 32;
  int* rsplit = rcur;                                   // row -> first segment, -1: not split
  int* segrow = hrid;                                   // segment -> row
  float4* lpart = reinterpret_cast<float4*>(sm + lay.lpart);   // [segment][Q] partial sums
  const int maxseg = quad ? lay.NSEG : 0;
  int* segidx = hrid + maxseg;
  #pragma unroll 1
  for (int r = tid; r < nrows; r += NT) {
    int b = -1;
    const int m = rcnt[r];
    if (quad && m > kLongRow) {
      const int S = (m + kLongRow - 1) / kLongRow;
      b = atomicAdd(&s_nseg, S);   // b + S <= NSEG by construction (sum of S over long rows)
      for (int t = 0; t < S; ++t) { segrow[b + t] = r; segidx[b + t] = t; }
    }
    rsplit[r] = b;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  trace_mark(p, 24);
  const int nseg = s_nseg;
  // ---- ordered sum of each distinct row's partials, one RMW of C; one thread
  // per (row, feature quad) when d % 4 == 0, else one warp per row
  if (quad) {
    const float4* S4 = reinterpret_cast<const float4*>(stage);
#pragma unroll 1
    for (int it = tid; it < (nrows + nseg) * Q; it += NT) {
      const int k = it / Q, q = it - k * Q;
      if (k < nseg) {   // one segment of a long row
        const int r = segrow[k];
        if (r >= 0) {
          const int s0 = segidx[k] * kLongRow, m = rcnt[r] - s0;
          lpart[k * Q + q] = ordered_quadsum(S4, hlist + roff[r] + s0, m < kLongRow ? m : kLongRow, Q, q);
        }
        continue;
      }
      const int ri = k - nseg;
      if (rsplit[ri] >= 0) continue;
      const float4 a = ordered_quadsum(S4, hlist + roff[ri], rcnt[ri], Q, q);
      if (emit_rows) {
        if (q == 0) emit_rows[ri] = rrow[ri];
        reinterpret_cast<float4*>(emit_vals + (size_t)ri * d)[q] = a;
      } else if (write) {
        float4* c4 = reinterpret_cast<float4*>(p.C + (size_t)rrow[ri] * d) + q;
        const float4 o = ri < ccap ? S4[(size_t)(M + ri) * Q + q] : __ldcg(c4);
        *c4 = make_float4(o.x + nlr * a.x, o.y + nlr * a.y, o.z + nlr * a.z, o.w + nlr * a.w);
      }
    }
    if (nseg > 0) {
      __syncthreads();
#pragma unroll 1
      for (int it = tid; it < nseg * Q; it += NT) {   // combine each split row's segments in order
        const int k = it / Q, q = it - k * Q;
        const int r = segrow[k];
        if (r < 0 || segidx[k] != 0) continue;
        const int S = (rcnt[r] + kLongRow - 1) / kLongRow;
        float4 a = lpart[k * Q + q];
        for (int t = 1; t < S; ++t) {
          const float4 v = lpart[(k + t) * Q + q];
          a = make_float4(a.x + v.x, a.y + v.y, a.z + v.z, a.w + v.w);
        }
        if (emit_rows) {
          if (q == 0) emit_rows[r] = rrow[r];
          reinterpret_cast<float4*>(emit_vals + (size_t)r * d)[q] = a;
        } else if (write) {
          float4* c4 = reinterpret_cast<float4*>(p.C + (size_t)rrow[r] * d) + q;
          const float4 o = r < ccap ? S4[(size_t)(M + r) * Q + q] : __ldcg(c4);
          *c4 = make_float4(o.x + nlr * a.x, o.y + nlr * a.y, o.z + nlr * a.z, o.w + nlr * a.w);
        }
      }
    }
  } else {
#pragma unroll 1
    for (int ri = warp; ri < nrows; ri += NW) {
      float* crow = p.C + (size_t)rrow[ri] * d;
      const int nm = rcnt[ri];
      const unsigned short* ps = hlist + roff[ri];
#pragma unroll 1
      for (int f0 = 0; f0 < d; f0 += 128) {
        const float4 a4 = ordered_rowsum(stage, ps, nm, d, f0);
        const float acc[4] = {a4.x, a4.y, a4.z, a4.w};
        if (emit_rows) {
          if (lane == 0 && f0 == 0) emit_rows[ri] = rrow[ri];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int f = f0 + lane + 32 * k;
            if (f < d) emit_vals[(size_t)ri * d + f] = acc[k];
          }
        } else if (write) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int f = f0 + lane + 32 * k;
            if (f < d) crow[f] = __ldcg(crow + f) + nlr * acc[k];
          }
        }
      }
    }
  }
  __syncthreads();
  return nrows;
}

// Atomic scatter: CTA b applies lists L = b, b+G, ... with red.global.add.v4.f32.
__device__ void phase2_scatter_atomic(const StepParams& p) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NW = blockDim.x >> 5;
  const int P = p.P, d = p.d;
  const float nlr = -p.lr;
  #pragma unroll 1
  for (int L = blockIdx.x; L < p.NL; L += gridDim.x) {
    const int U0 = __ldcg(p.list_off + (size_t)L * (P + 1));
    const int U1 = __ldcg(p.list_off + (size_t)L * (P + 1) + P);
    #pragma unroll 1
    for (int j = U0 + warp; j < U1; j += NW) {
      const size_t ix = (size_t)L * p.cap + j;
      const int row = __ldcg(p.list_rows + ix);
      const float* src = p.list_vals + ix * d;
      float* dst = p.C + (size_t)row * d;
      if ((d & 3) == 0) {
        #pragma unroll 1
        for (int f4 = lane; f4 < (d >> 2); f4 += 32) {
          float4 v = ldcg4(src + 4 * f4);
          v.x *= nlr; v.y *= nlr; v.z *= nlr; v.w *= nlr;
          red_add_v4(dst + 4 * f4, v);
        }
      } else {
        #pragma unroll 1
        for (int f = lane; f < d; f += 32) atomicAdd(dst + f, nlr * __ldcg(src + f));
      }
    }
  }
}

template <bool kGemm>
__device__ void phase2(const StepParams& p, unsigned char* sm) {
  __shared__ int s_flags;
  __shared__ float s_loss;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NT = blockDim.x;
  DevStatus* st = p.st;
  // ---- trip 1: everything that does not depend on the decision, all issued
  // before any of it is consumed (one round trip, not one per consumer)
  unsigned my_done = 0;
  int f0 = 0;
  unsigned long long bad = 0;
  if (tid == 0) {
    f0 = __ldcg(&st->flags);
    bad = __ldcg(&st->bad);
    my_done = atomicAdd(&st->done, 1u);   // result consumed only at the end (flag reset)
  }
  const int hoff = p.dense_len;   // record words [hoff, hoff+1] = (hinge sum, flags); hoff is even
  float2 hv[5];   // warp 1: the first 160 records' (hinge, flags)
  if (warp == 1) {
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const int r = lane + 32 * k;
      hv[k] = r < p.P ? __ldcg(reinterpret_cast<const float2*>(p.dense_part + (size_t)r * p.dense_stride + hoff))
                         : make_float2(0.f, 0.f);
    }
  }
  // owner counts for lists [0, NT)
  int pre_a = 0, pre_b = 0;
  if (p.mode == 0 && tid < p.NL) {
    const int32_t* off = p.list_off + (size_t)tid * (p.P + 1) + blockIdx.x;
    pre_a = __ldcg(off);
    pre_b = __ldcg(off + 1);
  }
  const DenseSlice ds = dense_slice(p);
  const int nq0 = min(NT, ds.q1 - ds.q0);
  const int groups0 = nq0 > 0 ? dense_groups(nq0, NT) : 1;
  float4 dacc0 = make_float4(0.f, 0.f, 0.f, 0.f);
  float cur0[4] = {0.f, 0.f, 0.f, 0.f};
  if (nq0 > 0) {
    if (tid < nq0) {   // the parameters this CTA updates
      const int ndh = p.n * p.d * p.h, base = 4 * (ds.q0 + tid);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (base + k < p.dense_len) cur0[k] = __ldcg(param_ptr(p, base + k, ndh));
    }
    dacc0 = dense_partial(p, ds.q0, nq0, groups0);   // issues its loads, then sums
  }
  if (warp == 1) {   // mean hinge, summed in record order; OR of the records' flags
    float acc = 0.f;
    unsigned fl = 0;
#pragma unroll
    for (int k = 0; k < 5; ++k) { acc += hv[k].x; fl |= (unsigned)__float_as_int(hv[k].y); }
    acc = warp_sum(acc);
    fl = __reduce_or_sync(0xffffffffu, fl);
    if (lane == 0) s_loss = acc * p.inv_B;
    (void)fl;
  }
  if (tid == 0) {
    s_flags = f0;
    if (blockIdx.x == 0) st->last_bad = bad;
  }
  trace_mark(p, 29);
  int M = 0;
  if (p.mode == 0) M = det_counts(p, sm, pre_a, pre_b);   // contains __syncthreads
  trace_mark(p, 30);
#ifdef PG_TRACE
  if (tid == 0 && p.trace != nullptr) p.trace[blockIdx.x * 64 + 31] = M;
#endif
  __syncthreads();
  const float loss = s_loss;
  const int flags = s_flags | (!isfinite(loss) ? 2 : 0);
  const bool write = flags == 0;   // no parameter changes on a bad index or a non-finite loss
  if (blockIdx.x == 0 && tid == 0) {
    st->last_loss = loss;
    st->last_flags = flags;
    st->rank_flags = flags;
    if (p.loss_out) *p.loss_out = loss;
    if (flags) {
      atomicOr(&st->sticky_flags, flags);
      atomicMin(&st->sticky_bad, st->last_bad);
    }
  }
  trace_mark(p, 8);
  const bool hashed = p.mode == 0 && M > 0 && M <= p.lay.MCAP;
  const Lists ls{p.list_rows, p.list_vals, p.cap, 0};
  if (hashed) det_issue(p, sm, M, p.NL, ls);   // trip 2 in flight during the dense update
  // ---- dense update (first block prefetched; further blocks only when P is small)
  if (nq0 > 0) dense_apply(p, sm, ds.q0, nq0, groups0, dacc0, make_float4(cur0[0], cur0[1], cur0[2], cur0[3]), write);
  #pragma unroll 1
  for (int qb = ds.q0 + nq0; qb < ds.q1; qb += NT) {
    const int nq = min(NT, ds.q1 - qb), groups = dense_groups(nq, NT);
    float cur[4] = {0.f, 0.f, 0.f, 0.f};
    if (tid < nq) {
      const int ndh = p.n * p.d * p.h, base = 4 * (qb + tid);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (base + k < p.dense_len) cur[k] = __ldcg(param_ptr(p, base + k, ndh));
    }
    dense_apply(p, sm, qb, nq, groups, dense_partial(p, qb, nq, groups),
                make_float4(cur[0], cur[1], cur[2], cur[3]), write);
  }
  trace_mark(p, 9);
  // ---- embedding scatter-add
  if (p.mode == 0) {
    if (hashed) det_merge(p, sm, M, write);
    else if (M > 0 && write) scatter_det_sorted(p, sm, ls);
  } else if (write) {
    phase2_scatter_atomic(p);
  }
  if (kGemm && p.dw1_gemm) {
    __syncthreads();   // the merge's shared memory is free
    trace_mark(p, 39);
    dw1_gemm_tiles(p, sm, write);
    trace_mark(p, 48);
  }
  if (tid == 0 && my_done == gridDim.x - 1) {   // every CTA has read this step's flags
    st->flags = 0;
    st->bad = kNoBad;
    st->done = 0;
  }
}

// ------------------------------------------------------------------ data parallel
// One synchronous DP step (PAPER.md:219-220 names distributed
// gradient descent as the next step).  Every rank runs phase 1 on its shard,
// then (publish) each owner CTA q merges the rows it owns over the rank's own
// lists -- one (row, gradient-sum) entry per distinct row, the "per-rank
// dedup" -- and writes them, with its slice of the rank's dense-gradient sum,
// the rank's hinge sum and error flags, into the rank's exchange window.
// (merge) CTA q of every rank then reads owner q's entries and dense slice of
// all G ranks, sums each row's and each dense element's G partials in rank
// order and applies the update.  Identical inputs in an identical order on
// every rank: replicas stay bit-identical, and the result does not depend on
// how the records travelled (peer loads over NVLink, an NCCL all-gather, or
// device copies between replicas of one GPU).

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// The rank's hinge sum over its P partial records (fixed association: lane-
// strided sums, then a butterfly) -- every CTA computes the same value.
__device__ __forceinline__ float rank_hinge(const StepParams& p) {
  const int lane = threadIdx.x & 31;
  float acc = 0.f;
  #pragma unroll 1
  for (int r = lane; r < p.P; r += 32) acc += __ldcg(p.dense_part + (size_t)r * p.dense_stride + p.dense_len);
  return warp_sum(acc);
}

__device__ void dp_publish(const StepParams& p, unsigned char* sm) {
  __shared__ unsigned s_epoch;
  __shared__ int s_flags;
  __shared__ float s_hinge;
  const int tid = threadIdx.x, NT = blockDim.x, warp = tid >> 5, q = blockIdx.x, d = p.d;
  DevStatus* st = p.st;
  unsigned my_done = 0;
  int pre_a = 0, pre_b = 0;
  if (tid < p.NL) {   // owner counts for lists [0, NT), issued with the other trip-1 reads
    const int32_t* off = p.list_off + (size_t)tid * (p.P + 1) + q;
    pre_a = __ldcg(off);
    pre_b = __ldcg(off + 1);
  }
  if (tid == 0) {
    s_epoch = p.xepoch[q] + 1u;
    s_flags = __ldcg(&st->flags);
    if (q == 0) st->last_bad = __ldcg(&st->bad);
    my_done = atomicAdd(&st->done, 1u);
  }
  if (warp == 1) {
    const float hsum = rank_hinge(p);
    if ((tid & 31) == 0) s_hinge = hsum;
  }
  int base = 0;
  const int M = det_counts(p, sm, pre_a, pre_b, &base);   // contains __syncthreads
  const unsigned epoch = s_epoch;
  const int par = p.xgathered ? 0 : (int)(epoch & 1u);
  unsigned char* blk = p.xwin + p.xl.blk[par];
  int32_t* erows = reinterpret_cast<int32_t*>(blk + p.xl.rows) + base;
  float* evals = reinterpret_cast<float*>(blk + p.xl.vals) + (size_t)base * d;
  float* dense = reinterpret_cast<float*>(p.xwin + p.xl.dense[par]);
  const Lists ls{p.list_rows, p.list_vals, p.cap, 0};
  const bool hashed = M > 0 && M <= p.lay.MCAP;
  if (hashed) det_issue(p, sm, M, p.NL, ls);   // entries in flight during the dense sums
  // this CTA's slice of the rank's dense-gradient sum (P records, record order)
  const DenseSlice ds = dense_slice(p);
  #pragma unroll 1
  for (int qb = ds.q0; qb < ds.q1; qb += NT) {
    const int nq = min(NT, ds.q1 - qb), groups = dense_groups(nq, NT);
    dense_apply(p, sm, qb, nq, groups, dense_partial(p, qb, nq, groups), make_float4(0.f, 0.f, 0.f, 0.f), false,
                dense);
  }
  if (q == 0 && tid == 0) {   // hinge | flags words (summed by the NCCL all-reduce exchanges)
    dense[p.dense_len] = s_hinge;
    dense[p.dense_len + 1] = s_flags ? 1.f : 0.f;
  }
  int count = 0;
  if (hashed) count = det_merge(p, sm, M, true, erows, evals);
  else if (M > 0) count = scatter_det_sorted(p, sm, ls, erows, evals);
  if (tid == 0) {
    XHdr* hdr = reinterpret_cast<XHdr*>(blk) + q;
    *hdr = XHdr{s_flags, s_hinge, base, count};
  }
  __syncthreads();
  if (tid == 0) {
    p.xepoch[q] = epoch;
    if (p.xpeer) {   // this CTA's part of the record is complete: tell every rank
      __threadfence_system();
      #pragma unroll 1
      for (int r = 0; r < p.world; ++r) {
        unsigned* f = reinterpret_cast<unsigned*>(const_cast<unsigned char*>(p.xbase) + (size_t)r * p.xstride + p.xl.flags);
        st_release_sys(f + (size_t)p.rank * kMaxSMs + q, epoch);
      }
    }
    if (my_done == gridDim.x - 1) {   // every CTA has read this step's flags
      st->flags = 0;
      st->bad = kNoBad;
      st->done = 0;
    }
  }
}

// Merge: owner q of all ranks, rank order.  Needs phase2_prep + a barrier first.
__device__ void dp_merge(const StepParams& p, unsigned char* sm) {
  __shared__ int s_flags, s_M;
  __shared__ float s_loss;
  __shared__ unsigned s_epoch;
  const Layout& lay = p.lay;
  const int tid = threadIdx.x, NT = blockDim.x, q = blockIdx.x, d = p.d, G = p.world;
  DevStatus* st = p.st;
  int* lbase = reinterpret_cast<int*>(sm + lay.lbase);
  int* loff = reinterpret_cast<int*>(sm + lay.loff);
  if (tid == 0) {
    const unsigned epoch = p.xepoch[q];
    s_epoch = epoch;
    int fl = 0;
    if (p.xpeer) {   // wait until owner q of every rank has published this step
      const unsigned* f = reinterpret_cast<const unsigned*>(p.xwin + p.xl.flags) + q;
      const unsigned long long t0 = globaltimer_ns();
      #pragma unroll 1
      for (int r = 0; r < G; ++r) {
        while ((int)(ld_acquire_sys(f + (size_t)r * kMaxSMs) - epoch) < 0) {
          if (globaltimer_ns() - t0 > 20000000000ull) { fl |= 4; break; }   // 20 s: a rank is gone
          __nanosleep(32);
        }
      }
    }
    s_flags = fl;
  }
  __syncthreads();
  const int par = p.xgathered ? 0 : (int)(s_epoch & 1u);
  const unsigned char* blk0 = p.xbase + (p.xgathered ? 0 : p.xl.blk[par]);
  // headers of owner q, every rank, summed in rank order by one thread
  if (tid == 0) {
    int fl = s_flags, M = 0;
    float hinge = 0.f;
    unsigned long long xb = 0;
    #pragma unroll 1
    for (int r = 0; r < G; ++r) {
      const int4 h = __ldcg(reinterpret_cast<const int4*>(blk0 + (size_t)r * p.xstride) + q);
      fl |= h.x;
      hinge += __int_as_float(h.y);
      loff[r] = h.z;
      lbase[r] = M;
      M += h.w;
      if (r != p.rank) xb += sizeof(XHdr) + (unsigned long long)h.w * (4ull + 4ull * d);
    }
    lbase[G] = M;
    s_M = M;
    const float loss = hinge * p.inv_B;
    s_loss = loss;
    s_flags = fl | (!isfinite(loss) ? 2 : 0);
    if (p.xstats) {
      const DenseSlice ds = dense_slice(p);
      if (!p.xdense) xb += (unsigned long long)(G - 1) * 16ull * (ds.q1 - ds.q0);
      atomicAdd(p.xstats, xb);
      atomicMax(p.xstats + 1, (unsigned long long)M);
    }
    if (q == 0) {
      const int flags = s_flags;
      st->last_loss = loss;
      st->last_flags = flags;
      st->rank_flags = flags;
      if (p.loss_out) *p.loss_out = loss;
      if (flags) {
        atomicOr(&st->sticky_flags, flags);
        atomicMin(&st->sticky_bad, st->last_bad);
      }
    }
  }
  __syncthreads();
  const int M = s_M;
  const bool write = s_flags == 0;
  const Lists ls{reinterpret_cast<const int32_t*>(blk0 + p.xl.rows), reinterpret_cast<const float*>(blk0 + p.xl.vals), 0,
                 p.xstride};
  const bool hashed = M > 0 && M <= lay.MCAP;
  if (hashed) det_issue(p, sm, M, G, ls);   // entries in flight during the dense update
  // dense: this CTA's slice, the G ranks' sums added in rank order (or the
  // NCCL all-reduced vector), then W1 / b1 / w2 -= lr * sum
  {
    const DenseSlice ds = dense_slice(p);
    const int ndh = p.n * p.d * p.h, DL = p.dense_len;
    #pragma unroll 1
    for (int qi = ds.q0 + tid; qi < ds.q1; qi += NT) {
      float4 acc;
      if (p.xdense) {
        acc = ldcg4(p.xdense + 4 * qi);
      } else {
        acc = make_float4(0.f, 0.f, 0.f, 0.f);
        const unsigned char* db = p.xbase + p.xl.dense[par];
        #pragma unroll 1
        for (int r = 0; r < G; ++r) {
          const float4 v = ldcg4(reinterpret_cast<const float*>(db + (size_t)r * p.xstride) + 4 * qi);
          acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
      }
      const float sv[4] = {acc.x, acc.y, acc.z, acc.w};
      const int base = 4 * qi;
      if (write) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (base + k >= DL) break;
          float* ptr = param_ptr(p, base + k, ndh);
          const float nv = __ldcg(ptr) - p.lr * sv[k];
          *ptr = nv;
          if (p.W1T != nullptr && base + k < ndh) {
            const int row = (base + k) / p.h, u = base + k - row * p.h;
            p.W1T[(size_t)u * (p.n * p.d) + row] = nv;
          }
        }
      }
    }
  }
  __syncthreads();
  if (hashed) det_merge(p, sm, M, write);
  else if (M > 0 && write) scatter_det_sorted(p, sm, ls);
}

// NCCL table exchange (PG_EXCHANGE_TABLE): this rank's merged rows into the
// zeroed V x d gradient table (a row is at most in two entries of one owner --
// sorted-fallback window split -- and two float adds commute exactly).
__global__ void dp_table_scatter_kernel(StepParams p, float* table) {
  const unsigned char* blk = p.xwin + p.xl.blk[0];
  const int q = blockIdx.x, d = p.d;
  const int4 h = __ldcg(reinterpret_cast<const int4*>(blk) + q);
  const int32_t* rows = reinterpret_cast<const int32_t*>(blk + p.xl.rows) + h.z;
  const float* vals = reinterpret_cast<const float*>(blk + p.xl.vals) + (size_t)h.z * d;
  #pragma unroll 1
  for (int t = threadIdx.x; t < h.w * d; t += blockDim.x) {
    const int e = t / d, f = t - e * d;
    atomicAdd(table + (size_t)rows[e] * d + f, vals[t]);
  }
}

// After the all-reduces: W1 / b1 / w2 -= lr * dense, C += -lr * table on every
// row (adding -lr * 0 leaves a row bit-identical), table re-zeroed; gated on
// the reduced flags / loss.  xdense = reduced [dense | hinge | flags].
__global__ void dp_table_apply_kernel(StepParams p, float* table, int zero) {
  const float hinge = __ldcg(p.xdense + p.dense_len), flagsum = __ldcg(p.xdense + p.dense_len + 1);
  const float loss = hinge * p.inv_B;
  const int flags = (flagsum != 0.f ? 1 : 0) | (!isfinite(loss) ? 2 : 0);
  const bool write = flags == 0;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, NT = (size_t)gridDim.x * blockDim.x;
  if (tid == 0) {
    DevStatus* st = p.st;
    st->last_loss = loss;
    st->last_flags = flags;
    st->rank_flags = flags;
    if (p.loss_out) *p.loss_out = loss;
    if (flags) {
      atomicOr(&st->sticky_flags, flags);
      atomicMin(&st->sticky_bad, st->last_bad);
    }
  }
  const int ndh = p.n * p.d * p.h;
  if (write)
    for (size_t i = tid; i < (size_t)p.dense_len; i += NT) {
      float* ptr = param_ptr(p, (int)i, ndh);
      const float nv = *ptr - p.lr * __ldcg(p.xdense + i);
      *ptr = nv;
      if (p.W1T != nullptr && (int)i < ndh) {
        const int row = (int)i / p.h, u = (int)i - row * p.h;
        p.W1T[(size_t)u * (p.n * p.d) + row] = nv;
      }
    }
  const size_t n4 = (size_t)p.V * p.d / 4;
  const float nlr = -p.lr;
  float4* T4 = reinterpret_cast<float4*>(table);
  float4* C4 = reinterpret_cast<float4*>(p.C);
  for (size_t i = tid; i < n4; i += NT) {
    const float4 g = T4[i];
    if (write) {
      float4 c = C4[i];
      c.x += nlr * g.x; c.y += nlr * g.y; c.z += nlr * g.z; c.w += nlr * g.w;
      C4[i] = c;
    }
    if (zero) T4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// ------------------------------------------------------------------ kernels
// PATH: 0 generic, 1 fast (h == 32), 2/3/4 tiled with 16/4/8-example chunks,
// 5 the fast path specialised to the Polyglot shape (d 64, n 5, h 32: the
// shape and the shape-only shared-memory offsets become compile-time
// constants, which removes most index arithmetic and shrinks the executed
// code -- the step is latency-bound and its code is fetched once per launch).
// ACT: the nonlinearity (PG_OPT_ACTIVATION), so a kernel carries one.
template <int PATH, int DP, int ACT>
__global__ void __launch_bounds__(384, 1) step_kernel(StepParams p_in, int phases) {
  extern __shared__ __align__(16) unsigned char smem[];
  // under PG_PDL=1 (launch_step_phases) the kernel may be placed before the
  // previous one has completed: nothing is read or written before it has
  asm volatile("griddepcontrol.wait;" ::: "memory");
  StepParams p = p_in;
  p.act = ACT;
  if (PATH == 5) {
    p.d = 64; p.n = 5; p.h = 32; p.T = kTMax;
    const Layout L = make_layout(64, 5, 32, kTMax, 384, 0, 1);
    const int lbase = p.lay.lbase, loff = p.lay.loff;
    p.lay = L;
    p.lay.lbase = lbase;
    p.lay.loff = loff;
  }
  trace_mark(p, 0);
  trace_clock(p, 12);
  if (phases & 1) {
    if (PATH == 1 || PATH == 5) phase1_fast(p, smem);
    else if (PATH == 2) phase1_tiled_t<kTT>(p, smem);
    else if (PATH == 3) phase1_tiled_t<kTTSmall>(p, smem);
    else if (PATH == 4) phase1_tiled_t<kTTMid>(p, smem);
    else phase1_generic(p, smem);
    __syncthreads();
    trace_mark(p, 6);
  }
  const bool prep = DP ? (phases & 8) != 0 : ((phases & 2) && p.mode == 0);
  if ((phases & 1) && (phases & 10)) {
    const unsigned long long target = grid_arrive(&p.st->bar_arrivals[gridDim.x - 1]);
    if (prep) phase2_prep(p, smem);   // overlaps the barrier
    grid_wait(&p.st->bar_arrivals[gridDim.x - 1], target);
  } else if (prep) {
    phase2_prep(p, smem);
    __syncthreads();
  }
  trace_mark(p, 7);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // the next step may begin its launch
  if (DP) {
    if (phases & 8) dp_publish(p, smem);
    if (phases & 16) {
      phase2_prep(p, smem);
      __syncthreads();
      dp_merge(p, smem);
    }
  } else if (phases & 2) {
    phase2<PATH == 3>(p, smem);
  }
  __syncthreads();
  trace_mark(p, 11);
  trace_clock(p, 13);
}

int step_dw1_gemm(int fast, int T) { return fast == 2 && T == kTTSmall; }

int step_fast_ok(int d, int n, int h) {
  const int nw = (n + 1) * (d / 32);
  if (h == 32 && d % 32 == 0 && d >= 32 && nw >= 8 && nw <= 12 && (n + 1) * kTMax <= kMaxKeys) return 1;
  if (d % 32 == 0 && h % 32 == 0 && h >= 64 && h <= 128 && (n + 1) * kTT <= kMaxKeys && (n + 1) * kTT <= 384)
    return 2;
  return 0;
}

int step_block_threads(int d, int n, int h, int fast) {
  if (fast == 1) return (n + 1) * (d / 32) * 32;  // 256..384 (step_fast_ok)
  return 384;
}

int step_chunk_T(int d, int n, int h, int fast, int per_cta) {
  // tiled path: the smallest of 4 / 8 / 16-example chunks that holds a CTA's
  // share (the large config at 512 examples per GPU: 3.5 per CTA)
  if (fast == 2) return per_cta <= kTTSmall ? kTTSmall : per_cta <= kTTMid ? kTTMid : kTT;
  int T = kTMax;
  while ((n + 1) * T > kMaxKeys) --T;
  if (!fast) {
    while (T > 1 && (T * (n + 1) * d + 5 * T * h) * 4 > 170 * 1024) --T;
  }
  return T;
}

static bool poly_shape(int d, int n, int h) { return d == 64 && n == 5 && h == 32; }

// The tiled path has one kernel per chunk size, so neither carries the other's
// code (a combined kernel ran the 16-example case 12 % slower); the data-
// parallel phases live in their own instantiations (DP = 1), so the one-GPU
// kernel carries none of their code either; likewise one kernel per
// nonlinearity, and the Polyglot shape has its own (PATH 5).
template <int DP, int ACT>
static const void* step_fn_t(int fast, int T, bool poly) {
  if (fast == 2)
    return T == kTTSmall ? (const void*)step_kernel<3, DP, ACT>
           : T == kTTMid ? (const void*)step_kernel<4, DP, ACT>
                         : (const void*)step_kernel<2, DP, ACT>;
  if (fast == 1) return poly ? (const void*)step_kernel<5, DP, ACT> : (const void*)step_kernel<1, DP, ACT>;
  return (const void*)step_kernel<0, DP, ACT>;
}
static const void* step_fn(int fast, int T, int dp, int act, bool poly) {
  if (dp) return act ? step_fn_t<1, 1>(fast, T, poly) : step_fn_t<1, 0>(fast, T, poly);
  return act ? step_fn_t<0, 1>(fast, T, poly) : step_fn_t<0, 0>(fast, T, poly);
}

// Allow up to the opt-in maximum minus the kernel's static shared memory.
cudaError_t step_prepare(int fast, size_t optin, size_t* usable) {
  size_t best = optin;
  for (int dp = 0; dp < 2; ++dp)
    for (int act = 0; act < 2; ++act)
      for (int poly = 0; poly < (fast == 1 ? 2 : 1); ++poly)
        for (int T : {kTT, kTTSmall, kTTMid}) {
          const void* fn = step_fn(fast, T, dp, act, poly != 0);
          cudaFuncAttributes fa;
          cudaError_t e = cudaFuncGetAttributes(&fa, fn);
          if (e != cudaSuccess) return e;
          const size_t smem = optin - fa.sharedSizeBytes;
          if (smem < best) best = smem;
          e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          if (e != cudaSuccess) return e;
          if (fast != 2) break;
        }
  if (usable) *usable = best;
  return cudaSuccess;
}

// Launch: the in-kernel grid barrier needs every CTA resident at once.  The
// default is a cooperative launch (the runtime co-schedules the grid even
// next to other work).  PG_PDL=1 selects a plain launch with programmatic
// stream serialisation instead: the kernel's first instruction is
// griddepcontrol.wait, so it reads nothing before the previous kernel on the
// stream has completed, but its CTAs are placed while the previous step drains
// (back-to-back steps: 2.5 -> 0.65 us between kernels, scripts/micro/launch_gap.cu;
// device-fed back-to-back Polyglot B = 4096 steps 28.4 -> 26.5 us; a
// cooperative launch does not overlap).  Co-residency is then by construction
// (P <= #SMs CTAs, one fits per SM), which holds only while no kernel that
// waits on this one occupies SMs concurrently -- hence opt-in.
void launch_step_phases(const StepParams& p, int phases, int fast, cudaStream_t s, int* launches) {
  const int NT = step_block_threads(p.d, p.n, p.h, fast);
  const bool poly = fast == 1 && poly_shape(p.d, p.n, p.h) && p.T == kTMax && NT == 384;
  const void* fn = step_fn(fast, p.T, (phases & 24) != 0, p.act, poly);
  void* args[] = {(void*)&p, (void*)&phases};
  static const int pdl = getenv("PG_PDL") ? atoi(getenv("PG_PDL")) : 0;
  const bool grid_sync = (phases & 1) && (phases & 10);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.P);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = (size_t)p.smem_bytes;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  if (pdl) {
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
  } else {
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
  }
  cfg.attrs = at;
  cfg.numAttrs = grid_sync || pdl ? 1 : 0;
  cudaLaunchKernelExC(&cfg, fn, args);
  *launches += 1;
}

void launch_step(const StepParams& p, int fused, int fast, cudaStream_t s, int* launches) {
  if (fused) {
    launch_step_phases(p, 3, fast, s, launches);
  } else {
    launch_step_phases(p, 1, fast, s, launches);
    launch_step_phases(p, 2, fast, s, launches);
  }
}

void launch_dp_table(const StepParams& p, float* table, int what, int num_sms, cudaStream_t s, int* launches) {
  if (what) dp_table_apply_kernel<<<num_sms * 4, 256, 0, s>>>(p, table, what == 2);
  else dp_table_scatter_kernel<<<p.P, 256, 0, s>>>(p, table);
  *launches += 1;
}

}  // namespace pg
