// scatter_det.cu -- deterministic W[I[k], :] += Y[k, :] (PAPER.md:98-102,
// 121-127) in ONE cooperative launch (n <= P * kOLoc; larger inputs take the
// radix-sort pipeline of scatter.cu).
//
// Each row's sum is formed in increasing k (one fixed association per row), so
// the result does not depend on timing: bit-reproducible run to run.  The
// north-star shape of the DET mode is "sort by row index, then a segmented
// reduction": here the sort is a bucket sort by OWNER CTA (row % P) -- one
// stable multi-split over the whole input -- followed by a stable sort of each
// owner's bucket by row / P in shared memory, and the segmented reduction runs
// over that order.  Rows the index stream hits very often (the Zipf head: one
// row alone takes 8 % of all entries) would overload their owner, so they are
// split by POSITION instead: every CTA reduces the head rows' entries of its
// own position range, and the per-CTA partials are summed in CTA order.
//
//   A  CTA c loads I[lo_c, hi_c) (its position range, <= kOLoc entries) into
//      registers, validates it, derives the head-row set from a fixed sample
//      (identical in every CTA: same sample, same ranking), tags each entry
//      with a digit -- owner o = row % P, or P + h for head row h -- and sorts
//      the range by that digit with ONE stable pass (warp-ballot ranks), so the
//      cold entries are grouped by owner and the head entries by (h, k).  The
//      per-owner counts H[c][o] are published.  Grid barrier (arrive); while it
//      completes:
//   H  the head entries' segmented sums (below) go to hpart[c][h].
//      Grid barrier (wait): a bad index anywhere stops every CTA here, before
//      any write to W.
//   B  every CTA reads H, forms each owner's bucket base (exclusive over
//      owners, then over CTAs) and copies its owner-sorted cold entries
//      (k, row / P) out, one contiguous run per owner -- so each bucket holds
//      its entries in increasing k.  Grid barrier.
//   C  owner o takes its bucket in windows of <= kOWin entries (k ranges),
//      sorts each window stably by row / P and runs the segmented reduction:
//      lane groups take fixed chunks of the sorted window, sum each segment's
//      Y rows in k order (kOU rows in flight per lane group), and a segment that
//      crosses a chunk boundary is finished, in chunk order, by the group it
//      starts in.  Each (row, window) total reaches W by ONE
//      red.global.add.v4.f32 (the row's only writer this call).
//   D  after a last grid barrier, head row h is finished by CTA h % P: its
//      partials summed in CTA order, one reduction into W.
#include "common.cuh"
#include "scatter.cuh"

#ifndef PG_OPF
#define PG_OPF 2
#endif

namespace pg {

#ifdef PG_TRACE
__device__ unsigned long long g_owner_tr[160][16];
#define OWN_MARK(k)                                                              \
  do {                                                                           \
    if (threadIdx.x == 0) {                                                      \
      unsigned long long t_;                                                     \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                     \
      g_owner_tr[blockIdx.x][k] = t_;                                            \
    }                                                                            \
  } while (0)
#else
#define OWN_MARK(k) do {} while (0)
#endif

constexpr int kOT = 1024;               // threads per CTA (one CTA per SM)
constexpr int kONW = kOT / 32;
constexpr int kOItems = 8;              // keys per thread in a block sort (kOT * kOItems = kOLoc)
constexpr int kOLoc = 8192;             // entries per position range (n <= P * kOLoc)
constexpr int kOWin = 8192;             // entries per owner window
constexpr int kOKeyBits = 13;           // window-local index bits of a sort key
constexpr int kOU = 4;                  // Y rows in flight per lane group (8 spills at 64 registers)
constexpr int kOMaxP = 181;             // P * P u16 counts fit the scratch; P + kOHot digits fit 9 bits
// head-row selection (the ATOMIC hot-set rule, scatter.cu, with a smaller
// sample): rows seen >= kOHotMin times in a fixed sample of kOSample entries
constexpr int kOSample = 2048;
constexpr int kOSampleHash = 4096;
constexpr int kOHotMin = 3;
constexpr int kOCand = 1024;            // >= kOSample / kOHotMin
constexpr int kOHot = 256;              // head rows at most
constexpr int kOHash = 1024;            // head-row lookup table
constexpr int kOTagBits = 9;            // digits of phase A: P + kOHot <= 512
constexpr int kORkBits = 10;            // digit width of phase C passes
static_assert(kOT * kOItems == kOLoc && kOLoc == kOWin && kOLoc == (1 << kOKeyBits), "tiles");
static_assert(kOMaxP + kOHot <= (1 << kOTagBits), "tag digits");

__host__ __device__ constexpr int o_align(int x) { return (x + 127) & ~127; }

// Shared-memory carve-up (bytes): a small header that lives to the end, the
// phase A-B region (row keys, head-row hash, the digit-sorted keys) and a
// scratch part reused by every phase; phase C takes the A-B region too.
struct OLayout {
  int hrow, misc, ab, srow, hkey, hslot, skeys, scratch, total;
};
__host__ __device__ inline OLayout o_layout(int P) {
  OLayout L{};
  int o = 0;
  L.hrow = o;    o = o_align(o + kOHot * 4);
  L.misc = o;    o = o_align(o + 64 * 4);
  L.ab = o;
  L.srow = o;    o = o_align(o + kOLoc * 4);
  L.hkey = o;    o = o_align(o + kOHash * 4);
  L.hslot = o;   o = o_align(o + kOHash * 4);
  L.skeys = o;   o = o_align(o + kOLoc * 4);
  L.scratch = o;
  const int abB = o - L.ab;
  const int pieceB = kONW * 32 * 2 * 16 + kONW * 32 * 4;                    // o_segreduce pieces + flags
  const int sampleB = 2 * kOSampleHash * 4 + kOCand * 8;                    // A: sample hash
  const int tagB = kONW * (1 << kOTagBits) * 2 + o_align(((1 << kOTagBits) + 1) * 4) + pieceB;   // A / H
  const int bucketB = o_align(kOMaxP * kOMaxP * 2) + 2 * 256 * 4;           // B: H as u16, bases
  const int winB = 3 * kOWin * 4 + kONW * (1 << kORkBits) * 2 + o_align(((1 << kORkBits) + 1) * 4) + pieceB - abB;   // C
  int s = sampleB;
  s = s > tagB ? s : tagB;
  s = s > bucketB ? s : bucketB;
  s = s > winB ? s : winB;
  (void)P;
  L.total = o + o_align(s);
  return L;
}

// One stable LSD pass of a block-wide radix sort on DB-bit digits: the keys sit
// in registers, warp w holding the strip [256 w, 256 (w+1)) (item j at
// 256 w + 32 j + lane), so strip order == key order; invalid items are
// dropped.  Ranks by warp ballots (one per digit bit), per-warp digit counts in
// `whist` ([kONW][2^DB] u16), then every valid key goes to out[digit start +
// warp offset + rank].  dstart[0..2^DB] receives the digit starts (and the
// total at [2^DB]).  Returns the number of valid keys.
template <int DB>
__device__ int o_pass(const unsigned (&key)[kOItems], const bool (&valid)[kOItems], int shift, unsigned* out,
                      unsigned short* whist, int* dstart, int* ws) {
  constexpr int kBins = 1 << DB;
  static_assert(kBins <= kOT, "one digit per thread in the scans");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  unsigned short* wh = whist + warp * kBins;
  for (int d = lane; d < kBins; d += 32) wh[d] = 0;
  __syncwarp();
  int lrank[kOItems];
  unsigned dig[kOItems];
#pragma unroll
  for (int j = 0; j < kOItems; ++j) {
    dig[j] = (key[j] >> shift) & (unsigned)(kBins - 1);
    unsigned peers = __ballot_sync(0xffffffffu, valid[j]);
#pragma unroll
    for (int b = 0; b < DB; ++b) {
      const bool bit = (dig[j] >> b) & 1u;
      const unsigned bb = __ballot_sync(0xffffffffu, bit);
      peers &= bit ? bb : ~bb;
    }
    const int before = valid[j] ? wh[dig[j]] : 0;
    __syncwarp();
    if (valid[j] && (peers & lt) == 0) wh[dig[j]] = (unsigned short)(before + __popc(peers));
    __syncwarp();
    lrank[j] = before + __popc(peers & lt);
  }
  __syncthreads();
  // per digit: exclusive over warps (warp order == strip order), then over digits
  int run = 0;
  if (tid < kBins) {
    for (int w = 0; w < kONW; ++w) {
      const int v = whist[w * kBins + tid];
      whist[w * kBins + tid] = (unsigned short)run;
      run += v;
    }
  }
  int total = 0;
  const int ex = block_excl_scan(run, ws, &total);
  if (tid < kBins) dstart[tid] = ex;
  if (tid == 0) dstart[kBins] = total;
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kOItems; ++j)
    if (valid[j]) out[dstart[dig[j]] + wh[dig[j]] + lrank[j]] = key[j];
  __syncthreads();
  return total;
}

// Segmented reduction over entries [0, cnt): ent(i) gives entry i's (k,
// segment); entries are sorted by segment, a segment's in increasing k.  Lane
// group g (q = cols / 4 lanes, one float4 of the row each) takes chunk
// [g E, (g+1) E) and sums each segment's Y rows in k order (the next batch's
// entries are fetched while the current batch's rows are in flight); complete
// segments go to emit(seg, sum4, lane quad), pieces of segments crossing a
// chunk boundary are parked in smem and finished, in chunk order, by the group
// the segment starts in.  `sm` holds the pieces ([NG][2][q] float4) and
// per-group flags.  Ends with a block barrier.
template <typename Ent, typename Emit>
__device__ void o_segreduce(int cnt, Ent&& ent, const float4* __restrict__ Y, int q, unsigned char* sm, Emit&& emit) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per = 32 / q;                 // lane groups per warp (q | 32, q <= 32)
  const int NG = kONW * per;
  const int sub = lane / q, gl = lane - sub * q;
  const int g = warp * per + sub;
  float4* piece = reinterpret_cast<float4*>(sm);                              // [NG][2][q]
  int* fl = reinterpret_cast<int*>(sm + (size_t)NG * 2 * q * 16);             // [NG]: bit0 crossR, bit1 middle piece
  int E = (cnt + NG - 1) / NG;
  if (E < 16) E = 16;
  const int s = g * E, e = min(cnt, s + E);
  const unsigned kEnd = 0xffffffffu;
  if (s < e) {
    const unsigned first = ent(s).y, last = ent(e - 1).y;
    const bool crossL = s > 0 && ent(s - 1).y == first;
    const bool crossR = e < cnt && ent(e).y == last;
    unsigned cur = first;
    bool atFirst = true;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    uint2 m[kOU];
#pragma unroll
    for (int u = 0; u < kOU; ++u) m[u] = s + u < e ? ent(s + u) : make_uint2(0u, kEnd);
    for (int i0 = s; i0 < e; i0 += kOU) {
      float4 v[kOU];
#pragma unroll
      for (int u = 0; u < kOU; ++u)
        v[u] = m[u].y != kEnd ? __ldcs(Y + (size_t)m[u].x * q + gl) : make_float4(0.f, 0.f, 0.f, 0.f);
      uint2 mn[kOU];
#pragma unroll
      for (int u = 0; u < kOU; ++u) mn[u] = i0 + kOU + u < e ? ent(i0 + kOU + u) : make_uint2(0u, kEnd);
#if PG_OPF > 0
      if (gl == 0) {   // rows PG_OPF batches ahead start moving into L2 (no registers held)
#pragma unroll
        for (int u = 0; u < kOU; ++u) {
          const int ip = i0 + (1 + PG_OPF) * kOU + u;
          if (ip < e) {
            const char* yr = reinterpret_cast<const char*>(Y + (size_t)ent(ip).x * q);
            for (int off = 0; off < 16 * q; off += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(yr + off));
          }
        }
      }
#endif
#pragma unroll
      for (int u = 0; u < kOU; ++u) {
        if (m[u].y == kEnd) break;
        if (m[u].y != cur) {   // segment `cur` ends inside the chunk
          if (atFirst && crossL) piece[(g * 2 + 0) * q + gl] = acc;   // head piece of a crossing segment
          else emit(cur, acc, gl);
          atFirst = false;
          cur = m[u].y;
          acc = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
      }
#pragma unroll
      for (int u = 0; u < kOU; ++u) m[u] = mn[u];
    }
    // the chunk's last segment
    if (crossR) {
      if (atFirst && crossL) piece[(g * 2 + 0) * q + gl] = acc;   // the whole chunk is one middle piece
      else piece[(g * 2 + 1) * q + gl] = acc;                     // tail piece
    } else if (atFirst && crossL) {
      piece[(g * 2 + 0) * q + gl] = acc;
    } else {
      emit(cur, acc, gl);
    }
    if (gl == 0) fl[g] = (crossR ? 1 : 0) | ((atFirst && crossL && crossR) ? 2 : 0);
  } else if (gl == 0) {
    fl[g] = 0;
  }
  __syncthreads();
  // finish crossing segments: the group holding a segment's first entry
  if (s < e && (fl[g] & 1) && !(fl[g] & 2)) {
    float4 a = piece[(g * 2 + 1) * q + gl];
    const unsigned segk = ent(e - 1).y;
    for (int h = g + 1; h < NG; ++h) {
      const float4 b = piece[(h * 2 + 0) * q + gl];
      a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
      if (!(fl[h] & 2)) break;   // h's head piece ends the segment
    }
    emit(segk, a, gl);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kOT, 1) sc_det_owner(const int32_t* __restrict__ I, const float* __restrict__ Y,
                                                       float* W, int64_t rows, int cols, int64_t n,
                                                       ScatterStatus* st, int par, int2* bucket, unsigned* Hcnt,
                                                       float* hpart, int* hmask, int64_t ypf_lines) {
  extern __shared__ __align__(128) unsigned char osm[];
  const int P = gridDim.x, c = blockIdx.x;
  const OLayout L = o_layout(P);
  int* hrow = reinterpret_cast<int*>(osm + L.hrow);
  int* misc = reinterpret_cast<int*>(osm + L.misc);
  int* srow = reinterpret_cast<int*>(osm + L.srow);
  int* hkey = reinterpret_cast<int*>(osm + L.hkey);
  int* hslot = reinterpret_cast<int*>(osm + L.hslot);
  unsigned* skeys = reinterpret_cast<unsigned*>(osm + L.skeys);
  unsigned char* scr = osm + L.scratch;
  __shared__ int ws[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = cols >> 2;
  const float4* Y4 = reinterpret_cast<const float4*>(Y);
  const int64_t lo = (int64_t)c * n / P, hi = (int64_t)(c + 1) * n / P;
  const int nl = (int)(hi - lo);

  OWN_MARK(0);
  // ---------------- A: this range's indices (strip layout) and the sample, all loads at once
  const int64_t ns = n < kOSample ? n : kOSample;
  const int64_t nruns = (ns + 31) / 32;
  const int64_t rstride = n / (nruns > 0 ? nruns : 1);
  constexpr int kSPer = (kOSample + kOT - 1) / kOT;
  int samp[kSPer];
#pragma unroll
  for (int j = 0; j < kSPer; ++j) {
    const int64_t i = (int64_t)j * kOT + tid;
    samp[j] = i < ns ? __ldg(I + (n <= kOSample ? i : (i >> 5) * rstride + (i & 31))) : -1;
  }
  int rv[kOItems];
#pragma unroll
  for (int j = 0; j < kOItems; ++j) {
    const int i = warp * 256 + j * 32 + lane;
    rv[j] = i < nl ? __ldg(I + lo + i) : 0;
  }
  {   // the head of Y into L2 while the serial phases run (HBM is otherwise idle)
    const char* yb = reinterpret_cast<const char*>(Y);
    for (int64_t l = (int64_t)c * kOT + tid; l < ypf_lines; l += (int64_t)P * kOT)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(yb + (l << 7)));
  }
  int* skey = reinterpret_cast<int*>(scr);
  int* scnt = skey + kOSampleHash;
  unsigned long long* cand = reinterpret_cast<unsigned long long*>(scnt + kOSampleHash);
  for (int i = tid; i < kOSampleHash; i += kOT) { skey[i] = -1; scnt[i] = 0; }
  for (int i = tid; i < kOHash; i += kOT) hkey[i] = -1;
  if (tid == 0) misc[0] = 0;
  bool bad[kOItems];
#pragma unroll
  for (int j = 0; j < kOItems; ++j) {
    const int i = warp * 256 + j * 32 + lane;
    bad[j] = i < nl && (rv[j] < 0 || (int64_t)rv[j] >= rows);
    if (bad[j]) {
      atomicMax(&st->hot[par].nbad, ~(((unsigned long long)(lo + i) << 32) | (unsigned)rv[j]));
      atomicOr(&st->hot[par].flag, 1);
    }
  }
  __syncthreads();
  OWN_MARK(10);
#pragma unroll
  for (int j = 0; j < kSPer; ++j) {
    const int row = samp[j];
    if (row < 0 || (int64_t)row >= rows) continue;
    unsigned h = ((unsigned)row * 2654435761u) & (kOSampleHash - 1);
    while (true) {
      const int prev = atomicCAS(&skey[h], -1, row);
      if (prev == -1 || prev == row) break;
      h = (h + 1) & (kOSampleHash - 1);
    }
    atomicAdd(&scnt[h], 1);
  }
  __syncthreads();
  OWN_MARK(11);
  for (int s2 = tid; s2 < kOSampleHash; s2 += kOT)
    if (skey[s2] != -1 && scnt[s2] >= kOHotMin) {
      const int a = atomicAdd(&misc[0], 1);
      cand[a] = ((unsigned long long)(kOSample - scnt[s2]) << 32) | (unsigned)skey[s2];
    }
  __syncthreads();
  const int nc = misc[0];
  if (nc > 1) {   // the same ranking in every CTA: (count desc, row asc)
    int npow = 32;
    while (npow < nc) npow <<= 1;
    for (int i = nc + tid; i < npow; i += kOT) cand[i] = ~0ull;
    __syncthreads();
    bitonic_sort_warp(cand, npow);
  }
  const int H = nc < kOHot ? nc : kOHot;
  for (int a = tid; a < H; a += kOT) {
    const int r = (int)(unsigned)(cand[a] & 0xffffffffull);
    hrow[a] = r;
    unsigned h = ((unsigned)r * 2654435761u) & (kOHash - 1);
    while (atomicCAS(&hkey[h], -1, r) != -1) h = (h + 1) & (kOHash - 1);
    hslot[h] = a;
  }
  __syncthreads();
  OWN_MARK(1);
  // digit: owner row % P (the entry keeps row / P), or P + h for head row h;
  // one stable pass sorts the range by digit
  unsigned short* whA = reinterpret_cast<unsigned short*>(scr);
  int* dsA = reinterpret_cast<int*>(scr + kONW * (1 << kOTagBits) * 2);
  unsigned char* rsm = scr + kONW * (1 << kOTagBits) * 2 + o_align(((1 << kOTagBits) + 1) * 4);
  {
    unsigned key[kOItems];
    bool val[kOItems];
#pragma unroll
    for (int j = 0; j < kOItems; ++j) {
      const int i = warp * 256 + j * 32 + lane;
      val[j] = i < nl && !bad[j];
      unsigned dg = 0;
      if (val[j]) {
        const int r = rv[j];
        int hid = -1;
        if (H > 0) {
          unsigned hh = ((unsigned)r * 2654435761u) & (kOHash - 1);
          int k;
          while ((k = hkey[hh]) != -1 && k != r) hh = (hh + 1) & (kOHash - 1);
          if (k == r) hid = hslot[hh];
        }
        if (hid >= 0) {
          dg = (unsigned)(P + hid);
        } else {
          const unsigned rk = (unsigned)r / (unsigned)P;
          dg = (unsigned)r - rk * (unsigned)P;
          srow[i] = (int)rk;
        }
      }
      key[j] = (dg << kOKeyBits) | (unsigned)i;
    }
    OWN_MARK(14);
    o_pass<kOTagBits>(key, val, kOKeyBits, skeys, whA, dsA, ws);
    OWN_MARK(15);
  }
  for (int o = tid; o < P; o += kOT) Hcnt[(size_t)c * P + o] = (unsigned)(dsA[o + 1] - dsA[o]);
  for (int h = tid; h < H; h += kOT) hmask[(size_t)c * kOHot + h] = dsA[P + h + 1] > dsA[P + h];
  const int ncold = dsA[P], nvalid = dsA[1 << kOTagBits];
  OWN_MARK(2);
  const unsigned long long target = grid_arrive(&st->hot_arrivals);

  // ---------------- H: the head entries (sorted by (P + h, k)), segmented sums into hpart[c][h]
  if (nvalid > ncold) {
    float4* hp = reinterpret_cast<float4*>(hpart) + (size_t)c * kOHot * q;
    const unsigned* hk = skeys + ncold;
    const unsigned klo = (unsigned)lo;
    o_segreduce(nvalid - ncold,
                [&](int i) { const unsigned kk = hk[i]; return make_uint2(klo + (kk & ((1u << kOKeyBits) - 1u)), kk >> kOKeyBits); },
                Y4, q, rsm, [&](unsigned dg, float4 a, int gl) { hp[(size_t)(dg - P) * q + gl] = a; });
  }
  OWN_MARK(3);
  grid_wait(&st->hot_arrivals, target);
  OWN_MARK(4);
  if (c == 0 && tid == 0) { st->hot[par ^ 1].flag = 0; st->hot[par ^ 1].nbad = 0ull; }
  if (*(volatile const int*)&st->hot[par].flag) return;

  // ---------------- B: bucket bases, then the owner-sorted cold entries copied out
  {
    unsigned short* Hs = reinterpret_cast<unsigned short*>(scr);                 // [P][P]
    int* base = reinterpret_cast<int*>(scr + o_align(kOMaxP * kOMaxP * 2));      // [P] this CTA's run starts
    int* dsB = base + 256;                                                        // dsA, kept (scr is reused)
    for (int o = tid; o <= P; o += kOT) dsB[o] = dsA[o];
    __syncthreads();
    {   // all of H in one round trip (P <= 181: <= 8 uint4 per thread)
      const int n4 = (P * P) >> 2;
      uint4 hv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = j * kOT + tid;
        hv[j] = i < n4 ? __ldcg(reinterpret_cast<const uint4*>(Hcnt) + i) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = j * kOT + tid;
        if (i < n4) {
          Hs[4 * i] = (unsigned short)hv[j].x; Hs[4 * i + 1] = (unsigned short)hv[j].y;
          Hs[4 * i + 2] = (unsigned short)hv[j].z; Hs[4 * i + 3] = (unsigned short)hv[j].w;
        }
      }
      for (int i = 4 * n4 + tid; i < P * P; i += kOT) Hs[i] = (unsigned short)__ldcg(Hcnt + i);
    }
    __syncthreads();
    OWN_MARK(12);
    int tot_o = 0, pre_o = 0;
    if (tid < P) {
#pragma unroll 8
      for (int cc = 0; cc < P; ++cc) {
        const int v = Hs[cc * P + tid];
        tot_o += v;
        pre_o += cc < c ? v : 0;
      }
    }
    int all;
    const int ex = block_excl_scan(tid < P ? tot_o : 0, ws, &all);
    if (tid < P) base[tid] = ex + pre_o;
    if (tid == c) { misc[1] = ex; misc[2] = ex + tot_o; }
    __syncthreads();
    OWN_MARK(13);
    for (int idx = tid; idx < ncold; idx += kOT) {   // coalesced: one contiguous run per owner
      const unsigned key = skeys[idx];
      const int o = (int)(key >> kOKeyBits), i = (int)(key & ((1u << kOKeyBits) - 1u));
      bucket[base[o] + (idx - dsB[o])] = make_int2((int)(lo + i), srow[i]);
    }
  }
  OWN_MARK(5);
  const unsigned long long t2 = grid_arrive(&st->hot_arrivals);
  grid_wait(&st->hot_arrivals, t2);
  OWN_MARK(6);

  // ---------------- C: owner c's bucket, windows of kOWin entries in k order,
  // each sorted stably by row / P, then segmented sums into W
  {
    const int b0 = misc[1], b1 = misc[2];
    int* wk = reinterpret_cast<int*>(osm + L.ab);                          // window entry j -> k
    unsigned* ka = reinterpret_cast<unsigned*>(osm + L.ab + kOWin * 4);
    unsigned* kb = ka + kOWin;
    unsigned short* wh = reinterpret_cast<unsigned short*>(osm + L.ab + 3 * kOWin * 4);
    int* ds = reinterpret_cast<int*>(osm + L.ab + 3 * kOWin * 4 + kONW * (1 << kORkBits) * 2);
    unsigned char* rsmC = osm + L.ab + 3 * kOWin * 4 + kONW * (1 << kORkBits) * 2 + o_align(((1 << kORkBits) + 1) * 4);
    const unsigned maxrk = (unsigned)((rows - 1) / P);
    const int sbits = maxrk ? 32 - __clz(maxrk) : 1;
    const int npass = (sbits + kORkBits - 1) / kORkBits;
    for (int w0 = b0; w0 < b1; w0 += kOWin) {
      const int m = min(kOWin, b1 - w0);
      unsigned key[kOItems];
      bool val[kOItems];
      int2 ev[kOItems];
#pragma unroll
      for (int j = 0; j < kOItems; ++j) {
        const int i = warp * 256 + j * 32 + lane;
        ev[j] = i < m ? __ldcg(bucket + w0 + i) : make_int2(0, 0);
      }
#pragma unroll
      for (int j = 0; j < kOItems; ++j) {
        const int i = warp * 256 + j * 32 + lane;
        val[j] = i < m;
        if (val[j]) wk[i] = ev[j].x;
        key[j] = ((unsigned)ev[j].y << kOKeyBits) | (unsigned)i;   // ev = (k, row / P)
      }
      unsigned* src = ka;
      o_pass<kORkBits>(key, val, kOKeyBits, src, wh, ds, ws);
      for (int ps = 1; ps < npass; ++ps) {
        unsigned* dst = src == ka ? kb : ka;
#pragma unroll
        for (int j = 0; j < kOItems; ++j) {
          const int i = warp * 256 + j * 32 + lane;
          key[j] = i < m ? src[i] : 0u;
        }
        o_pass<kORkBits>(key, val, kOKeyBits + ps * kORkBits, dst, wh, ds, ws);
        src = dst;
      }
      // (k, row / P) per sorted position, so the reduction needs one lookup per entry
      {
        unsigned sk[kOItems];
#pragma unroll
        for (int j = 0; j < kOItems; ++j) {
          const int i = warp * 256 + j * 32 + lane;
          sk[j] = i < m ? src[i] : 0u;
        }
        __syncthreads();
        uint2* ent = reinterpret_cast<uint2*>(ka);   // spans ka and kb
#pragma unroll
        for (int j = 0; j < kOItems; ++j) {
          const int i = warp * 256 + j * 32 + lane;
          if (i < m) ent[i] = make_uint2((unsigned)wk[sk[j] & ((1u << kOKeyBits) - 1u)], sk[j] >> kOKeyBits);
        }
        __syncthreads();
      }
      OWN_MARK(7);
      const uint2* ent = reinterpret_cast<const uint2*>(ka);
      o_segreduce(m, [&](int i) { return ent[i]; }, Y4, q, rsmC,
                  [&](unsigned rk, float4 a, int gl) { red_add_v4(W + ((size_t)rk * P + c) * cols + 4 * gl, a); });
    }
  }
  OWN_MARK(8);
  if (H == 0) return;
  // ---------------- D: head rows, partials summed in CTA order
  const unsigned long long t3 = grid_arrive(&st->hot_arrivals);
  grid_wait(&st->hot_arrivals, t3);
  {
    const int NGc = kOT / q;            // groups of q threads, one float4 each
    const int j = tid / q, f = tid - j * q;
    const int S = (P + NGc - 1) / NGc;  // consecutive CTAs per group (<= 6)
    float4* red = reinterpret_cast<float4*>(osm + L.ab);   // [NGc][q] (the A-B region is free)
    for (int h = c; h < H; h += P) {
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      int mk[8];
      float4 bv[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {   // every load at once
        const int cc = j * S + t;
        const bool ok = t < S && cc < P;
        mk[t] = ok ? __ldcg(hmask + (size_t)cc * kOHot + h) : 0;
        bv[t] = ok ? __ldcg(reinterpret_cast<const float4*>(hpart) + ((size_t)cc * kOHot + h) * q + f)
                   : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int t = 0; t < 8; ++t)
        if (mk[t]) { a.x += bv[t].x; a.y += bv[t].y; a.z += bv[t].z; a.w += bv[t].w; }
      red[j * q + f] = a;
      __syncthreads();
      if (tid < q) {
        float4 s4 = red[tid];
        for (int jj = 1; jj < NGc; ++jj) {
          const float4 b = red[jj * q + tid];
          s4.x += b.x; s4.y += b.y; s4.z += b.z; s4.w += b.w;
        }
        red_add_v4(W + (size_t)hrow[h] * cols + 4 * tid, s4);
      }
      __syncthreads();
    }
  }
  OWN_MARK(9);
}

#ifdef PG_TRACE
extern "C" int pg_debug_owner_trace(unsigned long long* out) {   // [160][16] globaltimer stamps
  return (int)cudaMemcpyFromSymbol(out, g_owner_tr, sizeof(g_owner_tr));
}
#endif

size_t det_owner_smem(int P) { return (size_t)o_layout(P).total; }

bool det_owner_ok(int64_t rows, int cols, int64_t n, int P) {
  // row / P must fit the 19 key bits above the window index
  return (cols & 3) == 0 && cols <= 128 && (32 % (cols / 4)) == 0 && P >= 2 && P <= kOMaxP &&
         n <= (int64_t)P * kOLoc && n < (1ll << 31) && rows < (1ll << 31) &&
         (rows - 1) / P < (1ll << (32 - kOKeyBits));
}

size_t det_owner_hpart_floats(int P, int cols) { return (size_t)P * kOHot * cols; }
size_t det_owner_hmask_ints(int P) { return (size_t)P * kOHot; }

cudaError_t det_owner_prepare() {
  return cudaFuncSetAttribute(sc_det_owner, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)det_owner_smem(kOMaxP));
}

cudaError_t det_owner_launch(const int32_t* I, const float* Y, float* W, int64_t rows, int cols, int64_t n,
                             ScatterStatus* st, int par, int2* bucket, unsigned* Hcnt, float* hpart, int* hmask,
                             int P, int64_t ypf_lines, cudaStream_t s) {
  void* args[] = {(void*)&I, (void*)&Y, (void*)&W, (void*)&rows, (void*)&cols, (void*)&n, (void*)&st, (void*)&par,
                  (void*)&bucket, (void*)&Hcnt, (void*)&hpart, (void*)&hmask, (void*)&ypf_lines};
  return cudaLaunchCooperativeKernel((const void*)sc_det_owner, P, kOT, args, det_owner_smem(P), s);
}

}  // namespace pg
