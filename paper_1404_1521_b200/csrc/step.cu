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
// The 6 rows per example (n+1 in general) replace the oracle's 2n unmerged
// rows; in exact arithmetic their scatter is identical (reading G7).
#include "common.cuh"
#include "step.cuh"

namespace pg {

constexpr int kTMax = 32;       // examples per chunk
constexpr int kMaxKeys = 256;   // (n+1)*T <= 256 keys per chunk
constexpr int kCapK = 2048;     // phase-2 owner-merge keys per window

// ------------------------------------------------------------------ smem layout
struct Layout {
  // phase 1
  int xs, pg, sig, gz, hinge, rows, skin, skey, uown, useg, ws, red;   // byte offsets
  // generic phase 1
  int A, Ac, SIG, DEL, DELc;
  // phase 2
  int lbase, keys, seg, stage, carry, dred, ws2;
  int SB;        // staged rows per sub-batch
  int total1, total2;
};

__host__ __device__ inline int align16(int x) { return (x + 15) & ~15; }

__host__ __device__ inline Layout make_layout(int d, int n, int h, int T, int NT, int NLtot, int fast) {
  Layout L{};
  int o = 0;
  const int NW = NT / 32;
  if (fast) {
    L.xs = o;    o = align16(o + NW * T * 32 * 4);
    L.pg = o;    o = align16(o + NW * T * 32 * 4);     // == T*(n+1)*d floats
    L.sig = o;   o = align16(o + 3 * T * 32 * 4);
    L.A = L.Ac = L.SIG = L.DEL = L.DELc = 0;
  } else {
    L.xs = o;    o = align16(o + T * (n + 1) * d * 4); // X, later G rows
    L.pg = L.xs;
    L.A = o;     o = align16(o + T * h * 4);
    L.Ac = o;    o = align16(o + T * h * 4);
    L.SIG = o;   o = align16(o + T * h * 4);
    L.DEL = o;   o = align16(o + T * h * 4);
    L.DELc = o;  o = align16(o + T * h * 4);
    L.sig = 0;
  }
  L.gz = o;    o = align16(o + kTMax * 4);
  L.hinge = o; o = align16(o + kTMax * 4);
  L.rows = o;  o = align16(o + kMaxKeys * 4);
  L.skin = o;  o = align16(o + kMaxKeys * 8);
  L.skey = o;  o = align16(o + kMaxKeys * 8);
  L.uown = o;  o = align16(o + kMaxKeys * 4);
  L.useg = o;  o = align16(o + (kMaxKeys + 1) * 4);
  L.ws = o;    o = align16(o + 64 * 4);
  L.red = o;   o = align16(o + 2 * 32 * 32 * 4);     // per-warp db1/dw2 partials
  L.total1 = o;
  // phase 2 (aliases phase 1 storage)
  o = 0;
  L.lbase = o; o = align16(o + (NLtot + 1) * 4);
  L.keys = o;  o = align16(o + kCapK * 8);
  L.seg = o;   o = align16(o + (kCapK + 1) * 4);
  int SB = 65536 / (d * 4);
  if (SB > 512) SB = 512;
  if (SB < 16) SB = 16;
  L.SB = SB;
  L.stage = o; o = align16(o + SB * d * 4);
  L.carry = o; o = align16(o + d * 4);
  L.dred = o;  o = align16(o + NT * 16);
  L.ws2 = o;   o = align16(o + 64 * 4);
  L.total2 = o;
  return L;
}

// ------------------------------------------------------------------ error reporting
__device__ __forceinline__ void report_bad(DevStatus* st, long long pos, int value) {
  unsigned long long packed = ((unsigned long long)pos << 32) | (unsigned)value;
  atomicMin(&st->bad, packed);
  atomicOr(&st->flags, 1);
}

// ------------------------------------------------------------------ CTA-local aggregation
// Keys: rows_s[i] for i < K (i = example*(n+1) + ext-slot), gradient rows Gs[i][0..d).
// Sort by (owner = row % P, row, i); sum each row's gradient rows in i order;
// write list L: rows, sums and per-owner offsets.
__device__ void aggregate_chunk(const StepParams& p, int L, int K, const int* rows_s,
                                const float* Gs, unsigned char* sm, const Layout& lay) {
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, warp = tid >> 5, NW = NT >> 5;
  unsigned long long* skin = reinterpret_cast<unsigned long long*>(sm + lay.skin);
  unsigned long long* skey = reinterpret_cast<unsigned long long*>(sm + lay.skey);
  int* uown = reinterpret_cast<int*>(sm + lay.uown);
  int* useg = reinterpret_cast<int*>(sm + lay.useg);
  int* ws = reinterpret_cast<int*>(sm + lay.ws);
  const int P = p.P, d = p.d;
  for (int i = tid; i < K; i += NT) {
    unsigned row = (unsigned)rows_s[i];
    unsigned owner = row % (unsigned)P;
    skin[i] = ((unsigned long long)owner << 40) | ((unsigned long long)row << 8) | (unsigned)i;
  }
  __syncthreads();
  // rank sort (keys unique): O(K^2) broadcast comparisons, K <= 256
  for (int i = tid; i < K; i += NT) {
    unsigned long long k = skin[i];
    int r = 0;
    for (int j = 0; j < K; ++j) r += skin[j] < k;
    skey[r] = k;
  }
  __syncthreads();
  int head = 0;
  if (tid < K) {
    unsigned long long k = skey[tid];
    head = (tid == 0) || (((k >> 8) & 0xffffffffull) != ((skey[tid - 1] >> 8) & 0xffffffffull));
  }
  int U;
  int hidx = block_excl_scan(head, ws, &U);
  int32_t* lrows = p.list_rows + (size_t)L * p.cap;
  float* lvals = p.list_vals + (size_t)L * p.cap * d;
  if (tid < K && head) {
    unsigned long long k = skey[tid];
    useg[hidx] = tid;
    uown[hidx] = (int)(k >> 40);
    lrows[hidx] = (int)((k >> 8) & 0xffffffffull);
  }
  if (tid == 0) useg[U] = K;
  __syncthreads();
  // per-owner offsets: off[q] = #unique entries with owner < q (uown ascending)
  int32_t* off = p.list_off + (size_t)L * (P + 1);
  for (int q = tid; q <= P; q += NT) {
    int lo = 0, hi = U;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (uown[mid] < q) lo = mid + 1; else hi = mid;
    }
    off[q] = lo;
  }
  // segment sums in position order
  for (int j = warp; j < U; j += NW) {
    const int s0 = useg[j], s1 = useg[j + 1];
    for (int f = lane; f < d; f += 32) {
      float acc = 0.f;
      for (int r = s0; r < s1; ++r) acc += Gs[(int)(skey[r] & 0xffull) * d + f];
      lvals[(size_t)j * d + f] = acc;
    }
  }
  __syncthreads();
}

__device__ void write_empty_list(const StepParams& p, int L) {
  int32_t* off = p.list_off + (size_t)L * (p.P + 1);
  for (int q = threadIdx.x; q <= p.P; q += blockDim.x) off[q] = 0;
}

// ------------------------------------------------------------------ FAST phase 1
// h == 32 (lane == hidden unit), d % 32 == 0, NW = (n+1)*d/32 warps; warp w owns
// the 32-feature block (slot = w / (d/32), blk = w % (d/32)) of the extended
// input [x_0 .. x_{n-1}, x'_c]; its W1 rows live in registers for the whole
// step (Wcol for the forward, Wrow for the gradient rows).
__device__ void phase1_fast(const StepParams& p, unsigned char* sm, const Layout& lay) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NW = blockDim.x >> 5;
  const int d = p.d, n = p.n, T = p.T, DB = d >> 5, c = n >> 1;
  const int slot = warp / DB, blk = warp % DB;
  const int wslot = slot == n ? c : slot;
  const int wrow0 = wslot * d + blk * 32;
  const int sel = slot == n ? 2 : (slot == c ? 1 : 0);  // sigma / delta / delta'
  float* xs = reinterpret_cast<float*>(sm + lay.xs);
  float* pg = reinterpret_cast<float*>(sm + lay.pg);
  float* sig = reinterpret_cast<float*>(sm + lay.sig);
  float* hinge_s = reinterpret_cast<float*>(sm + lay.hinge);
  int* rows_s = reinterpret_cast<int*>(sm + lay.rows);
  float* red = reinterpret_cast<float*>(sm + lay.red);

  float Wcol[32], Wrow[32], dacc[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) Wcol[k] = __ldg(p.W1 + (size_t)(wrow0 + k) * 32 + lane);
  {
    const float4* wr = reinterpret_cast<const float4*>(p.W1 + (size_t)(wrow0 + lane) * 32);
#pragma unroll
    for (int u4 = 0; u4 < 8; ++u4) {
      float4 v = __ldg(wr + u4);
      Wrow[4 * u4] = v.x; Wrow[4 * u4 + 1] = v.y; Wrow[4 * u4 + 2] = v.z; Wrow[4 * u4 + 3] = v.w;
    }
  }
#pragma unroll
  for (int u = 0; u < 32; ++u) dacc[u] = 0.f;
  const float b1 = __ldg(p.b1 + lane), w2 = __ldg(p.w2 + lane), b2 = __ldg(p.b2);
  float acc_db1 = 0.f, acc_dw2 = 0.f, acc_hinge = 0.f;

  const long long lo = (long long)blockIdx.x * p.B / p.P;
  const long long hi = (long long)(blockIdx.x + 1) * p.B / p.P;
  for (int r = 0; r < p.R; ++r) {
    const long long e0 = lo + (long long)r * T;
    const int cnt = (int)(hi - e0 < T ? (hi - e0 > 0 ? hi - e0 : 0) : T);
    const int L = blockIdx.x * p.R + r;
    if (cnt <= 0) { write_empty_list(p, L); continue; }
    // ---- gather (each warp its own feature block; warp-private smem)
    float* xw = xs + (size_t)warp * T * 32;
    for (int e = 0; e < cnt; ++e) {
      const long long ex = e0 + e;
      int row = slot < n ? __ldg(p.idx + ex * n + slot) : __ldg(p.corr + ex);
      const bool ok = row >= 0 && (long long)row < p.V;
      if (!ok && blk == 0 && lane == 0)
        report_bad(p.st, slot < n ? ex * n + slot : (long long)p.B * n + ex, row);
      xw[e * 32 + lane] = ok ? __ldg(p.C + (size_t)row * d + blk * 32 + lane) : 0.f;
      if (blk == 0 && lane == 0) rows_s[e * (n + 1) + slot] = ok ? row : 0;
    }
    __syncwarp();
    // ---- forward partials: part[warp][e][u] = sum_k x[e][k] W1[wrow0+k][u]
    float* part = pg;
    for (int e = 0; e < cnt; e += 4) {
      float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
      const float4* x0 = reinterpret_cast<const float4*>(xw + (e + 0) * 32);
      const float4* x1 = reinterpret_cast<const float4*>(xw + min(e + 1, cnt - 1) * 32);
      const float4* x2 = reinterpret_cast<const float4*>(xw + min(e + 2, cnt - 1) * 32);
      const float4* x3 = reinterpret_cast<const float4*>(xw + min(e + 3, cnt - 1) * 32);
#pragma unroll
      for (int k4 = 0; k4 < 8; ++k4) {
        float4 v0 = x0[k4], v1 = x1[k4], v2 = x2[k4], v3 = x3[k4];
        a0 = fmaf(v0.x, Wcol[4 * k4], a0); a0 = fmaf(v0.y, Wcol[4 * k4 + 1], a0);
        a0 = fmaf(v0.z, Wcol[4 * k4 + 2], a0); a0 = fmaf(v0.w, Wcol[4 * k4 + 3], a0);
        a1 = fmaf(v1.x, Wcol[4 * k4], a1); a1 = fmaf(v1.y, Wcol[4 * k4 + 1], a1);
        a1 = fmaf(v1.z, Wcol[4 * k4 + 2], a1); a1 = fmaf(v1.w, Wcol[4 * k4 + 3], a1);
        a2 = fmaf(v2.x, Wcol[4 * k4], a2); a2 = fmaf(v2.y, Wcol[4 * k4 + 1], a2);
        a2 = fmaf(v2.z, Wcol[4 * k4 + 2], a2); a2 = fmaf(v2.w, Wcol[4 * k4 + 3], a2);
        a3 = fmaf(v3.x, Wcol[4 * k4], a3); a3 = fmaf(v3.y, Wcol[4 * k4 + 1], a3);
        a3 = fmaf(v3.z, Wcol[4 * k4 + 2], a3); a3 = fmaf(v3.w, Wcol[4 * k4 + 3], a3);
      }
      part[(warp * T + e) * 32 + lane] = a0;
      if (e + 1 < cnt) part[(warp * T + e + 1) * 32 + lane] = a1;
      if (e + 2 < cnt) part[(warp * T + e + 2) * 32 + lane] = a2;
      if (e + 3 < cnt) part[(warp * T + e + 3) * 32 + lane] = a3;
    }
    __syncthreads();
    // ---- sigma stage: warp per example, lane = hidden unit
    for (int e = warp; e < cnt; e += NW) {
      float actx = 0.f, acen = 0.f, acor = 0.f;
      for (int s = 0; s < n; ++s) {
        if (s == c) continue;
        for (int b = 0; b < DB; ++b) actx += part[((s * DB + b) * T + e) * 32 + lane];
      }
      for (int b = 0; b < DB; ++b) {
        acen += part[((c * DB + b) * T + e) * 32 + lane];
        acor += part[((n * DB + b) * T + e) * 32 + lane];
      }
      const float base = b1 + actx;
      const float a = base + acen, ac = base + acor;
      const float z = fminf(fmaxf(a, -1.f), 1.f), zc = fminf(fmaxf(ac, -1.f), 1.f);
      const float s = warp_sum(w2 * z) + b2;
      const float sc = warp_sum(w2 * zc) + b2;
      const float m = 1.f - s + sc;
      const bool active = m > 0.f;
      const float g = active ? -p.inv_B : 0.f;
      const float dl = fabsf(a) < 1.f ? g * w2 : 0.f;
      const float dlc = fabsf(ac) < 1.f ? -g * w2 : 0.f;
      sig[(0 * T + e) * 32 + lane] = dl + dlc;
      sig[(1 * T + e) * 32 + lane] = dl;
      sig[(2 * T + e) * 32 + lane] = dlc;
      acc_db1 += dl + dlc;
      acc_dw2 += g * z + (-g) * zc;
      if (lane == 0) acc_hinge += active ? m : 0.f;
    }
    __syncthreads();
    // ---- backward: gradient rows G[e][slot][blk*32+lane] and dW1 rows
    float* Gs = pg;   // part is dead now
    const float* sv_base = sig + sel * T * 32;
    for (int e = 0; e < cnt; ++e) {
      const float xl = xw[e * 32 + lane];
      const float4* sv = reinterpret_cast<const float4*>(sv_base + e * 32);
      float g0 = 0.f, g1 = 0.f, g2 = 0.f, g3 = 0.f;
#pragma unroll
      for (int u4 = 0; u4 < 8; ++u4) {
        float4 v = sv[u4];
        g0 = fmaf(Wrow[4 * u4], v.x, g0);
        g1 = fmaf(Wrow[4 * u4 + 1], v.y, g1);
        g2 = fmaf(Wrow[4 * u4 + 2], v.z, g2);
        g3 = fmaf(Wrow[4 * u4 + 3], v.w, g3);
        dacc[4 * u4] = fmaf(xl, v.x, dacc[4 * u4]);
        dacc[4 * u4 + 1] = fmaf(xl, v.y, dacc[4 * u4 + 1]);
        dacc[4 * u4 + 2] = fmaf(xl, v.z, dacc[4 * u4 + 2]);
        dacc[4 * u4 + 3] = fmaf(xl, v.w, dacc[4 * u4 + 3]);
      }
      Gs[(e * (n + 1) + slot) * d + blk * 32 + lane] = (g0 + g1) + (g2 + g3);
    }
    __syncthreads();
    aggregate_chunk(p, L, cnt * (n + 1), rows_s, Gs, sm, lay);
  }
  // ---- per-CTA dense partial record: dW1 | db1 | dw2 | hinge
  float* rec = p.dense_part + (size_t)blockIdx.x * p.dense_stride;
  float* dsm = xs;   // [NW][32][33]
#pragma unroll
  for (int u = 0; u < 32; ++u) dsm[(warp * 32 + lane) * 33 + u] = dacc[u];
  red[warp * 32 + lane] = acc_db1;
  red[32 * 32 + warp * 32 + lane] = acc_dw2;
  if (lane == 0) hinge_s[warp] = acc_hinge;
  __syncthreads();
  const int ndh = n * d * 32;
  for (int i = tid; i < ndh; i += blockDim.x) {
    const int row = i >> 5, u = i & 31;
    const int s = row / d, j = row % d;
    const int w = s * DB + (j >> 5), l = j & 31;
    float v = dsm[(w * 32 + l) * 33 + u];
    if (s == c) v += dsm[((n * DB + (j >> 5)) * 32 + l) * 33 + u];
    rec[i] = v;
  }
  if (tid < 32) {
    float a = 0.f, b = 0.f;
    for (int w = 0; w < NW; ++w) { a += red[w * 32 + tid]; b += red[32 * 32 + w * 32 + tid]; }
    rec[ndh + tid] = a;
    rec[ndh + 32 + tid] = b;
  }
  if (tid == 0) {
    float hsum = 0.f;
    for (int w = 0; w < NW; ++w) hsum += hinge_s[w];
    rec[ndh + 64] = hsum;
    for (int i = ndh + 65; i < p.dense_stride; ++i) rec[i] = 0.f;
  }
}

// ------------------------------------------------------------------ GENERIC phase 1
// Any (d, n, h) with h <= 128: plain per-thread loops, W1 read through L1.
__device__ void phase1_generic(const StepParams& p, unsigned char* sm, const Layout& lay) {
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
    // gather rows of the extended window into X[e][slot][j]
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
      X[i] = row >= 0 ? __ldg(p.C + (size_t)row * d + j) : 0.f;
    }
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
    // sigma stage: warp per example
    for (int e = warp; e < cnt; e += NW) {
      float sp = 0.f, spc = 0.f;
      for (int u = lane; u < h; u += 32) {
        const float w2 = __ldg(p.w2 + u);
        sp += w2 * fminf(fmaxf(A[e * h + u], -1.f), 1.f);
        spc += w2 * fminf(fmaxf(Ac[e * h + u], -1.f), 1.f);
      }
      const float s = warp_sum(sp) + b2, sc = warp_sum(spc) + b2;
      const float m = 1.f - s + sc;
      const bool active = m > 0.f;
      const float g = active ? -p.inv_B : 0.f;
      for (int u = lane; u < h; u += 32) {
        const float w2 = __ldg(p.w2 + u);
        const float dl = fabsf(A[e * h + u]) < 1.f ? g * w2 : 0.f;
        const float dlc = fabsf(Ac[e * h + u]) < 1.f ? -g * w2 : 0.f;
        DEL[e * h + u] = dl; DELc[e * h + u] = dlc; SIG[e * h + u] = dl + dlc;
      }
      if (lane == 0) { gz[e] = g; hinge_s[e] = active ? m : 0.f; }
    }
    __syncthreads();
    // dense partials (accumulated across chunks in this CTA's record)
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
        const float z = fminf(fmaxf(A[e * h + u], -1.f), 1.f);
        const float zc = fminf(fmaxf(Ac[e * h + u], -1.f), 1.f);
        dw += gz[e] * z + (-gz[e]) * zc;
      }
      rec[ndh + u] = first ? db : rec[ndh + u] + db;
      rec[ndh + h + u] = first ? dw : rec[ndh + h + u] + dw;
    }
    if (tid == 0) for (int e = 0; e < cnt; ++e) hinge_acc += hinge_s[e];
    __syncthreads();
    // gradient rows into X's storage (X no longer needed)
    float* Gs = X;
    // compute into registers first, then write, to avoid overwriting X mid-use
    // (G does not read X, so write directly)
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
    aggregate_chunk(p, L, cnt * (n + 1), rows_s, Gs, sm, lay);
    first = false;
  }
  if (first) {  // no examples at all in this CTA
    for (int i = tid; i < p.dense_stride; i += NT) rec[i] = 0.f;
  } else if (tid == 0) {
    rec[ndh + 2 * h] = hinge_acc;
    for (int i = ndh + 2 * h + 1; i < p.dense_stride; ++i) rec[i] = 0.f;
  }
}

// ------------------------------------------------------------------ phase 2
__device__ __forceinline__ float* param_ptr(const StepParams& p, int i, int ndh) {
  if (i < ndh) return p.W1 + i;
  if (i < ndh + p.h) return p.b1 + (i - ndh);
  return p.w2 + (i - ndh - p.h);
}

__device__ void phase2_dense(const StepParams& p, unsigned char* sm, const Layout& lay) {
  const int tid = threadIdx.x, NT = blockDim.x;
  const int DL = p.dense_len, ndh = p.n * p.d * p.h;
  const int NQ = (DL + 3) / 4;
  const int G = gridDim.x;
  const int q0 = (int)((long long)blockIdx.x * NQ / G), q1 = (int)((long long)(blockIdx.x + 1) * NQ / G);
  float4* dred = reinterpret_cast<float4*>(sm + lay.dred);
  for (int qb = q0; qb < q1; qb += NT) {
    const int nq = min(NT, q1 - qb);
    int groups = NT / nq;
    if (groups > 32) groups = 32;
    const int qi = tid % nq, g = tid / nq;
    if (g < groups) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int r = g; r < p.Ptot; r += groups) {
        float4 v = ldcg4(p.dense_part + (size_t)r * p.dense_stride + 4 * (qb + qi));
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      dred[g * nq + qi] = acc;
    }
    __syncthreads();
    if (tid < nq) {
      float4 s = dred[tid];
      for (int gg = 1; gg < groups; ++gg) {
        float4 v = dred[gg * nq + tid];
        s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
      }
      const float sv[4] = {s.x, s.y, s.z, s.w};
      const int base = 4 * (qb + tid);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int i = base + k;
        if (i < DL) {
          float* q = param_ptr(p, i, ndh);
          *q = *q - p.lr * sv[k];
        }
      }
    }
    __syncthreads();
  }
}

// Bitonic sort of n (power of two) 64-bit keys in smem.
__device__ void bitonic_sort(unsigned long long* k, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
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

// Deterministic owner merge: CTA q owns rows with row % P == q.  Its entries
// from every list are sorted by (row, list) and each row's list partials are
// summed in list order, then C[row] += -lr * sum.
__device__ void phase2_scatter_det(const StepParams& p, unsigned char* sm, const Layout& lay) {
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, warp = tid >> 5, NW = NT >> 5;
  const int q = blockIdx.x, P = p.P, d = p.d, NL = p.NLtot;
  int* lbase = reinterpret_cast<int*>(sm + lay.lbase);
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(sm + lay.keys);
  int* seg = reinterpret_cast<int*>(sm + lay.seg);
  float* stage = reinterpret_cast<float*>(sm + lay.stage);
  float* carry = reinterpret_cast<float*>(sm + lay.carry);
  int* ws = reinterpret_cast<int*>(sm + lay.ws2);
  const float nlr = -p.lr;
  // counts per list, exclusive scan -> lbase
  int running = 0;
  for (int L0 = 0; L0 < NL; L0 += NT) {
    const int L = L0 + tid;
    int cnt = 0;
    if (L < NL) {
      const int32_t* off = p.list_off + (size_t)L * (P + 1);
      cnt = __ldcg(off + q + 1) - __ldcg(off + q);
    }
    int tot;
    int ex = block_excl_scan(cnt, ws, &tot);
    if (L < NL) lbase[L] = running + ex;
    running += tot;
  }
  if (tid == 0) lbase[NL] = running;
  __syncthreads();
  const int M = running;
  if (M == 0) return;
  // windows of whole lists with at most kCapK entries
  int La = 0;
  while (La < NL) {
    int Lb = La;
    while (Lb < NL && lbase[Lb + 1] - lbase[La] <= kCapK) ++Lb;
    const int base = lbase[La], Mw = lbase[Lb] - base;
    if (Mw > 0) {
      int npow = 1;
      while (npow < Mw) npow <<= 1;
      for (int e = tid; e < npow; e += NT) {
        if (e < Mw) {
          int lo = La, hi = Lb - 1;   // find L with lbase[L] <= base+e < lbase[L+1]
          while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (lbase[mid] <= base + e) lo = mid; else hi = mid - 1;
          }
          const int L = lo;
          const int j = __ldcg(p.list_off + (size_t)L * (P + 1) + q) + (base + e - lbase[L]);
          const unsigned row = (unsigned)__ldcg(p.list_rows + (size_t)L * p.cap + j);
          keys[e] = ((unsigned long long)row << 32) | ((unsigned long long)L << 8) | (unsigned)j;
        } else {
          keys[e] = ~0ull;
        }
      }
      __syncthreads();
      bitonic_sort(keys, npow);
      // segment heads
      int nseg_total = 0;
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
      // sub-batches of SB staged rows
      for (int sb0 = 0; sb0 < Mw; sb0 += lay.SB) {
        const int sb1 = min(Mw, sb0 + lay.SB);
        const int d4 = d >> 2;
        if ((d & 3) == 0) {
          for (int t = tid; t < (sb1 - sb0) * d4; t += NT) {
            const int e = sb0 + t / d4, f4 = t % d4;
            const unsigned long long k = keys[e];
            const int L = (int)((k >> 8) & 0xffffff), j = (int)(k & 0xff);
            reinterpret_cast<float4*>(stage)[t] = ldcg4(p.list_vals + ((size_t)L * p.cap + j) * d + 4 * f4);
          }
        } else {
          for (int t = tid; t < (sb1 - sb0) * d; t += NT) {
            const int e = sb0 + t / d, f = t % d;
            const unsigned long long k = keys[e];
            const int L = (int)((k >> 8) & 0xffffff), j = (int)(k & 0xff);
            stage[t] = __ldcg(p.list_vals + ((size_t)L * p.cap + j) * d + f);
          }
        }
        __syncthreads();
        // segments overlapping [sb0, sb1)
        int slo = 0, shi = nseg_total - 1;   // last segment starting <= sb0
        while (slo < shi) {
          int mid = (slo + shi + 1) >> 1;
          if (seg[mid] <= sb0) slo = mid; else shi = mid - 1;
        }
        for (int sidx = slo + warp; sidx < nseg_total && seg[sidx] < sb1; sidx += NW) {
          const int s0 = seg[sidx], s1 = seg[sidx + 1];
          const int a0 = max(s0, sb0), a1 = min(s1, sb1);
          const bool cont = s0 < sb0, fin = s1 <= sb1;
          const unsigned row = (unsigned)(keys[s0] >> 32);
          for (int f = lane; f < d; f += 32) {
            float acc = cont ? carry[f] : 0.f;
            for (int e = a0; e < a1; ++e) acc += stage[(e - sb0) * d + f];
            if (fin) {
              float* cp = p.C + (size_t)row * d + f;
              *cp = __ldcg(cp) + nlr * acc;
            } else {
              carry[f] = acc;
            }
          }
        }
        __syncthreads();
      }
    }
    La = Lb;
  }
}

// Atomic scatter: CTA b applies lists L = b, b+G, ... with red.global.add.v4.f32.
__device__ void phase2_scatter_atomic(const StepParams& p) {
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, warp = tid >> 5, NW = NT >> 5;
  const int P = p.P, d = p.d;
  const float nlr = -p.lr;
  for (int L = blockIdx.x; L < p.NLtot; L += gridDim.x) {
    const int U = __ldcg(p.list_off + (size_t)L * (P + 1) + P);
    for (int j = warp; j < U; j += NW) {
      const int row = __ldcg(p.list_rows + (size_t)L * p.cap + j);
      const float* src = p.list_vals + ((size_t)L * p.cap + j) * d;
      float* dst = p.C + (size_t)row * d;
      if ((d & 3) == 0) {
        for (int f4 = lane; f4 < (d >> 2); f4 += 32) {
          float4 v = ldcg4(src + 4 * f4);
          v.x *= nlr; v.y *= nlr; v.z *= nlr; v.w *= nlr;
          red_add_v4(dst + 4 * f4, v);
        }
      } else {
        for (int f = lane; f < d; f += 32) atomicAdd(dst + f, nlr * __ldcg(src + f));
      }
    }
  }
}

__device__ void phase2(const StepParams& p, unsigned char* sm, const Layout& lay) {
  __shared__ int s_flags;
  __shared__ float s_loss;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  DevStatus* st = p.st;
  if (tid == 0) {
    const int f = *(volatile int*)&st->flags;
    const unsigned long long bad = *(volatile unsigned long long*)&st->bad;
    s_flags = f;
    if (blockIdx.x == 0) {
      st->last_flags = f;
      st->last_bad = bad;
    }
    __threadfence();
    if (atomicAdd(&st->done, 1u) == gridDim.x - 1) {  // everyone has read the flags
      st->flags = 0;
      st->bad = kNoBad;
      st->done = 0;
      __threadfence();
    }
  }
  if (warp == 0) {
    float acc = 0.f;
    const int hoff = p.dense_len;
    for (int r = lane; r < p.Ptot; r += 32) acc += __ldcg(p.dense_part + (size_t)r * p.dense_stride + hoff);
    acc = warp_sum(acc);
    if (lane == 0) s_loss = acc * p.inv_B;
  }
  __syncthreads();
  const float loss = s_loss;
  const bool diverged = !isfinite(loss);
  const int flags = s_flags | (diverged ? 2 : 0);
  if (blockIdx.x == 0 && tid == 0) {
    st->last_loss = loss;
    st->last_flags = flags;
    if (p.loss_out) *p.loss_out = loss;
    if (flags) {
      atomicOr(&st->sticky_flags, flags);
      atomicMin(&st->sticky_bad, st->last_bad);
    }
  }
  if (flags) return;   // no parameter changes on a bad index or a non-finite loss
  phase2_dense(p, sm, lay);
  __syncthreads();
  if (p.mode == 0) phase2_scatter_det(p, sm, lay);
  else phase2_scatter_atomic(p);
}

// ------------------------------------------------------------------ kernels
template <bool FAST>
__global__ void __launch_bounds__(384, 1) step_kernel(StepParams p, int phases) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Layout lay = make_layout(p.d, p.n, p.h, p.T, blockDim.x, p.NLtot, FAST);
  if (phases & 1) {
    if (FAST) phase1_fast(p, smem, lay);
    else phase1_generic(p, smem, lay);
  }
  if (phases == 3) grid_barrier(&p.st->bar_count, &p.st->bar_gen);
  if (phases & 2) phase2(p, smem, lay);
}

int step_fast_ok(int d, int n, int h) {
  const int nw = (n + 1) * (d / 32);
  return h == 32 && d % 32 == 0 && d >= 32 && nw >= 8 && nw <= 12 && (n + 1) * kTMax <= kMaxKeys;
}

int step_block_threads(int d, int n, int h, int fast) {
  if (fast) return (n + 1) * (d / 32) * 32;  // 256..384 (step_fast_ok)
  return 384;
}

int step_chunk_T(int d, int n, int h, int fast) {
  int T = kTMax;
  while ((n + 1) * T > kMaxKeys) --T;
  if (!fast) {
    while (T > 1 && (T * (n + 1) * d + 5 * T * h) * 4 > 150 * 1024) --T;
  }
  return T;
}

size_t step_smem_bytes(int d, int n, int h, int T, int NLtot, int fast) {
  const int NT = step_block_threads(d, n, h, fast);
  Layout L = make_layout(d, n, h, T, NT, NLtot, fast);
  return (size_t)(L.total1 > L.total2 ? L.total1 : L.total2);
}

// Allow up to the opt-in maximum minus the kernel's static shared memory.
cudaError_t step_prepare(int fast, size_t optin, size_t* usable) {
  const void* fn = fast ? (const void*)step_kernel<true> : (const void*)step_kernel<false>;
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, fn);
  if (e != cudaSuccess) return e;
  const size_t smem = optin - fa.sharedSizeBytes;
  if (usable) *usable = smem;
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

int step_max_blocks(int fast, int threads, size_t smem, int* out) {
  cudaError_t e = fast ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, step_kernel<true>, threads, smem)
                       : cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, step_kernel<false>, threads, smem);
  return e == cudaSuccess;
}

void launch_step(const StepParams& p, int fused, int fast, cudaStream_t s, int* launches) {
  const int NT = step_block_threads(p.d, p.n, p.h, fast);
  const size_t smem = (size_t)p.smem_bytes;
  void* fn = fast ? (void*)step_kernel<true> : (void*)step_kernel<false>;
  if (fused) {
    int phases = 3;
    void* args[] = {(void*)&p, (void*)&phases};
    cudaLaunchCooperativeKernel(fn, dim3(p.P), dim3(NT), args, smem, s);
    *launches += 1;
  } else {
    int ph1 = 1, ph2 = 2;
    void* a1[] = {(void*)&p, (void*)&ph1};
    void* a2[] = {(void*)&p, (void*)&ph2};
    cudaLaunchKernel(fn, dim3(p.P), dim3(NT), a1, smem, s);
    cudaLaunchKernel(fn, dim3(p.P), dim3(NT), a2, smem, s);
    *launches += 2;
  }
}

}  // namespace pg
