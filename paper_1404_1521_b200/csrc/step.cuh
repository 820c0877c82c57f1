// step.cuh -- parameters shared by the host API (api.cu) and the step kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace pg {

constexpr int kTMax = 32;       // examples per chunk
constexpr int kMaxKeys = 256;   // (n+1)*T <= 256 gradient rows per chunk
constexpr int kCapK = 2048;     // phase-2 owner-merge keys per window (sorted fallback)

// Device-resident status / synchronisation block (one per model).  Words that
// all CTAs hit in the same phase live in separate 128 B lines: the barrier
// counter is polled by every CTA, `done` takes one atomic per CTA, and the
// current-step error words are read once per CTA -- sharing a line made those
// accesses serialise at one L2 slice.
struct DevStatus {
  // line 0: current step's error state (phase 1 writes on error; phase 2 reads)
  unsigned long long bad;        // min over (pos << 32 | uint32 value)
  int flags;                     // bit0 bad index
  int pad0[29];
  // lines 1-10: grid barrier -- monotonic arrival counts (never reset), one per
  // grid size: the barrier needs every launch that uses a counter to have the
  // same number of CTAs, and P = min(#SMs, batch) changes with the batch
  alignas(128) unsigned long long bar_arrivals[160];
  // line 2: phase-2 arrival counter (flag-reset protocol)
  alignas(128) unsigned done;
  unsigned pad2[31];
  // line 3: results of the most recent step, sticky state, pg_score check
  alignas(128) unsigned long long last_bad;
  unsigned long long sticky_bad; // min over asynchronous steps since pg_sync
  unsigned long long score_bad;  // pg_score index check
  int last_flags;                // most recent step: bit0 bad index, bit1 non-finite loss
  int sticky_flags;              // OR over asynchronous steps since pg_sync
  int rank_flags;                // data-parallel: OR over all ranks
  int score_flags;
  float last_loss;
  int pad3[21];
};
static_assert(sizeof(DevStatus) == 3 * 128 + 160 * 8, "DevStatus layout");

// Shared-memory carve-up (byte offsets), computed once on the host.
// phase-2 dW1 GEMM of the tiled path (step.cu dw1_gemm_tiles): RT x CT output
// tiles, EC examples staged per pass, 4 x 8 register micro-tiles, the 384
// threads split into kGNS example ranges
#ifndef PG_G_RT
#define PG_G_RT 16
#endif
#ifndef PG_G_CT
#define PG_G_CT 32
#endif
constexpr int kGRT = PG_G_RT, kGCT = PG_G_CT, kGEC = 128, kGBUF = 4;   // EC examples per pass, kGBUF passes in flight (TMA)
constexpr int kGMT = (kGRT / 4) * (kGCT / 8), kGNS = 384 / kGMT;
static_assert(kGNS * kGRT * kGCT <= kGBUF * kGEC * 2 * (kGRT + kGCT), "split sums fit the pass buffers");

struct Layout {
  // phase 1
  int xs, pg, sig, gz, hinge, rows, ws, red, wsm;
  int ahk, ahc, aslot, ocnt, ocur, hj, ecnt, eoff, ecur, spos, misc, amask, pu, urow, uslot;   // chunk aggregation
  int A, Ac, SIG, DEL, DELc;   // generic path
  int xt, sigu, sige, dwt;      // tiled path
  // phase 2
  int lbase, loff, keys, seg, stage, stagefb, carry, dred, ws2;
  int esrc, erow, hkey, hfirst, heads, hlist, rcnt, roff, rcur, misc2, rmask;
  int lpart;     // long-row segment partials [NSEG][d] (owner merge)
  int NSEG;      // worst-case segment count: every long row always splits
  int SB;        // staged rows per sub-batch (sorted fallback)
  int MCAP;      // owner entries handled by the hash fast path
  int HS;        // hash slots (power of two >= 2*MCAP)
  int total1, total2;
};

__host__ __device__ inline int align16(int x) { return (x + 15) & ~15; }

__host__ __device__ inline Layout make_layout(int d, int n, int h, int T, int NT, int NLtot, int fast) {
  Layout L{};
  int o = 32;
  const int NW = NT / 32;
  if (fast == 1) {
    L.xs = o;    o = align16(o + NW * T * 32 * 4);
    L.pg = o;    o = align16(o + NW * T * 32 * 4);     // == T*(n+1)*d floats
    const int sigf = 3 * T * 32 > (d / 32) * 32 * 33 ? 3 * T * 32 : (d / 32) * 32 * 33;
    L.sig = o;   o = align16(o + sigf * 4);
    L.wsm = o;   o = align16(o + NW * 32 * 33 * 4);    // per-warp W1 transpose tile (padded)
  } else if (fast == 2) {   // tiled path (h % 32 == 0, 64 <= h <= 128)
    const int K = (n + 1) * T;
    int a = K * d;                                     // deduped rows, then part [E][T][h], then G [T][E][d]
    if ((n + 1) * T * h > a) a = (n + 1) * T * h;
    L.xs = o;    o = align16(o + a * 4);
    L.pg = L.xs;
    L.xt = o;    o = align16(o + (n + 1) * d * (T + 4) * 4);   // X transposed [E][d][T + 4 pad]
    L.sigu = o;  o = align16(o + 3 * h * (T + 4) * 4);    // sigma|delta|delta' [3][h][T + 4 pad]
    L.sige = o;  o = align16(o + 3 * T * h * 4);          // the same as [3][T][h]
    L.dwt = o;   o = align16(o + T * h * 4);              // dw2 terms [T][h]
  } else {
    L.xs = o;    o = align16(o + T * (n + 1) * d * 4); // X, later G rows
    L.pg = L.xs;
    L.A = o;     o = align16(o + T * h * 4);
    L.Ac = o;    o = align16(o + T * h * 4);
    L.SIG = o;   o = align16(o + T * h * 4);
    L.DEL = o;   o = align16(o + T * h * 4);
    L.DELc = o;  o = align16(o + T * h * 4);
  }
  L.gz = o;    o = align16(o + kTMax * 4);
  L.hinge = o; o = align16(o + kTMax * 4);
  L.rows = o;  o = align16(o + kMaxKeys * 4);
  L.ahk = o;   o = align16(o + 2 * kMaxKeys * 4);
  L.aslot = o; o = align16(o + kMaxKeys * 4);
  L.ocnt = o;  o = align16(o + 256 * 4);
  L.ocur = o;  o = align16(o + 256 * 4);
  L.ahc = o;   o = align16(o + 2 * kMaxKeys * 4);
  L.hj = o;    o = align16(o + 2 * kMaxKeys * 4);
  L.ecnt = o;  o = align16(o + kMaxKeys * 4);
  L.eoff = o;  o = align16(o + (kMaxKeys + 1) * 4);
  L.ecur = o;  o = align16(o + kMaxKeys * 4);
  L.spos = o;  o = align16(o + kMaxKeys * 2);
  L.misc = o;  o = align16(o + 16 * 4);
  L.amask = o; o = align16(o + 2 * kMaxKeys * (kMaxKeys / 32) * 4);   // per hash slot: member positions
  L.pu = o;    o = align16(o + kMaxKeys * 4);     // position -> distinct row index
  L.urow = o;  o = align16(o + kMaxKeys * 4);     // distinct row index -> row
  L.uslot = o; o = align16(o + kMaxKeys * 4);     // distinct row index -> hash slot
  L.ws = o;    o = align16(o + 64 * 4);
  L.red = o;   o = align16(o + 2 * 32 * 32 * 4);
  L.total1 = o;
  // phase 2 (aliases phase 1 storage); the per-list tables (sized by the
  // list count) go last, so every other offset depends on the shape only
  // and a shape-specialised kernel can fold them (step_kernel PATH 5)
  o = 32;
  L.ws2 = o;   o = align16(o + 64 * 4);
  L.dred = o;  o = align16(o + NT * 16);
  const int p2fixed = o;
  // hash fast path
  int MCAP = (160 * 1024) / (d * 4 + 32);
  if (MCAP > 512) MCAP = 512;
  int HS = 1;
  while (HS < 2 * MCAP) HS <<= 1;
  L.MCAP = MCAP;
  L.HS = HS;
  L.esrc = o;   o = align16(o + MCAP * 4);
  L.erow = o;   o = align16(o + MCAP * 4);
  L.heads = o;  o = align16(o + (MCAP + 1) * 4);
  L.hlist = o;  o = align16(o + MCAP * 2);        // entries sorted by (row, list) (uint16)
  L.rcnt = o;   o = align16(o + MCAP * 4);
  L.roff = o;   o = align16(o + (MCAP + 1) * 4);
  L.rcur = o;   o = align16(o + (MCAP + 1) * 4);   // [MCAP] holds the distinct-row counter
  L.misc2 = o;  o = align16(o + HS * 4);          // hash slot -> distinct row index
  L.hkey = o;   o = align16(o + HS * 4);
  L.hfirst = o; o = align16(o + HS * 4);
  L.stage = o;  o = align16(o + MCAP * d * 4);
  L.rmask = o;  o = align16(o + MCAP * (512 / 32) * 4);   // per distinct row: member entries
  // long rows (> 32 entries) are summed in 32-entry segments: at most
  // ceil(MCAP/32) full segments plus one partial segment per long row, so the
  // split decision never depends on which row claimed capacity first
  L.NSEG = (MCAP + 31) / 32 + MCAP / 33 + 1;
  L.lpart = o;  o = align16(o + L.NSEG * d * 4);
  const int fast_end = o;
  // sorted fallback (aliases the hash path)
  o = p2fixed;
  L.keys = o;  o = align16(o + kCapK * 8);
  L.seg = o;   o = align16(o + (kCapK + 1) * 4);
  int SB = 131072 / (d * 4);   // fallback window: 512 entries at d = 64
  if (SB > 512) SB = 512;
  if (SB < 16) SB = 16;
  L.SB = SB;
  L.stagefb = o; o = align16(o + SB * d * 4);
  L.carry = o; o = align16(o + 2 * 4 * d * 4);   // [2][4 chains][d]
  o = o > fast_end ? o : fast_end;
  if (fast == 2) {   // the phase-2 dW1 GEMM staging (step.cu dw1_gemm_tiles)
    const int gemm = kGBUF * kGEC * 2 * (kGRT + kGCT) * 4 + 256;   // pass buffers (the split sums alias them) + mbarriers, 128 B alignment
    o = o > gemm ? o : gemm;
  }
  L.lbase = o; o = align16(o + (NLtot + 1) * 4);
  L.loff = o;  o = align16(o + (NLtot + 1) * 4);
  L.total2 = o;
  return L;
}

// Data-parallel exchange window of one rank (byte offsets; SURVEY.md §8(e),
// §8(f) NEXT-4).  Each rank publishes, per owner CTA q, the rows it owns
// (row % P == q) merged over its own lists -- one (row, gradient-sum) entry per
// distinct row -- plus its dense-gradient sum, hinge sum and error flags; the
// ranks' owner-q CTAs then merge the G records in rank order.
constexpr int kMaxRanks = 64;
constexpr unsigned kOffBits = 26;                 // ranked entry code: rank << 26 | offset
constexpr unsigned kOffMask = (1u << kOffBits) - 1u;
struct XHdr {
  int flags;     // the rank's error flags (bit0 bad index)
  float hinge;   // the rank's hinge sum (record order)
  int base;      // first entry of owner q in the rank's rows/vals
  int count;     // entries of owner q
};
struct XLayout {
  size_t flags;      // [kMaxRanks][kMaxSMs] u32: step epoch at which rank r's CTA q published
  size_t blk[2];     // per parity: [hdr kMaxSMs x XHdr | rows cap | vals cap x d]
  size_t blk_bytes;
  size_t rows, vals; // offsets inside a block
  size_t dense[2];   // per parity: the rank's dense-gradient sum [dense_stride]
  size_t total;
};

// Where the (row, gradient) entries of a list live.  Local lists (one GPU,
// the per-chunk lists of phase 1): entry code L * list_stride + off.  Ranked
// records (data-parallel merge): list L is rank L's owner-q region, code
// (L << kOffBits) | off, rank L's arrays xstride bytes after rank L-1's.
struct Lists {
  const int32_t* rows;
  const float* vals;
  int list_stride;
  size_t xstride;   // 0: local lists
  __device__ __forceinline__ unsigned code(int L, int off) const {
    return xstride ? ((unsigned)L << kOffBits) | (unsigned)off : (unsigned)(L * list_stride + off);
  }
  __device__ __forceinline__ const int32_t* row(unsigned c) const {
    return xstride ? reinterpret_cast<const int32_t*>(reinterpret_cast<const char*>(rows) + (size_t)(c >> kOffBits) * xstride) +
                         (c & kOffMask)
                   : rows + c;
  }
  __device__ __forceinline__ const float* val(unsigned c, int d) const {
    return xstride ? reinterpret_cast<const float*>(reinterpret_cast<const char*>(vals) + (size_t)(c >> kOffBits) * xstride) +
                         (size_t)(c & kOffMask) * d
                   : vals + (size_t)c * d;
  }
};

// Fixed per-step decomposition: P CTAs, CTA p
// owns examples [p*B/P, (p+1)*B/P), processed in R chunks of <= T examples.
// Chunk (p, r) is list L = p*R + r.
struct StepParams {
  // parameters
  float* C;
  float* W1;
  float* W1T;        // tiled path: W1 transposed [h][n*d], kept in step by the dense update (else null)
  // tiled path, small per-CTA batches (one GPU): dW1 as an output-tiled GEMM in
  // phase 2 over the batch's inputs and deltas instead of per-CTA records
  int dw1_gemm;
  float* xg;         // [B][n+1][d]: example inputs per slot, slot n = corrupt centre
  float* sg;         // [B][3][h]: sigma | delta | delta' per hidden unit
  const void* tmap;  // two CUtensorMaps (128 B each, device memory): xg as (d, n+1, B), sg as (h, 3, B)
  float* b1;
  float* w2;
  const float* b2;
  int64_t V;
  int d, n, h;
  // batch (this rank's shard)
  const int32_t* idx;
  const int32_t* corr;
  int B;
  float inv_B;   // 1 / global batch (or 1: summed loss)
  int act;       // 0 hardtanh, 1 tanh (PG_OPT_ACTIVATION)
  float lr;
  // decomposition
  int P, R, T, cap;     // cap = (n+1)*T list capacity
  // workspace: per-CTA dense partial records
  float* dense_part;    // [P][dense_stride]: dW1 | db1 | dw2 | hinge | flags
  int dense_len;        // n*d*h + 2h
  int dense_stride;     // multiple of 4, > dense_len + 1
  // per-chunk aggregated (row, gradient-sum) lists, bucketed by owner CTA
  int32_t* list_rows;   // [NL][cap]
  float* list_vals;     // [NL][cap][d]
  int32_t* list_off;    // [NL][P+1]  (owner q's entries: [off[q], off[q+1]))
  int NL;               // P * R
  DevStatus* st;
  float* loss_out;      // optional device pointer
  int mode;             // 0 det, 1 atomic
  int smem_bytes;       // dynamic smem requested
  unsigned long long* trace;  // optional [P][64] %globaltimer stamps (PG_OPT_TRACE)
  // ---- data parallel (phase bits 8: publish, 16: merge)
  int world, rank;
  unsigned char* xwin;        // this rank's exchange window
  const unsigned char* xbase; // rank 0's window (or gathered block) as addressed by this rank
  size_t xstride;             // bytes from rank r's window (block) to rank r + 1's
  XLayout xl;
  int xcap;                   // entries per rank record, (n+1)*B
  int xpeer;                  // 1: publish pushes ready epochs to every rank's window, merge waits
  int xgathered;              // 1: records were all-gathered into xbase (parity 0, blocks back to back)
  unsigned* xepoch;           // [P] per-CTA step counters (this rank)
  const float* xdense;        // all-reduced dense vector | hinge | flags (NCCL exchanges), else null
  unsigned long long* xstats; // [0] bytes read from other ranks' records, [1] max entries merged by one owner
  Layout lay;
};

void launch_step(const StepParams& p, int fused, int fast, cudaStream_t s, int* launches);
// phases: 1 phase 1, 2 phase 2 (one GPU), 8 data-parallel publish, 16 data-
// parallel merge; 1 together with 2 or 8 adds the in-rank grid barrier
void launch_step_phases(const StepParams& p, int phases, int fast, cudaStream_t s, int* launches);
// NCCL table exchange: what = 0 scatter this rank's merged rows into `table`,
// 1 apply the reduced table and dense vector, 2 apply and re-zero the table
void launch_dp_table(const StepParams& p, float* table, int what, int num_sms, cudaStream_t s, int* launches);
int step_fast_ok(int d, int n, int h);
int step_block_threads(int d, int n, int h, int fast);
int step_chunk_T(int d, int n, int h, int fast, int per_cta);   // per_cta = ceil(B / P)
int step_dw1_gemm(int fast, int T);   // 1: the tiled path takes dW1 as a phase-2 GEMM (small chunks)
cudaError_t step_prepare(int fast, size_t optin, size_t* usable);

}  // namespace pg
