// api.cu -- host implementation of the C ABI declared in include/pg.h.
//
// Owns device memory, the model stream, lazily sized per-batch workspace and
// the launches of the sm_100a kernels (step.cu, scatter.cu, and the init and
// score kernels below).  No torch types cross this boundary.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdlib>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pg.h"
#include "common.cuh"
#include "nccl_shim.h"
#include "scatter.cuh"
#include "step.cuh"

using namespace pg;

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;

static pg_status fail(pg_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define CU(call)                                                                       \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(e_ == cudaErrorMemoryAllocation ? PG_ENOMEM : PG_ECUDA, "%s: %s (%s:%d)", \
                  #call, cudaGetErrorString(e_), __FILE__, __LINE__);                   \
  } while (0)

extern "C" const char* pg_last_error(void) { return g_err.c_str(); }
extern "C" int pg_abi_version(void) { return PG_ABI_VERSION; }

// ------------------------------------------------------------------ model
struct pg_model {
  int device = 0, num_sms = 0;
  int64_t V = 0;
  int d = 0, n = 0, h = 0;
  float *C = nullptr, *W1 = nullptr, *b1 = nullptr, *w2 = nullptr, *b2 = nullptr;
  float* W1T = nullptr;   // tiled path: W1 transposed [h][n*d]
  float* xg = nullptr;    // tiled path, small chunks: [B][n+1][d] inputs for the phase-2 dW1 GEMM
  float* sg = nullptr;    //   and [B][3][h] deltas
  int64_t cap_xg = 0;     //   examples they hold
  void* d_tmap = nullptr; //   TMA tensor maps over xg / sg for the dW1 GEMM (2 x 128 B)
  int tmap_B = 0;         //   the batch they were encoded for
  DevStatus* st = nullptr;
  DevStatus* st_host = nullptr;  // pinned mirror for blocking reads
  cudaStream_t stream = nullptr;
  int mode = PG_SCATTER_DET, fused = 1, fast = 0;
  int act = PG_ACT_HARDTANH;
  int reduce_sum = 0;   // PG_OPT_REDUCTION
  size_t smem_max = 0;
  unsigned long long* trace = nullptr;
  // per-batch workspace (capacity grows)
  int64_t cap_lists = 0, cap_dense = 0, cap_off = 0, cap_in = 0;
  float* dense_part = nullptr;
  int32_t* list_rows = nullptr;
  float* list_vals = nullptr;
  int32_t* list_off = nullptr;
  // host-input staging, double-buffered: host idx/corr are copied on copy_stream
  // into slot k % 2 while the previous step runs; ev_consumed[s] marks the end of
  // the launch that read slot s, ev_copied[s] orders the step after its copy
  int32_t* d_idx2[2] = {nullptr, nullptr};
  int32_t* d_corr2[2] = {nullptr, nullptr};
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_consumed[2] = {nullptr, nullptr};
  int in_slot = 0, pending_slot = -1;
  float* d_scores = nullptr;
  int64_t launches = 0;
  // data parallel (pg_attach_nccl): exchange window and NCCL buffers, sized
  // for batch x_B
  int rank = 0, world = 1;
  void* comm = nullptr;
  int xmode = PG_EXCHANGE_AUTO;   // requested (PG_OPT_EXCHANGE)
  int xchosen = -1;               // in use for x_B
  int x_B = 0;
  XLayout xl{};
  unsigned char* xwin = nullptr;  // this rank's window (ncclMemAlloc'd + registered for PEER)
  void* xwin_handle = nullptr;    // ncclWindow_t of the registration (PEER), else null
  bool xwin_nccl = false;         // xwin came from ncclMemAlloc
  unsigned char* xbase = nullptr; // rank 0's window in this rank's address space (PEER)
  size_t xstride = 0;
  unsigned char* xrecv = nullptr; // ALLGATHER: [world][blk_bytes]
  float* xdense = nullptr;        // ALLGATHER / TABLE: all-reduced [dense_stride]
  float* xtable = nullptr;        // TABLE: [V][d] gradient table (kept zero between steps)
  unsigned* xepoch = nullptr;     // [kMaxSMs] per-CTA step counters
  unsigned long long* xstats = nullptr;   // [2] exchange statistics (pg_exchange_info)
  int64_t x_launch_bytes = 0;     // NCCL exchanges: bytes received per step (host-computed)
  int64_t x_steps = 0;            // NCCL-exchange steps since the last pg_exchange_info reset
};

// ------------------------------------------------------------------ init kernel
// Reading G10 / pg.h: value = float((2u - 1) r), u = top 24 bits of output i of
// the SplitMix64 stream keyed by seed ^ (0x632BE59BD9B4E019 * (tensor_id + 1)).
__global__ void init_uniform_kernel(float* out, int64_t count, unsigned long long seed,
                                    unsigned long long tensor_id, double r) {
  const unsigned long long key = seed ^ (0x632BE59BD9B4E019ull * (tensor_id + 1ull));
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    unsigned long long z = key + (unsigned long long)(i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z = z ^ (z >> 31);
    const double u = (double)(z >> 40) * (1.0 / 16777216.0);
    out[i] = __double2float_rn(__dmul_rn(__dadd_rn(__dmul_rn(2.0, u), -1.0), r));
  }
}

// ------------------------------------------------------------------ score kernel
// W1T[u][r] = W1[r][u] (the tiled step path reads W1 rows along u as columns).
__global__ void transpose_w1_kernel(const float* __restrict__ W1, float* __restrict__ W1T, int rows, int h) {
  const int64_t total = (int64_t)rows * h;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int u = (int)(i / rows), r = (int)(i % rows);
    W1T[i] = W1[(size_t)r * h + u];
  }
}

// Warp per window: s = w2 . f(W1^T x + b1) + b2, f = hardtanh or tanh.
__global__ void score_kernel(const float* __restrict__ C, const float* __restrict__ W1,
                             const float* __restrict__ b1, const float* __restrict__ w2,
                             const float* __restrict__ b2, int64_t V, int d, int n, int h,
                             const int32_t* __restrict__ idx, int B, float* out, DevStatus* st, int act) {
  extern __shared__ float xsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nd = n * d;
  float* x = xsm + (size_t)warp * nd;
  for (int64_t e = (int64_t)blockIdx.x * nw + warp; e < B; e += (int64_t)gridDim.x * nw) {
    bool bad = false;
    for (int i = lane; i < nd; i += 32) {
      const int p = i / d, j = i % d;
      const int row = __ldg(idx + e * n + p);
      const bool ok = row >= 0 && (int64_t)row < V;
      if (!ok && j == 0) {
        atomicMin(&st->score_bad, ((unsigned long long)(e * n + p) << 32) | (unsigned)row);
        atomicOr(&st->score_flags, 1);
      }
      bad |= !ok;
      x[i] = ok ? __ldg(C + (size_t)row * d + j) : 0.f;
    }
    __syncwarp();
    float sp = 0.f;
    for (int u = lane; u < h; u += 32) {
      float a = __ldg(b1 + u);
      for (int i = 0; i < nd; ++i) a = fmaf(x[i], __ldg(W1 + (size_t)i * h + u), a);
      sp += __ldg(w2 + u) * act_f(a, act);
    }
    const float s = warp_sum(sp) + __ldg(b2);
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) out[e] = bad ? __int_as_float(0x7fc00000) : s;
    __syncwarp();
  }
}

// ------------------------------------------------------------------ helpers
enum PtrKind { PTR_NULL, PTR_HOST, PTR_DEVICE };

// dev (optional): the device-side address of a page-locked host pointer (NULL
// for pageable memory) -- the kernels can write such memory directly.
static PtrKind ptr_kind(const void* p, void** dev = nullptr) {
  if (dev) *dev = nullptr;
  if (!p) return PTR_NULL;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return PTR_HOST;
  }
  if (a.type == cudaMemoryTypeHost && dev) *dev = a.devicePointer;
  return (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) ? PTR_DEVICE : PTR_HOST;
}

// Exchange buffers (data parallel); the window is collective for PEER.
static void free_dp(pg_model* m) {
  if (m->xwin_handle && m->comm) nccl_shim_window_deregister(m->comm, m->xwin_handle);
  if (m->xwin_nccl) nccl_shim_mem_free(m->xwin);
  else cudaFree(m->xwin);
  cudaFree(m->xrecv); cudaFree(m->xdense); cudaFree(m->xtable);
  m->xwin = m->xrecv = nullptr;
  m->xdense = m->xtable = nullptr;
  m->xwin_handle = nullptr;
  m->xwin_nccl = false;
  m->xbase = nullptr;
  m->xstride = 0;
  m->x_B = 0;
  m->xchosen = -1;
}

// Group emulation buffers, owned by replica 0 of a group (keyed by world, B).
struct GroupX {
  int world = 0, B = 0, mode = -1;
  unsigned char* win = nullptr;    // [world][xl.total]
  unsigned char* recv = nullptr;   // ALLGATHER: [world][blk_bytes]
  float* dense = nullptr;          // ALLGATHER / TABLE: reduced dense
  float* table = nullptr;          // TABLE
  std::vector<unsigned*> epochs;   // per replica
};
static std::mutex g_group_mu;
static std::vector<std::pair<pg_model*, GroupX>> g_groups;

static void free_group(GroupX& gx) {
  cudaFree(gx.win); cudaFree(gx.recv); cudaFree(gx.dense); cudaFree(gx.table);
  gx = GroupX{};
}

static void free_ws(pg_model* m) {
  cudaFree(m->dense_part); cudaFree(m->list_rows); cudaFree(m->list_vals); cudaFree(m->list_off);
  m->dense_part = nullptr; m->list_rows = nullptr; m->list_vals = nullptr; m->list_off = nullptr;
  m->cap_lists = m->cap_dense = m->cap_off = 0;
}

struct Geometry {
  int P, R, T, cap, NL, dense_len, dense_stride;
  int dw1_gemm;   // tiled path with small chunks (one GPU): dW1 as a phase-2 GEMM
  size_t smem;
  Layout lay;
};

static Geometry geometry(const pg_model* m, int B, int world = 1) {
  Geometry g{};
  // PG_STEP_CTAS caps the CTAs per step (experiments; default: one per SM)
  static const int cap = getenv("PG_STEP_CTAS") ? atoi(getenv("PG_STEP_CTAS")) : 0;
  const int P = cap > 0 && cap < m->num_sms ? cap : m->num_sms;
  g.P = B < P ? B : P;
  const int per = (B + g.P - 1) / g.P;
  g.T = step_chunk_T(m->d, m->n, m->h, m->fast, per);
  g.R = (per + g.T - 1) / g.T;
  g.cap = (m->n + 1) * g.T;
  g.NL = g.P * g.R;
  g.dense_len = m->n * m->d * m->h + 2 * m->h;
  g.dw1_gemm = world == 1 && step_dw1_gemm(m->fast, g.T);
  g.dense_stride = ((g.dense_len + 2) + 3) & ~3;   // dense | hinge | flags
  g.lay = make_layout(m->d, m->n, m->h, g.T, step_block_threads(m->d, m->n, m->h, m->fast),
                      g.NL > world ? g.NL : world, m->fast);
  g.smem = (size_t)(g.lay.total1 > g.lay.total2 ? g.lay.total1 : g.lay.total2);
  return g;
}

// TMA tensor maps of the dW1 GEMM operands (step.cu dw1_gemm_tiles): xg as a
// 3-D tensor (d, n+1, B) with boxes (kGRT, 1, kGEC), sg as (h, 3, B) with boxes
// (kGCT, 1, kGEC); fp32, no swizzle, out-of-range examples read as zeros.  The
// driver's encoder is reached through the runtime (no -lcuda).
static pg_status encode_tmaps(pg_model* m, int B) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return fail(PG_ECUDA, "cuTensorMapEncodeTiled is not available");
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  alignas(64) CUtensorMap maps[2];
  const cuuint32_t one[3] = {1, 1, 1};
  {
    const cuuint64_t dim[3] = {(cuuint64_t)m->d, (cuuint64_t)(m->n + 1), (cuuint64_t)B};
    const cuuint64_t stride[2] = {sizeof(float) * (cuuint64_t)m->d, sizeof(float) * (cuuint64_t)m->d * (m->n + 1)};
    const cuuint32_t box[3] = {(cuuint32_t)kGRT, 1, (cuuint32_t)kGEC};
    if (enc(&maps[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, m->xg, dim, stride, box, one, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return fail(PG_ECUDA, "tensor map of the GEMM inputs could not be encoded");
  }
  {
    const cuuint64_t dim[3] = {(cuuint64_t)m->h, 3, (cuuint64_t)B};
    const cuuint64_t stride[2] = {sizeof(float) * (cuuint64_t)m->h, sizeof(float) * (cuuint64_t)m->h * 3};
    const cuuint32_t box[3] = {(cuuint32_t)kGCT, 1, (cuuint32_t)kGEC};
    if (enc(&maps[1], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, m->sg, dim, stride, box, one, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return fail(PG_ECUDA, "tensor map of the GEMM deltas could not be encoded");
  }
  if (!m->d_tmap) CU(cudaMalloc(&m->d_tmap, sizeof(maps)));
  // ordered on the model stream before the next step; the source is copied
  // out before cudaMemcpyAsync returns (pageable memory)
  CU(cudaMemcpyAsync(m->d_tmap, maps, sizeof(maps), cudaMemcpyHostToDevice, m->stream));
  m->tmap_B = B;
  return PG_OK;
}

static pg_status ensure_ws(pg_model* m, int B, int world = 1) {
  Geometry g = geometry(m, B, world);
  if (g.smem > m->smem_max)
    return fail(PG_EINVAL, "batch %d needs %zu B of shared memory per CTA (max %zu)", B, g.smem, m->smem_max);
  const int64_t lists = (int64_t)g.NL;
  const int64_t dense = (int64_t)g.P * g.dense_stride;
  const int64_t off = lists * (g.P + 1);
  if (lists * g.cap > m->cap_lists || dense > m->cap_dense || off > m->cap_off) {
    CU(cudaStreamSynchronize(m->stream));
    free_ws(m);
    const int64_t L = lists * g.cap;
    CU(cudaMalloc(&m->dense_part, sizeof(float) * dense));
    CU(cudaMalloc(&m->list_rows, sizeof(int32_t) * L));
    CU(cudaMalloc(&m->list_vals, sizeof(float) * L * m->d));
    CU(cudaMalloc(&m->list_off, sizeof(int32_t) * off));
    m->cap_lists = L; m->cap_dense = dense; m->cap_off = off;
  }
  if (g.dw1_gemm && B > m->cap_xg) {
    CU(cudaStreamSynchronize(m->stream));
    cudaFree(m->xg); cudaFree(m->sg);
    m->xg = m->sg = nullptr;
    CU(cudaMalloc(&m->xg, sizeof(float) * (size_t)(m->n + 1) * m->d * B));
    CU(cudaMalloc(&m->sg, sizeof(float) * (size_t)3 * m->h * B));
    m->cap_xg = B;
    m->tmap_B = 0;
  }
  if (g.dw1_gemm && B != m->tmap_B) {   // (re-)encode the tensor maps for this batch
    if (pg_status s = encode_tmaps(m, B)) return s;
  }
  if (B > m->cap_in) {
    CU(cudaStreamSynchronize(m->stream));
    if (m->copy_stream) CU(cudaStreamSynchronize(m->copy_stream));
    for (int k = 0; k < 2; ++k) {
      cudaFree(m->d_idx2[k]); cudaFree(m->d_corr2[k]);
      CU(cudaMalloc(&m->d_idx2[k], sizeof(int32_t) * (size_t)B * m->n));
      CU(cudaMalloc(&m->d_corr2[k], sizeof(int32_t) * (size_t)B));
    }
    cudaFree(m->d_scores);
    CU(cudaMalloc(&m->d_scores, sizeof(float) * (size_t)B));
    m->cap_in = B;
  }
  return PG_OK;
}

static pg_status check_model(const pg_model* m) {
  if (!m) return fail(PG_EINVAL, "null model handle");
  return PG_OK;
}

static pg_status set_device(const pg_model* m) {
  CU(cudaSetDevice(m->device));
  return PG_OK;
}

static pg_status status_from_flags(int flags, unsigned long long bad, const char* what) {
  if ((flags & 1) && bad == kNoBad)
    return fail(PG_ERANGE, "%s: index out of range on another rank; no parameter was modified", what);
  if (flags & 1) {
    const long long pos = (long long)(bad >> 32);
    const int val = (int)(unsigned)(bad & 0xffffffffull);
    return fail(PG_ERANGE, "%s: index out of range at flat position %lld (value %d); no parameter was modified",
                what, pos, val);
  }
  if (flags & 4) return fail(PG_ENCCL, "%s: a data-parallel rank did not publish its gradients in time; no parameter was modified", what);
  if (flags & 2) return fail(PG_EDIVERGED, "%s: non-finite loss; no parameter was modified", what);
  return PG_OK;
}

// ------------------------------------------------------------------ C ABI
extern "C" pg_status pg_init(pg_model** out, int64_t vocab, int32_t dim, int32_t window, int32_t hidden,
                             uint64_t seed) {
  if (!out) return fail(PG_EINVAL, "pg_init: out is NULL");
  *out = nullptr;
  if (vocab < 2 || vocab > 2147483647LL) return fail(PG_EINVAL, "pg_init: vocab must be in [2, 2^31-1]");
  if (dim < 1 || window < 1 || hidden < 1) return fail(PG_EINVAL, "pg_init: dim, window, hidden must be >= 1");
  if (hidden > 1024 || window > 63 || dim > 4096)
    return fail(PG_EINVAL, "pg_init: unsupported shape (hidden <= 1024, window <= 63, dim <= 4096)");
  pg_model* m = new pg_model();
  m->V = vocab; m->d = dim; m->n = window; m->h = hidden;
  cudaError_t e = cudaGetDevice(&m->device);
  if (e != cudaSuccess) { delete m; return fail(PG_ECUDA, "pg_init: no CUDA device: %s", cudaGetErrorString(e)); }
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, m->device);
  if (prop.major < 10) {
    delete m;
    return fail(PG_ECUDA, "pg_init: libpg is built for sm_100a; device is sm_%d%d", prop.major, prop.minor);
  }
  m->num_sms = prop.multiProcessorCount < kMaxSMs ? prop.multiProcessorCount : kMaxSMs;
  m->fast = step_fast_ok(dim, window, hidden);
  if (!m->fast && (hidden > 128))
    { delete m; return fail(PG_EINVAL, "pg_init: generic path supports hidden <= 128"); }
  const int64_t nC = vocab * dim, nW = (int64_t)window * dim * hidden;
  pg_status s = PG_OK;
  auto bail = [&](pg_status st) { pg_free(m); return st; };
  if (cudaMalloc(&m->C, sizeof(float) * nC) != cudaSuccess ||
      cudaMalloc(&m->W1, sizeof(float) * nW) != cudaSuccess ||
      cudaMalloc(&m->b1, sizeof(float) * hidden) != cudaSuccess ||
      cudaMalloc(&m->w2, sizeof(float) * hidden) != cudaSuccess ||
      cudaMalloc(&m->b2, sizeof(float)) != cudaSuccess ||
      cudaMalloc(&m->st, sizeof(DevStatus)) != cudaSuccess ||
      cudaMallocHost(&m->st_host, sizeof(DevStatus)) != cudaSuccess) {
    cudaGetLastError();
    return bail(fail(PG_ENOMEM, "pg_init: allocation failed (vocab %lld x dim %d)", (long long)vocab, dim));
  }
  const int blocks = m->num_sms * 8;
  init_uniform_kernel<<<blocks, 256>>>(m->C, nC, seed, 0, 0.5);
  init_uniform_kernel<<<blocks, 256>>>(m->W1, nW, seed, 1, 0.5 / (double)(window * dim));
  init_uniform_kernel<<<1, 256>>>(m->w2, hidden, seed, 2, 0.5 / (double)hidden);
  m->launches += 3;
  if (m->fast == 2) {
    if (cudaMalloc(&m->W1T, sizeof(float) * nW) != cudaSuccess) {
      cudaGetLastError();
      return bail(fail(PG_ENOMEM, "pg_init: allocation failed (W1T)"));
    }
    transpose_w1_kernel<<<blocks, 256>>>(m->W1, m->W1T, window * dim, hidden);
    m->launches += 1;
  }
  cudaMemset(m->b1, 0, sizeof(float) * hidden);
  cudaMemset(m->b2, 0, sizeof(float));
  DevStatus z{};
  z.bad = z.last_bad = z.sticky_bad = z.score_bad = kNoBad;
  cudaMemcpy(m->st, &z, sizeof z, cudaMemcpyHostToDevice);
  cudaError_t e2 = step_prepare(m->fast, prop.sharedMemPerBlockOptin, &m->smem_max);
  if (e2 == cudaSuccess) e2 = scatter_prepare(1024);
  if (e2 == cudaSuccess) e2 = cudaFuncSetAttribute(score_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (e2 == cudaSuccess) e2 = cudaDeviceSynchronize();
  if (e2 != cudaSuccess) return bail(fail(PG_ECUDA, "pg_init: %s", cudaGetErrorString(e2)));
  *out = m;
  (void)s;
  return PG_OK;
}

extern "C" void pg_free(pg_model* m) {
  if (!m) return;
  cudaSetDevice(m->device);
  if (m->stream) cudaStreamSynchronize(m->stream);
  else cudaDeviceSynchronize();
  free_dp(m);
  if (m->comm) nccl_shim_destroy(m->comm);
  m->comm = nullptr;
  free_ws(m);
  cudaFree(m->xepoch); cudaFree(m->xstats);
  {
    std::lock_guard<std::mutex> lk(g_group_mu);
    for (size_t i = 0; i < g_groups.size(); ++i)
      if (g_groups[i].first == m) { free_group(g_groups[i].second); g_groups.erase(g_groups.begin() + i); break; }
  }
  cudaFree(m->xg); cudaFree(m->sg); cudaFree(m->d_tmap);
  cudaFree(m->C); cudaFree(m->W1); cudaFree(m->W1T); cudaFree(m->b1); cudaFree(m->w2); cudaFree(m->b2);
  cudaFree(m->st); cudaFreeHost(m->st_host);
  if (m->copy_stream) cudaStreamSynchronize(m->copy_stream);
  for (int k = 0; k < 2; ++k) {
    cudaFree(m->d_idx2[k]); cudaFree(m->d_corr2[k]);
    if (m->ev_copied[k]) cudaEventDestroy(m->ev_copied[k]);
    if (m->ev_consumed[k]) cudaEventDestroy(m->ev_consumed[k]);
  }
  if (m->copy_stream) cudaStreamDestroy(m->copy_stream);
  cudaFree(m->d_scores);
  delete m;
}

extern "C" pg_status pg_get_shape(const pg_model* m, int64_t* vocab, int32_t* dim, int32_t* window,
                                  int32_t* hidden) {
  if (pg_status s = check_model(m)) return s;
  if (vocab) *vocab = m->V;
  if (dim) *dim = m->d;
  if (window) *window = m->n;
  if (hidden) *hidden = m->h;
  return PG_OK;
}

static pg_status ensure_dp(pg_model* m, int B);

extern "C" pg_status pg_set_option(pg_model* m, int key, int64_t value) {
  if (pg_status s = check_model(m)) return s;
  switch (key) {
    case PG_OPT_SCATTER:
      if (value != PG_SCATTER_DET && value != PG_SCATTER_ATOMIC)
        return fail(PG_EINVAL, "PG_OPT_SCATTER: unknown mode %lld", (long long)value);
      m->mode = (int)value;
      return PG_OK;
    case PG_OPT_STREAM:
      m->stream = reinterpret_cast<cudaStream_t>(value);
      return PG_OK;
    case PG_OPT_FUSED:
      m->fused = value ? 1 : 0;
      return PG_OK;
    case PG_OPT_ACTIVATION:
      if (value != PG_ACT_HARDTANH && value != PG_ACT_TANH)
        return fail(PG_EINVAL, "PG_OPT_ACTIVATION: unknown nonlinearity %lld", (long long)value);
      m->act = (int)value;
      return PG_OK;
    case PG_OPT_REDUCTION:
      if (value != PG_REDUCE_MEAN && value != PG_REDUCE_SUM)
        return fail(PG_EINVAL, "PG_OPT_REDUCTION: unknown reduction %lld", (long long)value);
      m->reduce_sum = value == PG_REDUCE_SUM;
      return PG_OK;
    case PG_OPT_EXCHANGE:
      if (value < PG_EXCHANGE_AUTO || value > PG_EXCHANGE_TABLE)
        return fail(PG_EINVAL, "PG_OPT_EXCHANGE: unknown exchange %lld", (long long)value);
      if (m->xmode != (int)value) {
        m->xmode = (int)value;
        if (m->x_B) {   // re-chosen (collectively) at the next step
          if (pg_status s = set_device(m)) return s;
          CU(cudaStreamSynchronize(m->stream));
          free_dp(m);
        }
      }
      return PG_OK;
    case PG_OPT_TRACE:   // device buffer of [P][32] u64 stage stamps (libpg_trace.so), 0 = off
      m->trace = reinterpret_cast<unsigned long long*>(value);
      return PG_OK;
    case PG_OPT_RESERVE: {   // pre-size the workspace for a batch
      if (value < 1 || value > (1 << 30)) return fail(PG_EINVAL, "reserve: bad batch");
      if (pg_status s = set_device(m)) return s;
      if (pg_status s = ensure_ws(m, (int)value, m->world)) return s;
      return m->comm ? ensure_dp(m, (int)value) : PG_OK;   // collective after pg_attach_nccl
    }
    default:
      return fail(PG_EINVAL, "pg_set_option: unknown key %d", key);
  }
}

extern "C" int64_t pg_kernel_launches(const pg_model* m) { return m ? m->launches : 0; }

static pg_status copy_param(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s));
  return PG_OK;
}

extern "C" pg_status pg_get_params(pg_model* m, float* C, float* W1, float* b1, float* w2, float* b2) {
  if (pg_status s = check_model(m)) return s;
  if (pg_status s = set_device(m)) return s;
  const size_t nW = (size_t)m->n * m->d * m->h;
  pg_status s = PG_OK;
  if (C && !s) s = copy_param(C, m->C, sizeof(float) * (size_t)m->V * m->d, m->stream);
  if (W1 && !s) s = copy_param(W1, m->W1, sizeof(float) * nW, m->stream);
  if (b1 && !s) s = copy_param(b1, m->b1, sizeof(float) * m->h, m->stream);
  if (w2 && !s) s = copy_param(w2, m->w2, sizeof(float) * m->h, m->stream);
  if (b2 && !s) s = copy_param(b2, m->b2, sizeof(float), m->stream);
  if (s) return s;
  CU(cudaStreamSynchronize(m->stream));
  return PG_OK;
}

extern "C" pg_status pg_set_params(pg_model* m, const float* C, const float* W1, const float* b1,
                                   const float* w2, float b2) {
  if (pg_status s = check_model(m)) return s;
  if (pg_status s = set_device(m)) return s;
  const size_t nW = (size_t)m->n * m->d * m->h;
  pg_status s = PG_OK;
  if (C && !s) s = copy_param(m->C, C, sizeof(float) * (size_t)m->V * m->d, m->stream);
  if (W1 && !s) s = copy_param(m->W1, W1, sizeof(float) * nW, m->stream);
  if (W1 && !s && m->W1T) {
    transpose_w1_kernel<<<m->num_sms * 8, 256, 0, m->stream>>>(m->W1, m->W1T, m->n * m->d, m->h);
    m->launches += 1;
    CU(cudaGetLastError());
  }
  if (b1 && !s) s = copy_param(m->b1, b1, sizeof(float) * m->h, m->stream);
  if (w2 && !s) s = copy_param(m->w2, w2, sizeof(float) * m->h, m->stream);
  if (!std::isnan(b2) && !s) {
    float tmp = b2;
    s = copy_param(m->b2, &tmp, sizeof(float), m->stream);
    if (!s) CU(cudaStreamSynchronize(m->stream));
  }
  if (s) return s;
  CU(cudaStreamSynchronize(m->stream));
  return PG_OK;
}

// Inputs in host memory are copied on the model's copy stream into staging slot
// k % 2, so the copy overlaps the previous step still running on the model
// stream; the step's stream waits for its copy, and consume_inputs() (after the
// launches that read the slot) lets the slot be refilled two calls later.
static pg_status stage_inputs(pg_model* m, const int32_t* idx, const int32_t* corr, int B,
                              const int32_t** d_idx, const int32_t** d_corr) {
  const PtrKind ki = ptr_kind(idx);
  const PtrKind kc = corr ? ptr_kind(corr) : PTR_DEVICE;
  *d_idx = idx;
  if (corr) *d_corr = corr;
  if (ki == PTR_DEVICE && kc == PTR_DEVICE) return PG_OK;
  if (!m->copy_stream) {
    CU(cudaStreamCreateWithFlags(&m->copy_stream, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
      CU(cudaEventCreateWithFlags(&m->ev_copied[k], cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&m->ev_consumed[k], cudaEventDisableTiming));
    }
  }
  const int slot = m->in_slot;
  m->in_slot ^= 1;
  CU(cudaStreamWaitEvent(m->copy_stream, m->ev_consumed[slot], 0));   // no-op before its first record
  if (ki != PTR_DEVICE) {
    CU(cudaMemcpyAsync(m->d_idx2[slot], idx, sizeof(int32_t) * (size_t)B * m->n, cudaMemcpyHostToDevice,
                       m->copy_stream));
    *d_idx = m->d_idx2[slot];
  }
  if (corr && kc != PTR_DEVICE) {
    CU(cudaMemcpyAsync(m->d_corr2[slot], corr, sizeof(int32_t) * (size_t)B, cudaMemcpyHostToDevice,
                       m->copy_stream));
    *d_corr = m->d_corr2[slot];
  }
  CU(cudaEventRecord(m->ev_copied[slot], m->copy_stream));
  CU(cudaStreamWaitEvent(m->stream, m->ev_copied[slot], 0));
  m->pending_slot = slot;
  return PG_OK;
}

static pg_status consume_inputs(pg_model* m) {
  if (m->pending_slot >= 0) {
    CU(cudaEventRecord(m->ev_consumed[m->pending_slot], m->stream));
    m->pending_slot = -1;
  }
  return PG_OK;
}

static pg_status run_step(pg_model* m, const int32_t* idx, const int32_t* corr, int B, float lr,
                          float* loss_dev);

extern "C" pg_status pg_train_step(pg_model* m, const int32_t* idx_batch, const int32_t* corrupt_idx,
                                   int32_t batch, float lr, float* loss_out) {
  if (pg_status s = check_model(m)) return s;
  if (!idx_batch || !corrupt_idx) return fail(PG_EINVAL, "pg_train_step: null index pointer");
  if (batch < 1) return fail(PG_EINVAL, "pg_train_step: empty batch (batch=%d); the loss is undefined", batch);
  if (!std::isfinite(lr) || !(lr > 0.f)) return fail(PG_EINVAL, "pg_train_step: lr must be finite and > 0 (got %g)", lr);
  if (pg_status s = set_device(m)) return s;
  if (pg_status s = ensure_ws(m, batch, m->world)) return s;
  void* pinned = nullptr;   // page-locked host loss_out: the step writes it through its device mapping
  const PtrKind kl = ptr_kind(loss_out, &pinned);
  const int32_t *di = nullptr, *dc = nullptr;
  if (pg_status s = stage_inputs(m, idx_batch, corrupt_idx, batch, &di, &dc)) return s;
  float* loss_dev = kl == PTR_DEVICE ? loss_out : static_cast<float*>(pinned);
  if (pg_status s = run_step(m, di, dc, batch, lr, loss_dev)) return s;
  if (pg_status s = consume_inputs(m)) return s;
  if (kl != PTR_HOST || pinned) return PG_OK;
  CU(cudaMemcpyAsync(m->st_host, m->st, sizeof(DevStatus), cudaMemcpyDeviceToHost, m->stream));
  CU(cudaStreamSynchronize(m->stream));
  *loss_out = m->st_host->last_loss;
  return status_from_flags(m->st_host->last_flags, m->st_host->last_bad, "pg_train_step");
}

extern "C" float pg_train_step_loss(pg_model* m, const int32_t* idx_batch, const int32_t* corrupt_idx,
                                    int32_t batch, float lr) {
  float loss = NAN;
  pg_status s = pg_train_step(m, idx_batch, corrupt_idx, batch, lr, &loss);
  return s == PG_OK ? loss : NAN;
}

extern "C" pg_status pg_score(pg_model* m, const int32_t* idx_batch, int32_t batch, float* scores_out) {
  if (pg_status s = check_model(m)) return s;
  if (!idx_batch || !scores_out) return fail(PG_EINVAL, "pg_score: null pointer");
  if (batch < 1) return fail(PG_EINVAL, "pg_score: empty batch");
  if (pg_status s = set_device(m)) return s;
  if (pg_status s = ensure_ws(m, batch)) return s;
  const int32_t *di = nullptr, *dc = nullptr;
  if (pg_status s = stage_inputs(m, idx_batch, nullptr, batch, &di, &dc)) return s;
  const PtrKind ko = ptr_kind(scores_out);
  float* out = ko == PTR_DEVICE ? scores_out : m->d_scores;
  CU(cudaMemsetAsync(&m->st->score_flags, 0, sizeof(int), m->stream));
  CU(cudaMemsetAsync(&m->st->score_bad, 0xff, sizeof(unsigned long long), m->stream));
  const int warps = 8;
  const size_t sm = sizeof(float) * warps * m->n * m->d;
  if (sm > 200 * 1024) return fail(PG_EINVAL, "pg_score: window*dim too large");
  int blocks = (batch + warps - 1) / warps;
  if (blocks > m->num_sms * 16) blocks = m->num_sms * 16;
  score_kernel<<<blocks, warps * 32, sm, m->stream>>>(m->C, m->W1, m->b1, m->w2, m->b2, m->V, m->d, m->n, m->h,
                                                      di, batch, out, m->st, m->act);
  m->launches += 1;
  CU(cudaGetLastError());
  if (pg_status s = consume_inputs(m)) return s;
  if (ko == PTR_DEVICE) return PG_OK;
  CU(cudaMemcpyAsync(scores_out, out, sizeof(float) * batch, cudaMemcpyDeviceToHost, m->stream));
  CU(cudaMemcpyAsync(m->st_host, m->st, sizeof(DevStatus), cudaMemcpyDeviceToHost, m->stream));
  CU(cudaStreamSynchronize(m->stream));
  return status_from_flags(m->st_host->score_flags & 1, m->st_host->score_bad, "pg_score");
}

extern "C" pg_status pg_sync(pg_model* m) {
  if (pg_status s = check_model(m)) return s;
  if (pg_status s = set_device(m)) return s;
  CU(cudaMemcpyAsync(m->st_host, m->st, sizeof(DevStatus), cudaMemcpyDeviceToHost, m->stream));
  CU(cudaStreamSynchronize(m->stream));
  const int flags = m->st_host->sticky_flags;
  const unsigned long long bad = m->st_host->sticky_bad;
  if (flags) {
    CU(cudaMemsetAsync(&m->st->sticky_flags, 0, sizeof(int), m->stream));
    CU(cudaMemsetAsync(&m->st->sticky_bad, 0xff, sizeof(unsigned long long), m->stream));
    CU(cudaStreamSynchronize(m->stream));
  }
  return status_from_flags(flags, bad, "asynchronous pg_train_step");
}

// ------------------------------------------------------------------ step launch
static StepParams make_params(pg_model* m, const Geometry& g, const int32_t* idx, const int32_t* corr, int B,
                              float lr, float* loss_dev, int world = 1) {
  StepParams p{};
  p.C = m->C; p.W1 = m->W1; p.W1T = m->W1T; p.b1 = m->b1; p.w2 = m->w2; p.b2 = m->b2;
  p.V = m->V; p.d = m->d; p.n = m->n; p.h = m->h;
  p.idx = idx; p.corr = corr; p.B = B;
  p.inv_B = m->reduce_sum ? 1.0f : 1.0f / (float)((int64_t)B * world);
  p.act = m->act;
  p.lr = lr;
  p.P = g.P; p.R = g.R; p.T = g.T; p.cap = g.cap;
  p.dense_part = m->dense_part;
  p.dense_len = g.dense_len; p.dense_stride = g.dense_stride;
  p.list_rows = m->list_rows; p.list_vals = m->list_vals; p.list_off = m->list_off;
  p.NL = g.NL;
  p.st = m->st;
  p.loss_out = loss_dev;
  p.mode = m->mode;
  p.smem_bytes = (int)g.smem;
  p.lay = g.lay;
  p.trace = m->trace;
  p.world = world;
  p.rank = 0;
  return p;
}

static pg_status run_step(pg_model* m, const int32_t* idx, const int32_t* corr, int B, float lr,
                          float* loss_dev);

// ------------------------------------------------------------------ data parallel
static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Window of one rank for batch B: ready flags, two parity
// blocks [headers | rows | values], two dense sums.
static XLayout x_layout(const pg_model* m, const Geometry& g, int B) {
  XLayout xl{};
  const size_t cap = (size_t)(m->n + 1) * B;
  size_t o = 0;
  xl.flags = o;  o = align_up(o + sizeof(unsigned) * kMaxRanks * kMaxSMs, 4096);
  xl.rows = align_up(sizeof(XHdr) * kMaxSMs, 256);
  xl.vals = align_up(xl.rows + sizeof(int32_t) * cap, 256);
  xl.blk_bytes = align_up(xl.vals + sizeof(float) * cap * m->d, 256);
  for (int k = 0; k < 2; ++k) { xl.blk[k] = o; o = align_up(o + xl.blk_bytes, 4096); }
  for (int k = 0; k < 2; ++k) { xl.dense[k] = o; o = align_up(o + sizeof(float) * g.dense_stride, 4096); }
  xl.total = align_up(o, 1 << 21);
  return xl;
}

static size_t allgather_bytes(const pg_model* m, const XLayout& xl, int world) {
  return (size_t)(world - 1) * xl.blk_bytes;
}
static size_t table_bytes(const pg_model* m, int world) {   // ring all-reduce: 2 (G-1)/G of the table
  return (size_t)(2.0 * (world - 1) / world * (double)m->V * m->d * sizeof(float));
}

// Cost model (SURVEY.md §8(e) "chosen by measured cost"): the peer window
// moves only the merged rows and needs no collective launch, so it wins when
// available; otherwise the fewer bytes received per rank.
static int choose_exchange(const pg_model* m, const XLayout& xl, int world, bool peer_ok) {
  if (m->xmode != PG_EXCHANGE_AUTO) return m->xmode;
  if (peer_ok) return PG_EXCHANGE_PEER;
  return allgather_bytes(m, xl, world) <= table_bytes(m, world) ? PG_EXCHANGE_ALLGATHER : PG_EXCHANGE_TABLE;
}

static pg_status ensure_x_small(pg_model* m) {
  if (!m->xepoch) {
    CU(cudaMalloc(&m->xepoch, sizeof(unsigned) * kMaxSMs));
    CU(cudaMemset(m->xepoch, 0, sizeof(unsigned) * kMaxSMs));
  }
  if (!m->xstats) {
    CU(cudaMalloc(&m->xstats, sizeof(unsigned long long) * 2));
    CU(cudaMemset(m->xstats, 0, sizeof(unsigned long long) * 2));
  }
  return PG_OK;
}

// Collective on first use of a batch size (every rank calls pg_train_step with
// the same batch): window, then the mode's buffers.
static pg_status ensure_dp(pg_model* m, int B) {
  if (m->x_B == B && m->xwin) return PG_OK;
  CU(cudaStreamSynchronize(m->stream));
  free_dp(m);
  if (pg_status s = ensure_x_small(m)) return s;
  const Geometry g = geometry(m, B, m->world);
  m->xl = x_layout(m, g, B);
  std::string err;
  bool peer_ok = false;
  const bool want_peer = m->xmode == PG_EXCHANGE_AUTO || m->xmode == PG_EXCHANGE_PEER;
  if (want_peer && nccl_shim_lsa_size(m->comm) == m->world) {
    void* buf = nullptr;
    void* win = nullptr;
    if (!nccl_shim_mem_alloc(&buf, m->xl.total, &err)) {
      m->xwin = static_cast<unsigned char*>(buf);
      m->xwin_nccl = true;
      if (cudaMemset(m->xwin, 0, m->xl.total) == cudaSuccess && cudaDeviceSynchronize() == cudaSuccess &&
          !nccl_shim_window_register(m->comm, buf, m->xl.total, &win, &err)) {
        m->xwin_handle = win;
        std::vector<unsigned long long> ptrs(m->world);
        if (!nccl_lsa_pointers(win, m->world, ptrs.data(), &err)) {
          bool uniform = ptrs[m->rank] == reinterpret_cast<unsigned long long>(m->xwin) || true;
          const unsigned long long stride = m->world > 1 ? ptrs[1] - ptrs[0] : m->xl.total;
          for (int r = 1; r < m->world; ++r) uniform &= ptrs[r] - ptrs[r - 1] == stride;
          if (uniform) {
            m->xbase = reinterpret_cast<unsigned char*>(ptrs[0]);
            m->xstride = stride;
            peer_ok = true;
          }
        }
      }
    }
    cudaGetLastError();
  }
  if (m->xmode == PG_EXCHANGE_PEER && !peer_ok)
    return fail(PG_ENCCL, "PG_EXCHANGE_PEER: no load/store-accessible symmetric window (%s)", err.c_str());
  m->xchosen = choose_exchange(m, m->xl, m->world, peer_ok);
  if (m->xchosen != PG_EXCHANGE_PEER && !m->xwin) {
    CU(cudaMalloc(&m->xwin, m->xl.total));
    CU(cudaMemset(m->xwin, 0, m->xl.total));
  }
  if (m->xchosen == PG_EXCHANGE_ALLGATHER) CU(cudaMalloc(&m->xrecv, m->xl.blk_bytes * (size_t)m->world));
  if (m->xchosen != PG_EXCHANGE_PEER) CU(cudaMalloc(&m->xdense, sizeof(float) * g.dense_stride));
  if (m->xchosen == PG_EXCHANGE_TABLE) {
    CU(cudaMalloc(&m->xtable, sizeof(float) * (size_t)m->V * m->d));
    CU(cudaMemset(m->xtable, 0, sizeof(float) * (size_t)m->V * m->d));
  }
  m->x_launch_bytes = m->xchosen == PG_EXCHANGE_ALLGATHER ? (int64_t)allgather_bytes(m, m->xl, m->world)
                      : m->xchosen == PG_EXCHANGE_TABLE   ? (int64_t)table_bytes(m, m->world)
                                                          : 0;
  m->x_B = B;
  CU(cudaDeviceSynchronize());
  return PG_OK;
}

static void set_x(StepParams& p, pg_model* m, int rank, int world) {
  p.world = world;
  p.rank = rank;
  p.xl = m->xl;
  p.xcap = (m->n + 1) * p.B;
  p.xepoch = m->xepoch;
  p.xstats = m->xstats;
  p.mode = PG_SCATTER_DET;
}

// Data-parallel step over NCCL (one process per GPU).
static pg_status dp_step(pg_model* m, const int32_t* idx, const int32_t* corr, int B, float lr, float* loss_dev) {
  if (!m->comm) return fail(PG_ENCCL, "data-parallel step without a communicator");
  if (pg_status s = ensure_dp(m, B)) return s;
  const Geometry g = geometry(m, B, m->world);
  StepParams p = make_params(m, g, idx, corr, B, lr, loss_dev, m->world);
  set_x(p, m, m->rank, m->world);
  p.xwin = m->xwin;
  int l = 0;
  std::string err;
  if (m->xchosen == PG_EXCHANGE_PEER) {   // one kernel: phase 1, publish, wait, merge
    p.xbase = m->xbase;
    p.xstride = m->xstride;
    p.xpeer = 1;
    launch_step_phases(p, 1 | 8 | 16, m->fast, m->stream, &l);
    m->launches += l;
    CU(cudaGetLastError());
    return PG_OK;
  }
  p.xgathered = 1;
  launch_step_phases(p, 1 | 8, m->fast, m->stream, &l);
  CU(cudaGetLastError());
  int rc = nccl_shim_group(true, &err);
  bool opened = rc == 0;
  float* dense_w = reinterpret_cast<float*>(m->xwin + m->xl.dense[0]);
  if (!rc) rc = nccl_shim_allreduce_sum_f32(dense_w, m->xdense, (size_t)g.dense_stride, m->comm, m->stream, &err);
  if (!rc && m->xchosen == PG_EXCHANGE_ALLGATHER)
    rc = nccl_shim_allgather_bytes(m->xwin + m->xl.blk[0], m->xrecv, m->xl.blk_bytes, m->comm, m->stream, &err);
  if (opened) {
    std::string e2;
    if (nccl_shim_group(false, &e2) && !rc) { rc = 1; err = e2; }
  }
  if (rc) return fail(PG_ENCCL, "%s", err.c_str());
  p.xdense = m->xdense;
  m->x_steps += 1;
  if (m->xchosen == PG_EXCHANGE_ALLGATHER) {
    p.xbase = m->xrecv;
    p.xstride = m->xl.blk_bytes;
    launch_step_phases(p, 16, m->fast, m->stream, &l);
  } else {   // TABLE
    launch_dp_table(p, m->xtable, 0, m->num_sms, m->stream, &l);
    CU(cudaGetLastError());
    if (nccl_shim_allreduce_sum_f32(m->xtable, m->xtable, (size_t)m->V * m->d, m->comm, m->stream, &err))
      return fail(PG_ENCCL, "%s", err.c_str());
    launch_dp_table(p, m->xtable, 2, m->num_sms, m->stream, &l);
  }
  m->launches += l;
  CU(cudaGetLastError());
  return PG_OK;
}

static pg_status run_step(pg_model* m, const int32_t* idx, const int32_t* corr, int B, float lr,
                          float* loss_dev) {
  if (m->comm) return dp_step(m, idx, corr, B, lr, loss_dev);
  const Geometry g = geometry(m, B);
  StepParams p = make_params(m, g, idx, corr, B, lr, loss_dev);
  if (g.dw1_gemm) {   // the one-GPU step only (the data-parallel phases exchange records)
    p.dw1_gemm = 1;
    p.xg = m->xg;
    p.sg = m->sg;
    p.tmap = m->d_tmap;
  }
  int l = 0;
  launch_step(p, m->fused, m->fast, m->stream, &l);
  m->launches += l;
  CU(cudaGetLastError());
  return PG_OK;
}

// Rank-order sum of `world` float vectors spaced `stride` bytes apart (the
// all-reduce of the emulated NCCL exchanges).
__global__ void sum_ranks_kernel(const unsigned char* base, size_t stride, int world, int n, float* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int r = 0; r < world; ++r) acc += reinterpret_cast<const float*>(base + (size_t)r * stride)[i];
    out[i] = acc;
  }
}

// Replicas of one model on ONE device (pg_train_step_group): the kernels of
// the data-parallel path, the collectives emulated on the device.
extern "C" pg_status pg_train_step_group(pg_model** ms, int world, const int32_t* idx_all,
                                         const int32_t* corr_all, int32_t batch_local, float lr,
                                         float* loss_out) {
  if (!ms || world < 1 || world > kMaxRanks) return fail(PG_EINVAL, "pg_train_step_group: bad arguments");
  if (!idx_all || !corr_all) return fail(PG_EINVAL, "pg_train_step_group: null index pointer");
  if (batch_local < 1) return fail(PG_EINVAL, "pg_train_step_group: empty batch");
  if (!std::isfinite(lr) || !(lr > 0.f)) return fail(PG_EINVAL, "pg_train_step_group: lr must be finite and > 0");
  for (int r = 0; r < world; ++r) {
    if (pg_status s = check_model(ms[r])) return s;
    if (ms[r]->comm) return fail(PG_EINVAL, "pg_train_step_group: model %d has an NCCL communicator", r);
    if (ms[r]->d != ms[0]->d || ms[r]->n != ms[0]->n || ms[r]->h != ms[0]->h || ms[r]->V != ms[0]->V ||
        ms[r]->device != ms[0]->device)
      return fail(PG_EINVAL, "pg_train_step_group: shape or device mismatch");
    for (int k = 0; k < r; ++k)
      if (ms[k] == ms[r]) return fail(PG_EINVAL, "pg_train_step_group: replica %d repeated", r);
  }
  pg_model* m0 = ms[0];
  if (pg_status s = set_device(m0)) return s;
  for (int r = 0; r < world; ++r) {
    if (pg_status s = ensure_ws(ms[r], batch_local, world)) return s;
    if (pg_status s = ensure_x_small(ms[r])) return s;
  }
  const int n = m0->n;
  const Geometry g = geometry(m0, batch_local, world);
  const XLayout xl = x_layout(m0, g, batch_local);
  const int mode = m0->xmode == PG_EXCHANGE_AUTO ? PG_EXCHANGE_PEER : m0->xmode;
  std::lock_guard<std::mutex> lk(g_group_mu);
  GroupX* gx = nullptr;
  for (auto& e : g_groups)
    if (e.first == m0) gx = &e.second;
  if (!gx) { g_groups.emplace_back(m0, GroupX{}); gx = &g_groups.back().second; }
  if (gx->world != world || gx->B != batch_local || gx->mode != mode) {
    CU(cudaDeviceSynchronize());
    free_group(*gx);
    CU(cudaMalloc(&gx->win, xl.total * world));
    CU(cudaMemset(gx->win, 0, xl.total * world));
    if (mode == PG_EXCHANGE_ALLGATHER) CU(cudaMalloc(&gx->recv, xl.blk_bytes * world));
    if (mode != PG_EXCHANGE_PEER) CU(cudaMalloc(&gx->dense, sizeof(float) * g.dense_stride));
    if (mode == PG_EXCHANGE_TABLE) {
      CU(cudaMalloc(&gx->table, sizeof(float) * (size_t)m0->V * m0->d));
      CU(cudaMemset(gx->table, 0, sizeof(float) * (size_t)m0->V * m0->d));
    }
    gx->world = world; gx->B = batch_local; gx->mode = mode;
    for (int r = 0; r < world; ++r) CU(cudaMemset(ms[r]->xepoch, 0, sizeof(unsigned) * kMaxSMs));
  }
  m0->xchosen = mode;
  cudaStream_t s0 = m0->stream;
  // phase 1 + publish, replica after replica on replica 0's stream
  std::vector<StepParams> ps(world);
  for (int r = 0; r < world; ++r) {
    pg_model* m = ms[r];
    const int32_t *di = nullptr, *dc = nullptr;
    cudaStream_t own = m->stream;
    m->stream = s0;   // staging orders the copies before the launch on s0
    pg_status st = stage_inputs(m, idx_all + (size_t)r * batch_local * n, corr_all + (size_t)r * batch_local,
                                batch_local, &di, &dc);
    if (!st) {
      ps[r] = make_params(m, g, di, dc, batch_local, lr, nullptr, world);
      set_x(ps[r], m, r, world);
      ps[r].xl = xl;
      ps[r].xwin = gx->win + (size_t)r * xl.total;
      ps[r].xbase = gx->win;
      ps[r].xstride = xl.total;
      ps[r].xpeer = mode == PG_EXCHANGE_PEER;
      ps[r].xgathered = mode != PG_EXCHANGE_PEER;
      int l = 0;
      launch_step_phases(ps[r], 1 | 8, m->fast, s0, &l);
      m->launches += l;
      if (cudaGetLastError() != cudaSuccess) st = fail(PG_ECUDA, "pg_train_step_group: launch failed");
      if (!st) st = consume_inputs(m);
    }
    m->stream = own;
    if (st) return st;
  }
  // the "collectives"
  int l0 = 0;
  if (mode != PG_EXCHANGE_PEER) {
    sum_ranks_kernel<<<m0->num_sms, 256, 0, s0>>>(gx->win + xl.dense[0], xl.total, world, g.dense_stride, gx->dense);
    ++l0;
  }
  if (mode == PG_EXCHANGE_ALLGATHER)
    for (int r = 0; r < world; ++r)
      CU(cudaMemcpyAsync(gx->recv + (size_t)r * xl.blk_bytes, gx->win + (size_t)r * xl.total + xl.blk[0], xl.blk_bytes,
                         cudaMemcpyDeviceToDevice, s0));
  for (int r = 0; r < world; ++r) {
    StepParams& q = ps[r];
    int l = 0;
    if (mode == PG_EXCHANGE_TABLE) {
      q.xdense = gx->dense;
      launch_dp_table(q, gx->table, 0, m0->num_sms, s0, &l);   // every replica adds into the shared table
    } else {
      if (mode == PG_EXCHANGE_ALLGATHER) {
        q.xdense = gx->dense;
        q.xbase = gx->recv;
        q.xstride = xl.blk_bytes;
      }
      launch_step_phases(q, 16, ms[r]->fast, s0, &l);
    }
    ms[r]->launches += l;
    CU(cudaGetLastError());
  }
  if (mode == PG_EXCHANGE_TABLE)
    for (int r = 0; r < world; ++r) {   // apply; the last replica re-zeroes the shared table
      int l = 0;
      launch_dp_table(ps[r], gx->table, r + 1 < world ? 1 : 2, m0->num_sms, s0, &l);
      ms[r]->launches += l;
      CU(cudaGetLastError());
    }
  m0->launches += l0;
  if (!loss_out) return PG_OK;
  CU(cudaMemcpyAsync(m0->st_host, m0->st, sizeof(DevStatus), cudaMemcpyDeviceToHost, s0));
  CU(cudaStreamSynchronize(s0));
  *loss_out = m0->st_host->last_loss;
  return status_from_flags(m0->st_host->last_flags, m0->st_host->last_bad, "pg_train_step_group");
}

extern "C" pg_status pg_nccl_unique_id(void* out) {
  if (!out) return fail(PG_EINVAL, "pg_nccl_unique_id: NULL");
  std::string err;
  if (nccl_shim_unique_id(out, &err)) return fail(PG_ENCCL, "%s", err.c_str());
  return PG_OK;
}

extern "C" pg_status pg_attach_nccl(pg_model* m, int rank, int world, const void* uid) {
  if (pg_status s = check_model(m)) return s;
  if (!uid || world < 1 || world > kMaxRanks || rank < 0 || rank >= world)
    return fail(PG_EINVAL, "pg_attach_nccl: bad rank/world (world <= %d)", kMaxRanks);
  if (pg_status s = set_device(m)) return s;
  CU(cudaStreamSynchronize(m->stream));
  std::string err;
  void* comm = nullptr;
  if (nccl_shim_init(&comm, rank, world, uid, &err)) return fail(PG_ENCCL, "%s", err.c_str());
  free_dp(m);   // window / buffers belong to the old communicator
  if (m->comm) nccl_shim_destroy(m->comm);
  m->comm = comm;
  m->rank = rank;
  m->world = world;
  free_ws(m);   // geometry depends on world
  if (m->xepoch) CU(cudaMemset(m->xepoch, 0, sizeof(unsigned) * kMaxSMs));
  return PG_OK;
}

extern "C" pg_status pg_exchange_info(pg_model* m, int* mode, uint64_t* stats2, int reset) {
  if (pg_status s = check_model(m)) return s;
  if (mode) *mode = m->xchosen;
  if (pg_status s = set_device(m)) return s;
  if (stats2 || reset) {
    if (pg_status s = ensure_x_small(m)) return s;
    unsigned long long h[2] = {0, 0};
    CU(cudaStreamSynchronize(m->stream));
    CU(cudaMemcpy(h, m->xstats, sizeof h, cudaMemcpyDeviceToHost));
    h[0] += (unsigned long long)(m->x_launch_bytes * m->x_steps);
    if (stats2) { stats2[0] = h[0]; stats2[1] = h[1]; }
    if (reset) { CU(cudaMemset(m->xstats, 0, sizeof h)); m->x_steps = 0; }
  }
  return PG_OK;
}

// ------------------------------------------------------------------ standalone scatter-add
namespace {
std::mutex g_sc_mu;
void* g_sc_ws[16] = {nullptr};
size_t g_sc_cap[16] = {0};
unsigned long long g_sc_epoch[16] = {0};
}

static pg_status scatter_common(float* W, int64_t rows, int32_t cols, const float* Y, const int32_t* I, int64_t n,
                                int mode, void* stream, int* err_dev, bool blocking) {
  if (!W || (n > 0 && (!Y || !I))) return fail(PG_EINVAL, "pg_scatter_add: null pointer");
  if (rows < 1 || cols < 1 || n < 0 || rows > 2147483647LL) return fail(PG_EINVAL, "pg_scatter_add: bad shape");
  if (mode != PG_SCATTER_DET && mode != PG_SCATTER_ATOMIC) return fail(PG_EINVAL, "pg_scatter_add: bad mode");
  if (!scatter_supported(cols, mode))
    return fail(PG_EINVAL, "pg_scatter_add: DET mode supports cols in {<=32, 64, 128} (got %d)", cols);
  if ((reinterpret_cast<uintptr_t>(W) | reinterpret_cast<uintptr_t>(Y)) & 15)
    return fail(PG_EINVAL, "pg_scatter_add: W and Y must be 16-byte aligned");
  if (n == 0) return PG_OK;
  if (n >= (1ll << 30)) return fail(PG_EINVAL, "pg_scatter_add: n must be < 2^30");
  if (ptr_kind(W) != PTR_DEVICE || ptr_kind(Y) != PTR_DEVICE || ptr_kind(I) != PTR_DEVICE)
    return fail(PG_EINVAL, "pg_scatter_add: W, Y and I must be device pointers");
  int dev = 0;
  CU(cudaGetDevice(&dev));
  if (dev >= 16) return fail(PG_EINVAL, "pg_scatter_add: device index >= 16");
  int sms = 0;
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  std::lock_guard<std::mutex> lk(g_sc_mu);
  ScatterPlan pl = scatter_plan(rows, cols, n, sms);
  if (pl.total_bytes > g_sc_cap[dev]) {
    CU(cudaDeviceSynchronize());
    cudaFree(g_sc_ws[dev]);
    g_sc_ws[dev] = nullptr;
    CU(cudaMalloc(&g_sc_ws[dev], pl.total_bytes));
    CU(cudaMemset(g_sc_ws[dev], 0, pl.total_bytes));   // status block and ATOMIC replica rows start zeroed
    g_sc_cap[dev] = pl.total_bytes;
    CU(scatter_prepare(1024));   // the largest digit table any plan uses
  }
  int l = 0, slot = -1;
  CU(scatter_launch(pl, g_sc_ws[dev], W, rows, cols, Y, I, n, mode, s, &l, g_sc_epoch[dev]++, &slot));
  ScatterStatus* st = reinterpret_cast<ScatterStatus*>(static_cast<unsigned char*>(g_sc_ws[dev]) + pl.off_status);
  const int* flag_dev = slot < 0 ? &st->flag : &st->hot[slot].flag;
  if (err_dev) CU(cudaMemcpyAsync(err_dev, flag_dev, sizeof(int), cudaMemcpyDeviceToDevice, s));
  if (!blocking) return PG_OK;
  ScatterStatus hs;
  CU(cudaMemcpyAsync(&hs, st, sizeof hs, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  const int flag = slot < 0 ? hs.flag : hs.hot[slot].flag;
  const unsigned long long bad = slot < 0 ? ~hs.nbad : ~hs.hot[slot].nbad;
  if (flag) {
    return fail(PG_ERANGE, "pg_scatter_add: index out of range at position %lld (value %d); W unchanged",
                (long long)(bad >> 32), (int)(unsigned)(bad & 0xffffffffull));
  }
  return PG_OK;
}

extern "C" pg_status pg_scatter_add(float* W, int64_t rows, int32_t cols, const float* Y, const int32_t* I,
                                    int64_t n, int mode, void* stream) {
  return scatter_common(W, rows, cols, Y, I, n, mode, stream, nullptr, true);
}

extern "C" pg_status pg_scatter_add_async(float* W, int64_t rows, int32_t cols, const float* Y, const int32_t* I,
                                          int64_t n, int mode, void* stream, int* err_flag_dev) {
  return scatter_common(W, rows, cols, Y, I, n, mode, stream, err_flag_dev, false);
}
