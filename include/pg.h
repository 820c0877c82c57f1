/*
 * pg.h -- C ABI of the B200-native Polyglot/SENNA window-LM SGD step
 * (arXiv:1404.1521).  Library: paper_1404_1521_b200/libpg.so (sm_100a).
 *
 * The operation (PAPER.md gives no formulas; readings in DESIGN.md / SURVEY.md
 * §8(c)).  For every example k of a batch, with n-word window idx[k][0..n-1],
 * centre c = floor(n/2) and corrupt centre word corr[k]:
 *   x   = concat_p C[idx[k][p]]                 gather  (dual of PAPER.md:98-102)
 *   x'  = x with block c replaced by C[corr[k]]
 *   a   = W1^T x + b1,  z = hardtanh(a) = clamp(a, -1, 1)       (north_star;
 *                        tanh instead with PG_OPT_ACTIVATION = PG_ACT_TANH)
 *   s   = w2 . z + b2;  s' likewise for x'
 *   l_k = max(0, 1 - s + s')                    (north_star)
 *   L   = (1/B) sum_k l_k                       (mean, reading G4)
 * and one synchronous SGD update with the gradients of L at the pre-step
 * parameters: theta -= lr * dL/dtheta for W1, b1, w2, b2 (db2 == 0 exactly),
 * and the embedding update as the paper's scatter-add ("advanced indexing",
 * PAPER.md:98-102): C[row_j] += -lr * G_j for every gradient row, duplicates
 * accumulating.  hardtanh'(+-1) = 0 and the hinge is active only for m > 0
 * (readings G2, G3).
 *
 * Layouts (row-major, fp32 parameters, int32 indices):
 *   C [vocab][dim]; W1 [window*dim][hidden] (row p*dim+j = feature j of slot p);
 *   b1 [hidden]; w2 [hidden]; b2 scalar;
 *   idx_batch [batch][window]; corrupt_idx [batch]; scores [batch].
 *
 * Pointers: any pointer argument may be HOST (pageable or pinned) or DEVICE
 * memory of the model's device; the library detects which with
 * cudaPointerGetAttributes.  Input pointers are borrowed until the call
 * returns (blocking calls) or until the stream work that reads them completes
 * (asynchronous calls).  The model owns all of its device memory.
 *
 * Errors: every function returns pg_status.  Host-checked PG_EINVAL happens
 * before any launch (null handle/pointer, batch < 1, lr not finite or <= 0,
 * dim/window/hidden < 1, vocab < 2 or > INT32_MAX).  Out-of-range indices are
 * detected ON THE DEVICE: the step is then skipped as a whole (no parameter
 * changes) and PG_ERANGE is reported with the first
 * offending flat position (idx positions 0..B*n-1, then corrupt positions
 * B*n..B*n+B-1) and its value in pg_last_error().  A non-finite loss skips the
 * update the same way and reports PG_EDIVERGED.  Device errors
 * of asynchronous steps are sticky and surface at the next blocking call or
 * pg_sync().  A model is not thread-safe: one model per host thread.
 */
#ifndef PG_H
#define PG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PG_ABI_VERSION 1

typedef struct pg_model pg_model; /* opaque; owns all device memory */

typedef enum {
  PG_OK = 0,
  PG_EINVAL = 1,     /* bad argument, detected on the host before any launch */
  PG_ERANGE = 2,     /* index outside [0, vocab); nothing was modified */
  PG_ENOMEM = 3,     /* device or pinned-host allocation failed */
  PG_ECUDA = 4,      /* CUDA runtime error (message in pg_last_error) */
  PG_ENCCL = 5,      /* NCCL error in the data-parallel exchange */
  PG_EDIVERGED = 6   /* non-finite loss; nothing was modified */
} pg_status;

/* Embedding scatter-add strategies (PAPER.md:121-127 leaves the duplicate-row
 * conflict policy unstated; SPEC.md:111-115 names both). */
enum {
  PG_SCATTER_DET = 0,    /* sort by row, fixed-order segmented sums: bit-reproducible */
  PG_SCATTER_ATOMIC = 1  /* repeated rows pre-summed per tile, then vector atomic adds
                            (red.global.add.v4.f32: FTZ, order varies run to run) */
};

/* pg_set_option keys */
enum {
  PG_OPT_SCATTER = 1, /* value: PG_SCATTER_DET (default) or PG_SCATTER_ATOMIC */
  PG_OPT_STREAM = 2,  /* value: (int64_t)(cudaStream_t); 0 = legacy default stream */
  PG_OPT_FUSED = 3,   /* 1 (default): one persistent cooperative kernel per step;
                         0: two ordinary kernels (phase 1 | phase 2), same results */
  PG_OPT_RESERVE = 4, /* value: batch size; allocates the step workspace for it now
                         (so later steps at <= that batch never allocate -- e.g.
                         before CUDA-graph capture).  After pg_attach_nccl it also
                         sets up the data-parallel exchange for exactly that batch
                         and is then collective (every rank, same value).
                         PG_EINVAL unless 1..2^30. */
  PG_OPT_TRACE = 5,   /* value: (int64_t) device pointer to >= 64*P uint64 slots, 0 = off.
                         Per-CTA %globaltimer stamps of the step's stages; honoured
                         only by the instrumented build libpg_trace.so (-DPG_TRACE),
                         ignored by libpg.so.  For scripts/trace_step.py. */
  PG_OPT_ACTIVATION = 6, /* value: PG_ACT_HARDTANH (default) or PG_ACT_TANH; applies
                            to pg_train_step* and pg_score from the next call on.
                            PG_EINVAL for any other value. */
  PG_OPT_REDUCTION = 7,  /* value: PG_REDUCE_MEAN (default: L = (1/B) sum_k l_k and
                            its gradient, B the global batch; reading G4) or
                            PG_REDUCE_SUM (L = sum_k l_k: the same step as MEAN at
                            lr * B; the reading PAPER.md:197-198 hints at).
                            PG_EINVAL for any other value. */
  PG_OPT_EXCHANGE = 8    /* value: PG_EXCHANGE_* -- how data-parallel ranks exchange
                            gradients (after pg_attach_nccl, and in
                            pg_train_step_group).  Takes effect at the next step. */
};

/* Data-parallel gradient exchange.  Every
 * rank first merges its own embedding-gradient rows per row (one entry per
 * distinct row); then:
 *   PEER      one kernel per step: each rank's owner CTAs read the other
 *             ranks' merged rows and dense-gradient sums directly from their
 *             NCCL symmetric-memory windows over NVLink (load/store
 *             accessible peers), ready flags pushed by the writers; bytes on
 *             the wire = the merged rows;
 *   ALLGATHER ncclAllReduce of the dense gradient + ncclAllGather of the
 *             merged (row, gradient) records, padded to capacity;
 *   TABLE     ncclAllReduce of the dense gradient and of a full vocab x dim
 *             embedding-gradient table;
 *   AUTO      (default) PEER when every rank is load/store accessible, else
 *             the cheaper of ALLGATHER and TABLE by bytes received per rank.
 * PEER and ALLGATHER sum each row's and each dense element's per-rank parts in
 * rank order on every rank (bit-identical replicas, and bit-identical to each
 * other); TABLE's sums are NCCL's (identical on all ranks). */
enum { PG_EXCHANGE_AUTO = 0, PG_EXCHANGE_PEER = 1, PG_EXCHANGE_ALLGATHER = 2, PG_EXCHANGE_TABLE = 3 };

enum { PG_REDUCE_MEAN = 0, PG_REDUCE_SUM = 1 };

/* Hidden-layer nonlinearity f (PG_OPT_ACTIVATION).  HARDTANH: f(a) =
 * clamp(a, -1, 1), f'(a) = 1 for |a| < 1 and 0 otherwise (north_star; SENNA's
 * HardTanh; subgradient 0 at |a| = 1).  TANH: f(a) = tanh(a), f'(a) =
 * 1 - tanh(a)^2 (the CPU spec's model). */
enum { PG_ACT_HARDTANH = 0, PG_ACT_TANH = 1 };

/* pg_init -- allocate a model on the current CUDA device and initialise it:
 * C ~ U[-0.5, 0.5), W1 ~ U[-0.5/(window*dim), +), w2 ~ U[-0.5/hidden, +),
 * b1 = b2 = 0, each value float32((2u-1)*r) with u the top 24 bits of output i
 * of a SplitMix64 stream keyed by seed ^ (0x632BE59BD9B4E019*(tensor_id+1)),
 * tensor ids C=0, W1=1, w2=2 (reading G10).  North-star name:
 * pg_init(vocab, dim, window, hidden, seed).  *out receives the handle. */
pg_status pg_init(pg_model** out, int64_t vocab, int32_t dim, int32_t window,
                  int32_t hidden, uint64_t seed);

/* pg_train_step -- one SGD step on `batch` windows (the north-star
 * pg_train_step(idx_batch, corrupt_idx, lr) -> loss).
 *   loss_out: pageable HOST pointer -> blocking: waits, reports device errors,
 *             writes L;
 *             DEVICE pointer, or PAGE-LOCKED host pointer (cudaHostAlloc /
 *             cudaHostRegister / torch pin_memory) -> asynchronous on the model
 *             stream: the step kernel writes L (float) there itself (a 4-byte
 *             device-to-host store for pinned memory), valid once the stream
 *             has reached the step (pg_sync); errors are sticky;
 *             NULL -> asynchronous, loss discarded.
 * The returned loss is computed with the pre-step parameters.
 * After pg_attach_nccl, `batch` is this rank's shard (equal on all ranks), the
 * gradient is that of the GLOBAL mean loss, and L is the global mean. */
pg_status pg_train_step(pg_model* m, const int32_t* idx_batch,
                        const int32_t* corrupt_idx, int32_t batch, float lr,
                        float* loss_out);

/* Literal north-star form: returns L, or NaN on any failure (see pg_last_error). */
float pg_train_step_loss(pg_model* m, const int32_t* idx_batch,
                         const int32_t* corrupt_idx, int32_t batch, float lr);

/* pg_score -- s = w2 . f(W1^T x + b1) + b2 for each window (f: PG_OPT_ACTIVATION)
 * (SPEC.md:204-212).  Blocking if scores_out is host memory, else asynchronous. */
pg_status pg_score(pg_model* m, const int32_t* idx_batch, int32_t batch,
                   float* scores_out);

void pg_free(pg_model* m);

/* Thread-local message describing the last non-PG_OK status. */
const char* pg_last_error(void);

/* Parameters in the canonical layouts above; blocking copies.  Any pointer
 * may be NULL to skip that tensor.  pg_set_params does not change b2 when
 * b2 is NaN. */
pg_status pg_get_params(pg_model* m, float* C, float* W1, float* b1,
                        float* w2, float* b2);
pg_status pg_set_params(pg_model* m, const float* C, const float* W1,
                        const float* b1, const float* w2, float b2);
pg_status pg_get_shape(const pg_model* m, int64_t* vocab, int32_t* dim,
                       int32_t* window, int32_t* hidden);

pg_status pg_set_option(pg_model* m, int key, int64_t value);

/* Waits for the model stream and reports (then clears) sticky device errors. */
pg_status pg_sync(pg_model* m);

/* pg_scatter_add -- the paper's operation on its own (PAPER.md:98-102,
 * 121-136): for k = 0..n-1, W[I[k], :] += Y[k, :], duplicates accumulating.
 * W [rows][cols], Y [n][cols] fp32 and I [n] int32 are DEVICE pointers.
 * mode PG_SCATTER_DET: stable radix sort of (I[k], k), then segmented sums in
 * k order within fixed-size chunks, chunk partials combined in chunk order:
 * bit-reproducible run to run (cols in {1..32, 64, 128}).  mode
 * PG_SCATTER_ATOMIC: one streaming pass over Y; the rows that a fixed
 * spread sample of I shows to be frequent (>~0.1 % of entries) are summed in
 * shared memory per CTA (the most frequent) or spread over replica rows in the
 * library's workspace, every other entry reaches W through
 * red.global.add.v4.f32 per 16 B (cols % 4 == 0, cols <= 128; other widths
 * use scalar atomics); the summation order is not fixed.
 * Both modes use one library workspace per device: calls on the same device
 * must not overlap in time on different streams.
 * W and Y must be 16-byte aligned (cudaMalloc memory is), else PG_EINVAL.
 * n == 0 is a no-op.  Out-of-range I[k] -> PG_ERANGE and W unchanged.
 * stream: a cudaStream_t (NULL = legacy default).  Blocking (it reports the
 * index check); see pg_scatter_add_async for the graph-capturable variant. */
pg_status pg_scatter_add(float* W, int64_t rows, int32_t cols, const float* Y,
                         const int32_t* I, int64_t n, int mode, void* stream);

/* Asynchronous variant: no host synchronisation; an out-of-range index makes
 * the call a no-op on W and sets *err_flag_dev (device int, may be NULL). */
pg_status pg_scatter_add_async(float* W, int64_t rows, int32_t cols,
                               const float* Y, const int32_t* I, int64_t n,
                               int mode, void* stream, int* err_flag_dev);

/* Data parallelism over NCCL (one process per GPU).  rank 0 calls
 * pg_nccl_unique_id, the caller broadcasts the 128 bytes (torch.distributed),
 * then every rank calls pg_attach_nccl (world == 1 is allowed: a one-rank
 * communicator, the same code path).  Afterwards pg_train_step is collective:
 * every rank passes its own shard with the same batch, the gradient is that of
 * the global mean loss, and the update is exchanged as PG_OPT_EXCHANGE says.
 * The embedding update is always deterministic in data-parallel steps
 * (PG_OPT_SCATTER is ignored), so replicas stay bit-identical.  The first step
 * at a new batch size allocates (collectively) the exchange buffers.
 * Re-attaching replaces the communicator and frees the exchange buffers. */
pg_status pg_nccl_unique_id(void* out_128_bytes);
pg_status pg_attach_nccl(pg_model* m, int rank, int world,
                         const void* nccl_unique_id_128_bytes);

/* The exchange in use (PG_EXCHANGE_*, -1 before the first data-parallel step)
 * and statistics since the last call with reset != 0: stats[0] = bytes this
 * rank read from other ranks' records (PEER / group emulation; the NCCL
 * exchanges report their per-step receive volume times the steps), stats[1]
 * = the most (row, gradient) entries one owner CTA merged in one step.  Any
 * pointer may be NULL. */
pg_status pg_exchange_info(pg_model* m, int* mode, uint64_t* stats2, int reset);

/* pg_train_step_group -- `world` replicas of one model on ONE device take one
 * data-parallel step together: replica r trains on windows
 * idx_all[r*batch_local .. (r+1)*batch_local) (contiguous shards).  The same
 * kernels as the NCCL path run; the replicas' exchange windows are one device
 * buffer (PEER: read in place; ALLGATHER / TABLE: the collectives are
 * emulated by device copies and rank-order sums), so every replica applies
 * the same update (tests and single-GPU emulation of G ranks; the exchange
 * mode is replica 0's PG_OPT_EXCHANGE).  loss_out (host, may be NULL) gets
 * the global mean loss.  The replicas' own settings (stream, world) are left
 * as they were; models attached to NCCL are rejected. */
pg_status pg_train_step_group(pg_model** models, int world, const int32_t* idx_all,
                              const int32_t* corr_all, int32_t batch_local, float lr,
                              float* loss_out);

/* Number of kernels the library launched since the model was created
 * (counts host-side launches; graph replays are not counted). */
int64_t pg_kernel_launches(const pg_model* m);

int pg_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PG_H */
