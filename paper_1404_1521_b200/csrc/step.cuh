// step.cuh -- parameters shared by the host API (api.cu) and the step kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pg {

// Device-resident status / synchronisation block (one per model).
struct DevStatus {
  unsigned long long bad;        // current step: min over (pos << 32 | uint32 value)
  unsigned long long last_bad;   // result of the most recent step
  unsigned long long sticky_bad; // min over asynchronous steps since pg_sync
  unsigned long long score_bad;  // pg_score index check
  unsigned bar_count;            // grid barrier arrivals (returns to 0)
  unsigned bar_gen;              // grid barrier generation
  unsigned done;                 // phase-2 arrival counter (flag-reset protocol)
  int flags;                     // current step: bit0 bad index
  int last_flags;                // most recent step: bit0 bad index, bit1 non-finite loss
  int sticky_flags;              // OR over asynchronous steps since pg_sync
  int rank_flags;                // data-parallel: OR over all ranks
  int score_flags;
  float last_loss;
  int pad[3];
};

// Fixed per-step decomposition: P CTAs, CTA p
// owns examples [p*B/P, (p+1)*B/P), processed in R chunks of <= T examples.
// Chunk (p, r) is list L = p*R + r.
struct StepParams {
  // parameters
  float* C;
  float* W1;
  float* b1;
  float* w2;
  const float* b2;
  int64_t V;
  int d, n, h;
  // batch (this rank's shard)
  const int32_t* idx;
  const int32_t* corr;
  int B;
  float inv_B;   // 1 / global batch
  float lr;
  // decomposition
  int P, R, T, cap;     // cap = (n+1)*T list capacity
  // workspace: per-CTA dense partial records
  float* dense_part;    // [Ptot][dense_stride]: dW1 | db1 | dw2 | hinge
  int dense_len;        // n*d*h + 2h
  int dense_stride;     // multiple of 4, > dense_len
  // per-chunk aggregated (row, gradient-sum) lists, bucketed by owner CTA
  int32_t* list_rows;   // [NLtot][cap]
  float* list_vals;     // [NLtot][cap][d]
  int32_t* list_off;    // [NLtot][P+1]  (owner q's entries: [off[q], off[q+1]))
  // phase 2 sees Ptot records / NLtot lists (== P / P*R on one GPU;
  // world*P / world*P*R after a data-parallel all-gather)
  int Ptot, NLtot;
  DevStatus* st;
  float* loss_out;      // optional device pointer
  int mode;             // 0 det, 1 atomic
  int smem_bytes;       // dynamic smem available
};

void launch_step(const StepParams& p, int fused, int fast, cudaStream_t s, int* launches);
int step_fast_ok(int d, int n, int h);
int step_block_threads(int d, int n, int h, int fast);
int step_chunk_T(int d, int n, int h, int fast);
size_t step_smem_bytes(int d, int n, int h, int T, int P, int fast);
cudaError_t step_prepare(int fast, size_t optin, size_t* usable);
int step_max_blocks(int fast, int threads, size_t smem, int* out);

}  // namespace pg
