// scatter.cuh -- host interface of the standalone scatter-add pipelines.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace pg {

struct ScatterStatus {
  int flag;                 // 1: an index was out of range -> nothing applied
  int pad;
  unsigned long long nbad;  // max over ~(position << 32 | uint32 value): 0 = no bad index, so one memset resets the block
  unsigned long long arrivals;   // grid-barrier counter of the cooperative kernels
  // sc_atomic_hot (no per-call memset): call e uses hot[e & 1] and clears
  // hot[(e + 1) & 1] for the next call; nbad = ~(position << 32 | value),
  // max-reduced, so 0 means "no bad index".  hot_arrivals is its own
  // monotonic barrier counter (fixed grid size).
  struct { int flag; int pad; unsigned long long nbad; } hot[2];
  unsigned long long hot_arrivals;
};

struct ScatterPlan {
  int passes, bits, bins, num_sms;
  int64_t ntiles, nchunks;
  size_t off_status, off_hist, off_ctr, off_lookback, zero_bytes;
  size_t off_ka, off_va, off_kb, off_vb, off_carry, off_cfk, off_clk, off_rep, total_bytes;
  // DET owner-bucket kernel (scatter_det.cu): used when det_owner is set
  int det_owner;
  size_t off_bucket, off_hcnt, off_hpart, off_hmask;
};

// scatter_det.cu
bool det_owner_ok(int64_t rows, int cols, int64_t n, int P);
size_t det_owner_hpart_floats(int P, int cols);
size_t det_owner_hmask_ints(int P);
cudaError_t det_owner_prepare();
cudaError_t det_owner_launch(const int32_t* I, const float* Y, float* W, int64_t rows, int cols, int64_t n,
                             ScatterStatus* st, int par, int2* bucket, unsigned* Hcnt, float* hpart, int* hmask,
                             int P, int64_t ypf_lines, cudaStream_t s);

ScatterPlan scatter_plan(int64_t rows, int cols, int64_t n, int num_sms);
int scatter_supported(int cols, int mode);
cudaError_t scatter_prepare(int bins);
// epoch: per-workspace call counter; *slot = -1 if the call reports through
// (flag, bad), else the hot[] slot it used.
cudaError_t scatter_launch(const ScatterPlan& pl, void* ws, float* W, int64_t rows, int cols,
                           const float* Y, const int32_t* I, int64_t n, int mode, cudaStream_t s,
                           int* launches, unsigned long long epoch, int* slot);

}  // namespace pg
