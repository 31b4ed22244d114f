// Shared internals of libtt_b200: context, tensors, device buffers, error handling,
// warp/block reductions.  sm_100a only.
#pragma once

#include <nvtx3/nvToolsExt.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <string>
#include <vector>

#include "../../include/tt_b200.h"

namespace ttb {

// ------------------------------------------------------------------ errors
struct Error {
  tt_status status;
  std::string msg;
};

[[noreturn]] void fail(tt_status s, const std::string& msg);
void check_cuda(cudaError_t e, const char* what, const char* file, int line);
#define TTB_CUDA(x) ::ttb::check_cuda((x), #x, __FILE__, __LINE__)
#define TTB_LAUNCHED(ctx) do { (ctx)->launches++; TTB_CUDA(cudaGetLastError()); } while (0)
// NVTX range (one range per rounding phase and driver step; header-only NVTX3, a
// no-op unless a profiler is attached): TTB_RANGE("name") covers the enclosing scope.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define TTB_RANGE_CAT2(a, b) a##b
#define TTB_RANGE_CAT(a, b) TTB_RANGE_CAT2(a, b)
#define TTB_RANGE(name) ::ttb::NvtxRange TTB_RANGE_CAT(_ttb_range_, __LINE__)(name)

// Profiled launch: TTB_RUN(ctx, "class", flops, bytes, kernel<<<...>>>(...));
#define TTB_RUN(ctx, cls, fl, by, ...)                      \
  do {                                                      \
    const int _ttb_tok = ::ttb::prof_begin(ctx);            \
    __VA_ARGS__;                                            \
    TTB_LAUNCHED(ctx);                                      \
    ::ttb::prof_end(ctx, _ttb_tok, cls, (double)(fl), (double)(by)); \
    if ((ctx)->debug_sync) ::ttb::debug_check(ctx, cls, __FILE__, __LINE__); \
  } while (0)

}  // namespace ttb

struct TTProfEntry {
  std::string name;
  int64_t launches = 0;
  double ms = 0.0, flops = 0.0, bytes = 0.0;
};

struct TTProfPending {
  cudaEvent_t start, stop;
  int cls;
  double flops, bytes;
};

struct tt_ctx_s {
  int device = 0;
  // per-kernel-class CUDA-event timing (tt_ctx_profile); events recorded on ctx->stream
  bool prof = false;
  bool debug_sync = false;  // TT_B200_DEBUG_SYNC=1: synchronise and check after every launch
  std::vector<TTProfEntry> prof_cls;
  std::vector<TTProfPending> prof_pending;
  std::vector<cudaEvent_t> prof_pool;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  std::string last_error;
  int64_t launches = 0;
  double* h_pinned = nullptr;   // small pinned staging area for scalar reads
  size_t h_pinned_bytes = 0;
  void* scratch = nullptr;      // grow-only device workspace of the batched engine
  size_t scratch_bytes = 0;
  // pinned ring for small host->device uploads (descriptor tables): a copy from pinned memory
  // is truly asynchronous, a pageable one waits for the stream (BBuf::upload)
  char* up_ring = nullptr;
  size_t up_cap = 0, up_off = 0;
  struct UpPending { size_t start, end; cudaEvent_t ev; };
  std::vector<UpPending> up_pending;
  std::vector<cudaEvent_t> up_events;  // free events
  // host-to-host batched rounding (tt_round_batch_host, host_pipe.cu): persistent copy streams
  // (one per direction: the two directions use different copy engines) and two device staging
  // buffers, so repeated calls allocate nothing
  cudaStream_t hp_h2d = nullptr, hp_d2h = nullptr;
  // batched engine: second stream for the other half of a wave (kernel tails of one half fill with
  // the other half's CTAs) and its fork / join events
  cudaStream_t br_aux[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t br_fork = nullptr, br_join[3] = {nullptr, nullptr, nullptr};
  double* hp_stage[2] = {nullptr, nullptr};
  size_t hp_stage_doubles = 0;
  // optional communicator (comm.cu): sharded Gram / dot batches / phase-2 roundings
  struct TTComm* comm = nullptr;
  // observer of the drivers' rounding calls (tt_ctx_round_hook)
  tt_round_hook round_hook = nullptr;
  void* round_hook_user = nullptr;
};

struct tt_tensor_s {
  int d = 0;
  std::vector<int64_t> n, r;
  std::vector<double*> core;
  std::vector<const double*> core_c;
  double norm = NAN;
  double* block = nullptr;  // one allocation holding every core
  // Batched results share one arena (batch_round.cu): block stays null, the cores point into
  // `arena`, freed when the last tensor of the batch is freed (host refcount).
  void* arena = nullptr;
  int64_t* arena_refs = nullptr;
};

namespace ttb {

// ------------------------------------------------------------------ device buffers
// Stream-ordered allocations (cudaMallocAsync on the ctx stream, default mempool).
struct DBuf {
  tt_ctx ctx = nullptr;
  double* p = nullptr;
  size_t count = 0;
  DBuf() = default;
  DBuf(tt_ctx c, size_t n) { alloc(c, n); }
  void alloc(tt_ctx c, size_t n);
  void release();
  ~DBuf() { release(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : ctx(o.ctx), p(o.p), count(o.count) { o.p = nullptr; o.count = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); ctx = o.ctx; p = o.p; count = o.count; o.p = nullptr; o.count = 0; }
    return *this;
  }
};

struct IBuf {  // int32 device buffer
  tt_ctx ctx = nullptr;
  int* p = nullptr;
  size_t count = 0;
  IBuf() = default;
  IBuf(tt_ctx c, size_t n) { alloc(c, n); }
  void alloc(tt_ctx c, size_t n);
  void release();
  ~IBuf() { release(); }
  IBuf(const IBuf&) = delete;
  IBuf& operator=(const IBuf&) = delete;
};

struct BBuf {  // raw byte device buffer (descriptor tables)
  tt_ctx ctx = nullptr;
  void* p = nullptr;
  BBuf() = default;
  ~BBuf() { if (p && ctx) cudaFreeAsync(p, ctx->stream); }
  BBuf(const BBuf&) = delete;
  BBuf& operator=(const BBuf&) = delete;
  // allocate and copy `bytes` from host (pageable copy: the host buffer may be reused on return)
  // via_sm: copy out of the pinned ring with a kernel instead of the copy engine (for uploads
  // that must not queue behind a caller's bulk transfer on another stream)
  void upload(tt_ctx c, const void* host, size_t bytes, bool via_sm = false);
};

// ------------------------------------------------------------------ profiling
int prof_begin(tt_ctx ctx);  // returns a token (-1 when profiling is off)
void prof_end(tt_ctx ctx, int token, const char* cls, double flops, double bytes);
void prof_resolve(tt_ctx ctx);  // synchronises and folds pending events into the classes
void prof_reset(tt_ctx ctx);
// add algorithmic flops to a class after the fact (work known only once ranks are read back)
void prof_credit(tt_ctx ctx, const char* cls, double flops);
void debug_check(tt_ctx ctx, const char* cls, const char* file, int line);

// device -> host copy of a few doubles through the pinned staging buffer (synchronises)
void d2h_small(tt_ctx ctx, double* host, const double* dev, size_t n);
void d2h_small_int(tt_ctx ctx, int* host, const int* dev, size_t n);
// grow-only context workspace (cudaMalloc, kept until tt_ctx_destroy); synchronises on growth
void* ctx_scratch(tt_ctx ctx, size_t bytes);

// ------------------------------------------------------------------ tensors
tt_tensor tensor_alloc(tt_ctx ctx, int d, const std::vector<int64_t>& n, const std::vector<int64_t>& r);
void tensor_free(tt_ctx ctx, tt_tensor t);

// Shape of a borrowed view, validated.
struct TTShape {
  int d;
  std::vector<int64_t> n, r;
};
TTShape view_shape(const tt_view& v);

// ------------------------------------------------------------------ reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum; red must hold >= 32 doubles; all threads get the result.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (warp == 0) {
    t = (lane < nw) ? red[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

constexpr double U_ROUND = 1.1102230246251565e-16;  // 2^-53

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace ttb
