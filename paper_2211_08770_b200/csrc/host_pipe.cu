// tt_round_batch_host: B independent roundings (BASELINE configs[3], "C4") from HOST inputs to
// HOST results in one C-ABI call -- the end-to-end path a user without device buffers takes.
//
// The batch is cut into contiguous slices of whole waves of the batched engine.  Three streams:
//   hp_h2d      host -> device copy of slice c+1 into staging buffer (c+1) % 2
//   ctx->stream the rounding of slice c (run_batch, batch_round.cu)
//   hp_d2h      device -> host copy of slice c-1's compacted results
// The two copy directions run on different copy engines, so both overlap the rounding.  Staging
// buffer s is rewritten only after the rounding that read it (event `consumed`).  The streams and
// buffers persist on the context (no allocation in steady state).
#include <algorithm>
#include <cmath>
#include <cstring>

#include "batch_round.cuh"

namespace ttb {

void host_pipe_release(tt_ctx ctx) {
  if (ctx->hp_h2d) { cudaStreamSynchronize(ctx->hp_h2d); cudaStreamDestroy(ctx->hp_h2d); ctx->hp_h2d = nullptr; }
  if (ctx->hp_d2h) { cudaStreamSynchronize(ctx->hp_d2h); cudaStreamDestroy(ctx->hp_d2h); ctx->hp_d2h = nullptr; }
  for (double*& p : ctx->hp_stage) {
    if (p) cudaFree(p);
    p = nullptr;
  }
  ctx->hp_stage_doubles = 0;
}

namespace {

struct Ev {  // RAII event
  cudaEvent_t e = nullptr;
  Ev() { TTB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming)); }
  ~Ev() { if (e) cudaEventDestroy(e); }
  Ev(const Ev&) = delete;
  Ev& operator=(const Ev&) = delete;
  Ev(Ev&& o) noexcept : e(o.e) { o.e = nullptr; }
};

void ensure_pipe(tt_ctx ctx, size_t stage_doubles) {
  if (!ctx->hp_h2d) TTB_CUDA(cudaStreamCreateWithFlags(&ctx->hp_h2d, cudaStreamNonBlocking));
  if (!ctx->hp_d2h) TTB_CUDA(cudaStreamCreateWithFlags(&ctx->hp_d2h, cudaStreamNonBlocking));
  if (ctx->hp_stage_doubles >= stage_doubles) return;
  TTB_CUDA(cudaStreamSynchronize(ctx->hp_h2d));
  TTB_CUDA(cudaStreamSynchronize(ctx->stream));
  for (double*& p : ctx->hp_stage) {
    if (p) cudaFree(p);
    p = nullptr;
  }
  ctx->hp_stage_doubles = 0;
  for (double*& p : ctx->hp_stage)
    if (cudaMalloc(reinterpret_cast<void**>(&p), stage_doubles * sizeof(double)) != cudaSuccess) {
      (void)cudaGetLastError();
      fail(TT_ENOMEM, "tt_round_batch_host: staging allocation failed");
    }
  ctx->hp_stage_doubles = stage_doubles;
}

}  // namespace

void round_batch_host(tt_ctx ctx, const BatchDesc& shape, const double* const* host_core, const int64_t* item_stride,
                      const double* coeff, const double* norms, const tt_round_opts& o, int slices, double* out_host,
                      int64_t out_capacity, int64_t* out_count, int64_t* ranks_out, double* norms_out) {
  const int B = shape.B, K = shape.K, d = shape.d;
  // doubles of core k of term l per item, and per item in total
  std::vector<int64_t> sz((size_t)K * d);
  int64_t item_doubles = 0;
  for (int l = 0; l < K; ++l)
    for (int k = 0; k < d; ++k) {
      sz[(size_t)l * d + k] = shape.r[(size_t)l][(size_t)k] * shape.n[(size_t)k] * shape.r[(size_t)l][(size_t)k + 1];
      if (item_stride[(size_t)l * d + k] < sz[(size_t)l * d + k] && B > 1)
        fail(TT_EINVAL, "tt_round_batch_host: item_stride smaller than the core size");
      item_doubles += sz[(size_t)l * d + k];
    }
  // slices of whole waves: one CTA per item, 2 resident per SM in the right-to-left kernel and 3 in
  // the left-to-right ones, so 6 x SMs items fill both without a partial wave per slice
  const int64_t wave = 6 * (int64_t)ctx->num_sms;
  const int64_t S = std::max(1, slices);
  int64_t step;
  if (B > wave * S) step = std::max<int64_t>(wave, (int64_t)std::llround((double)B / (double)S / (double)wave) * wave);
  else step = std::max<int64_t>(1, ceil_div(B, S));
  std::vector<int64_t> bounds;
  for (int64_t a = 0; a < B; a += step) bounds.push_back(a);
  bounds.push_back(B);
  const int C = (int)bounds.size() - 1;
  int64_t max_items = 0;
  for (int c = 0; c < C; ++c) max_items = std::max(max_items, bounds[(size_t)c + 1] - bounds[(size_t)c]);
  ensure_pipe(ctx, (size_t)std::max<int64_t>(max_items * item_doubles, 1));
  cudaStream_t h2d = ctx->hp_h2d, d2h = ctx->hp_d2h;
  // everything queued on the ctx stream before this call is ordered before the pipeline, and the
  // ctx stream waits for the last copies at the end: the call is one unit in ctx-stream order
  Ev entry;
  TTB_CUDA(cudaEventRecord(entry.e, ctx->stream));
  TTB_CUDA(cudaStreamWaitEvent(h2d, entry.e, 0));
  TTB_CUDA(cudaStreamWaitEvent(d2h, entry.e, 0));
  std::vector<Ev> staged((size_t)C), consumed((size_t)C), rounded((size_t)C);
  auto copy_in = [&](int c) {
    const int64_t a = bounds[(size_t)c], nb = bounds[(size_t)c + 1] - a;
    double* buf = ctx->hp_stage[c % 2];
    if (c >= 2) TTB_CUDA(cudaStreamWaitEvent(h2d, consumed[(size_t)c - 2].e, 0));
    int64_t off = 0;
    for (int l = 0; l < K; ++l)
      for (int k = 0; k < d; ++k) {
        const size_t q = (size_t)l * d + k;
        const double* src = host_core[q] + a * item_stride[q];
        if (item_stride[q] == sz[q] || nb == 1)
          TTB_CUDA(cudaMemcpyAsync(buf + off, src, sizeof(double) * (size_t)(nb * sz[q]), cudaMemcpyHostToDevice, h2d));
        else
          TTB_CUDA(cudaMemcpy2DAsync(buf + off, sizeof(double) * (size_t)sz[q], src, sizeof(double) * (size_t)item_stride[q],
                                     sizeof(double) * (size_t)sz[q], (size_t)nb, cudaMemcpyHostToDevice, h2d));
        off += nb * sz[q];
      }
    TTB_CUDA(cudaEventRecord(staged[(size_t)c].e, h2d));
  };
  std::vector<BatchOut> live;  // results whose device->host copies may still run
  live.reserve((size_t)C);
  int64_t offset = 0;
  bool overflow = false;
  try {
    copy_in(0);
    for (int c = 0; c < C; ++c) {
      if (c + 1 < C) copy_in(c + 1);
      const int64_t a = bounds[(size_t)c], nb = bounds[(size_t)c + 1] - a;
      BatchDesc in;
      in.B = (int)nb;
      in.K = K;
      in.d = d;
      in.n = shape.n;
      in.r = shape.r;
      in.tab.resize((size_t)nb * K * d);
      const double* buf = ctx->hp_stage[c % 2];
      int64_t off = 0;
      for (int l = 0; l < K; ++l)
        for (int k = 0; k < d; ++k) {
          const size_t q = (size_t)l * d + k;
          for (int64_t b = 0; b < nb; ++b) in.tab[((size_t)b * K + l) * d + k] = buf + off + b * sz[q];
          off += nb * sz[q];
        }
      in.coef.assign(coeff + (size_t)a * K, coeff + (size_t)(a + nb) * K);
      if (norms) in.norm.assign(norms + (size_t)a * K, norms + (size_t)(a + nb) * K);
      else in.norm.assign((size_t)nb * K, NAN);
      TTB_CUDA(cudaStreamWaitEvent(ctx->stream, staged[(size_t)c].e, 0));
      live.emplace_back();
      BatchOut& res = live.back();
      run_batch(ctx, in, o, res);
      TTB_CUDA(cudaEventRecord(consumed[(size_t)c].e, ctx->stream));  // staging read, results compacted
      TTB_CUDA(cudaStreamWaitEvent(d2h, consumed[(size_t)c].e, 0));
      for (int64_t b = 0; b < nb; ++b) {
        if (ranks_out)
          std::memcpy(ranks_out + (size_t)(a + b) * (d + 1), res.ranks.data() + (size_t)b * (d + 1), sizeof(int64_t) * (d + 1));
        if (norms_out) norms_out[a + b] = res.norm[(size_t)b];
      }
      for (size_t w = 0; w < res.arenas.size(); ++w) {
        const int64_t cnt = res.arena_size[w];
        if (!overflow && offset + cnt <= out_capacity)
          TTB_CUDA(cudaMemcpyAsync(out_host + offset, res.arenas[w], sizeof(double) * (size_t)cnt, cudaMemcpyDeviceToHost, d2h));
        else
          overflow = true;
        offset += cnt;
      }
      // the arenas go back to the pool once their copies are done (stream-ordered on d2h)
      for (void* p : res.arenas) TTB_CUDA(cudaFreeAsync(p, d2h));
      res.arenas.clear();
      TTB_CUDA(cudaEventRecord(rounded[(size_t)c].e, d2h));
    }
  } catch (...) {
    for (BatchOut& r : live)
      for (void* p : r.arenas) cudaFreeAsync(p, ctx->stream);
    cudaStreamSynchronize(h2d);
    cudaStreamSynchronize(d2h);
    throw;
  }
  Ev done_in, done_out;
  TTB_CUDA(cudaEventRecord(done_in.e, h2d));
  TTB_CUDA(cudaEventRecord(done_out.e, d2h));
  TTB_CUDA(cudaStreamWaitEvent(ctx->stream, done_in.e, 0));
  TTB_CUDA(cudaStreamWaitEvent(ctx->stream, done_out.e, 0));
  TTB_CUDA(cudaStreamSynchronize(d2h));
  TTB_CUDA(cudaStreamSynchronize(h2d));
  if (out_count) *out_count = offset;
  if (overflow)
    fail(TT_EINVAL, "tt_round_batch_host: out_host holds " + std::to_string(out_capacity) + " doubles, the results need " +
                        std::to_string(offset) + " (*out_count)");
}

}  // namespace ttb

using namespace ttb;

extern "C" tt_status tt_round_batch_host(tt_ctx ctx, int32_t B, int32_t K, int32_t d, const int64_t* n, const int64_t* r,
                                         const double* const* host_core, const int64_t* item_stride, const double* coeff,
                                         const double* norms, const tt_round_opts* opts, int32_t slices,
                                         double* out_host, int64_t out_capacity, int64_t* out_count, int64_t* ranks_out,
                                         double* norms_out) {
  if (!ctx || B < 0 || K < 1 || d < 1 || !n || !r || !host_core || !item_stride || (B > 0 && !coeff) ||
      out_capacity < 0 || (out_capacity > 0 && !out_host))
    return TT_EINVAL;
  try {
    BatchDesc shape;
    batch_desc_shape(shape, B, K, d, n, r);
    for (int q = 0; q < K * d; ++q)
      if (!host_core[q]) fail(TT_EINVAL, "null host core base pointer");
    tt_round_opts o = default_round_opts();
    if (opts) o = *opts;
    if (out_count) *out_count = 0;
    if (B == 0) return TT_OK;
    round_batch_host(ctx, shape, host_core, item_stride, coeff, norms, o, slices, out_host, out_capacity, out_count,
                     ranks_out, norms_out);
    return TT_OK;
  } catch (const Error& e) {
    ctx->last_error = e.msg;
    return e.status;
  } catch (const std::bad_alloc&) {
    ctx->last_error = "host allocation failed";
    return TT_ENOMEM;
  } catch (const std::exception& e) {
    ctx->last_error = e.what();
    return TT_EINVAL;
  }
}
