#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <sstream>

#include "common.cuh"

namespace ttb {

void fail(tt_status s, const std::string& msg) { throw Error{s, msg}; }

void debug_check(tt_ctx ctx, const char* cls, const char* file, int line) {
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) {
    std::ostringstream os;
    os << "kernel class '" << cls << "' launched at " << file << ":" << line << " failed: " << cudaGetErrorString(e);
    fail(TT_ECUDA, os.str());
  }
}

void check_cuda(cudaError_t e, const char* what, const char* file, int line) {
  if (e == cudaSuccess) return;
  std::ostringstream os;
  os << "CUDA error '" << cudaGetErrorString(e) << "' in " << what << " at " << file << ":" << line;
  fail(e == cudaErrorMemoryAllocation ? TT_ENOMEM : TT_ECUDA, os.str());
}

void DBuf::alloc(tt_ctx c, size_t n) {
  release();
  ctx = c;
  count = n;
  if (n == 0) return;
  void* q = nullptr;
  cudaError_t e = cudaMallocAsync(&q, n * sizeof(double), c->stream);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    fail(TT_ENOMEM, "device allocation of " + std::to_string(n * 8) + " bytes failed");
  }
  p = static_cast<double*>(q);
}

void DBuf::release() {
  if (p && ctx) cudaFreeAsync(p, ctx->stream);
  p = nullptr;
  count = 0;
}

void IBuf::alloc(tt_ctx c, size_t n) {
  release();
  ctx = c;
  count = n;
  if (n == 0) return;
  void* q = nullptr;
  cudaError_t e = cudaMallocAsync(&q, n * sizeof(int), c->stream);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    fail(TT_ENOMEM, "device allocation failed");
  }
  p = static_cast<int*>(q);
}

void IBuf::release() {
  if (p && ctx) cudaFreeAsync(p, ctx->stream);
  p = nullptr;
  count = 0;
}

// Stage `bytes` of host data in the ctx's pinned ring (16 MiB) and return its address, or null
// when it does not fit (then the caller copies from pageable memory).  A region is reused only
// after the copy that last read it has completed (event per staged copy, waited on overlap).
static const char* stage_pinned(tt_ctx c, const void* host, size_t bytes) {
  constexpr size_t cap = (size_t)16 << 20;
  if (bytes > cap / 4) return nullptr;
  if (!c->up_ring) {
    if (cudaMallocHost(reinterpret_cast<void**>(&c->up_ring), cap) != cudaSuccess) {
      (void)cudaGetLastError();
      c->up_ring = nullptr;
      return nullptr;
    }
    c->up_cap = cap;
    c->up_off = 0;
  }
  size_t off = (c->up_off + 255) & ~(size_t)255;
  if (off + bytes > c->up_cap) off = 0;
  // wait for pending copies that read [off, off + bytes)
  for (size_t q = 0; q < c->up_pending.size();) {
    const auto& pd = c->up_pending[q];
    if (pd.start < off + bytes && off < pd.end) {
      TTB_CUDA(cudaEventSynchronize(pd.ev));
      c->up_events.push_back(pd.ev);
      c->up_pending.erase(c->up_pending.begin() + (ptrdiff_t)q);
    } else {
      ++q;
    }
  }
  std::memcpy(c->up_ring + off, host, bytes);
  c->up_off = off + bytes;
  return c->up_ring + off;
}

static void staged_done(tt_ctx c, const char* src, size_t bytes) {
  cudaEvent_t ev;
  if (!c->up_events.empty()) { ev = c->up_events.back(); c->up_events.pop_back(); }
  else TTB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  TTB_CUDA(cudaEventRecord(ev, c->stream));
  const size_t start = (size_t)(src - c->up_ring);
  c->up_pending.push_back({start, start + bytes, ev});
  if (c->up_pending.size() > 256) {  // bound the list: retire the oldest
    TTB_CUDA(cudaEventSynchronize(c->up_pending.front().ev));
    c->up_events.push_back(c->up_pending.front().ev);
    c->up_pending.erase(c->up_pending.begin());
  }
}

// Device-side copy out of the pinned ring (mapped host memory, same address under UVA): an SM
// load over PCIe instead of a copy-engine transfer, so a small descriptor upload is never
// queued behind a caller's multi-GB host-to-device copy on another stream (the copy engine
// serves transfers in submission order).
__global__ void upload_kernel(unsigned long long* __restrict__ dst, const unsigned long long* __restrict__ src,
                              size_t words, unsigned char* __restrict__ dtail, const unsigned char* __restrict__ stail,
                              int tail) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < words; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
  if (blockIdx.x == 0 && (int)threadIdx.x < tail) dtail[threadIdx.x] = stail[threadIdx.x];
}

void BBuf::upload(tt_ctx c, const void* host, size_t bytes, bool via_sm) {
  if (p && ctx) cudaFreeAsync(p, ctx->stream);
  ctx = c;
  p = nullptr;
  if (bytes == 0) return;
  cudaError_t e = cudaMallocAsync(&p, bytes, c->stream);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    p = nullptr;
    fail(TT_ENOMEM, "descriptor allocation failed");
  }
  const char* src = stage_pinned(c, host, bytes);
  static const bool sm_ok = [] {
    const char* e = std::getenv("TT_B200_UPLOAD_SM");
    return !(e && e[0] == '0');
  }();
  if (src && !(via_sm && sm_ok)) {
    TTB_CUDA(cudaMemcpyAsync(p, src, bytes, cudaMemcpyHostToDevice, c->stream));
    staged_done(c, src, bytes);
  } else if (src) {
    const size_t words = bytes / 8;
    const int tail = (int)(bytes - words * 8);
    const int blocks = (int)std::min<size_t>(std::max<size_t>((words + 255) / 256, 1), 64);
    TTB_RUN(c, "aux", 0.0, 2.0 * bytes,
            upload_kernel<<<blocks, 256, 0, c->stream>>>(
                static_cast<unsigned long long*>(p), reinterpret_cast<const unsigned long long*>(src), words,
                static_cast<unsigned char*>(p) + words * 8, reinterpret_cast<const unsigned char*>(src) + words * 8,
                tail));
    staged_done(c, src, bytes);
  } else {
    TTB_CUDA(cudaMemcpyAsync(p, host, bytes, cudaMemcpyHostToDevice, c->stream));
  }
}

static cudaEvent_t pool_event(tt_ctx ctx) {
  if (!ctx->prof_pool.empty()) {
    cudaEvent_t e = ctx->prof_pool.back();
    ctx->prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  TTB_CUDA(cudaEventCreate(&e));
  return e;
}

int prof_begin(tt_ctx ctx) {
  if (!ctx->prof) return -1;
  TTProfPending p;
  p.start = pool_event(ctx);
  p.stop = pool_event(ctx);
  p.cls = -1;
  p.flops = p.bytes = 0.0;
  TTB_CUDA(cudaEventRecord(p.start, ctx->stream));
  ctx->prof_pending.push_back(p);
  return (int)ctx->prof_pending.size() - 1;
}

void prof_end(tt_ctx ctx, int token, const char* cls, double flops, double bytes) {
  if (token < 0 || !ctx->prof) return;
  TTProfPending& p = ctx->prof_pending[(size_t)token];
  TTB_CUDA(cudaEventRecord(p.stop, ctx->stream));
  int idx = -1;
  for (size_t i = 0; i < ctx->prof_cls.size(); ++i)
    if (ctx->prof_cls[i].name == cls) { idx = (int)i; break; }
  if (idx < 0) {
    ctx->prof_cls.push_back(TTProfEntry{cls});
    idx = (int)ctx->prof_cls.size() - 1;
  }
  p.cls = idx;
  p.flops = flops;
  p.bytes = bytes;
  if (ctx->prof_pending.size() > 4096) prof_resolve(ctx);
}

void prof_resolve(tt_ctx ctx) {
  if (ctx->prof_pending.empty()) return;
  TTB_CUDA(cudaStreamSynchronize(ctx->stream));
  for (TTProfPending& p : ctx->prof_pending) {
    if (p.cls >= 0) {
      float ms = 0.f;
      TTB_CUDA(cudaEventElapsedTime(&ms, p.start, p.stop));
      TTProfEntry& e = ctx->prof_cls[(size_t)p.cls];
      e.launches++;
      e.ms += ms;
      e.flops += p.flops;
      e.bytes += p.bytes;
    }
    ctx->prof_pool.push_back(p.start);
    ctx->prof_pool.push_back(p.stop);
  }
  ctx->prof_pending.clear();
}

void prof_credit(tt_ctx ctx, const char* cls, double flops) {
  if (!ctx->prof) return;
  for (TTProfEntry& e : ctx->prof_cls)
    if (e.name == cls) { e.flops += flops; return; }
}

void prof_reset(tt_ctx ctx) {
  prof_resolve(ctx);
  ctx->prof_cls.clear();
}

static void ensure_pinned(tt_ctx ctx, size_t bytes) {
  if (ctx->h_pinned_bytes >= bytes) return;
  if (ctx->h_pinned) cudaFreeHost(ctx->h_pinned);
  size_t b = bytes < 4096 ? 4096 : bytes;
  TTB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&ctx->h_pinned), b));
  ctx->h_pinned_bytes = b;
}

void d2h_small(tt_ctx ctx, double* host, const double* dev, size_t n) {
  if (n == 0) return;
  ensure_pinned(ctx, n * sizeof(double));
  TTB_CUDA(cudaMemcpyAsync(ctx->h_pinned, dev, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  TTB_CUDA(cudaStreamSynchronize(ctx->stream));
  std::memcpy(host, ctx->h_pinned, n * sizeof(double));
}

void d2h_small_int(tt_ctx ctx, int* host, const int* dev, size_t n) {
  if (n == 0) return;
  ensure_pinned(ctx, n * sizeof(int));
  TTB_CUDA(cudaMemcpyAsync(ctx->h_pinned, dev, n * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  TTB_CUDA(cudaStreamSynchronize(ctx->stream));
  std::memcpy(host, ctx->h_pinned, n * sizeof(int));
}

void* ctx_scratch(tt_ctx ctx, size_t bytes) {
  if (bytes <= ctx->scratch_bytes) return ctx->scratch;
  TTB_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ctx->scratch) cudaFree(ctx->scratch);
  ctx->scratch = nullptr;
  ctx->scratch_bytes = 0;
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    (void)cudaGetLastError();
    fail(TT_ENOMEM, "workspace allocation of " + std::to_string(bytes) + " bytes failed");
  }
  ctx->scratch = p;
  ctx->scratch_bytes = bytes;
  return p;
}

tt_tensor tensor_alloc(tt_ctx ctx, int d, const std::vector<int64_t>& n, const std::vector<int64_t>& r) {
  tt_tensor t = new tt_tensor_s();
  t->d = d;
  t->n = n;
  t->r = r;
  size_t total = 0;
  for (int k = 0; k < d; ++k) total += (size_t)(r[k] * n[k] * r[k + 1]);
  void* q = nullptr;
  cudaError_t e = cudaMallocAsync(&q, (total ? total : 1) * sizeof(double), ctx->stream);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    delete t;
    fail(TT_ENOMEM, "tensor allocation failed");
  }
  t->block = static_cast<double*>(q);
  t->core.resize(d);
  t->core_c.resize(d);
  size_t off = 0;
  for (int k = 0; k < d; ++k) {
    t->core[k] = t->block + off;
    t->core_c[k] = t->core[k];
    off += (size_t)(r[k] * n[k] * r[k + 1]);
  }
  return t;
}

void tensor_free(tt_ctx ctx, tt_tensor t) {
  if (!t) return;
  if (t->block) cudaFreeAsync(t->block, ctx->stream);
  if (t->arena_refs && --*t->arena_refs == 0) {
    cudaFreeAsync(t->arena, ctx->stream);
    delete t->arena_refs;
  }
  delete t;
}

TTShape view_shape(const tt_view& v) {
  if (v.d < 1) fail(TT_EINVAL, "TT order d must be >= 1");
  if (!v.n || !v.r || !v.core) fail(TT_EINVAL, "null shape/core pointer in tt_view");
  TTShape s;
  s.d = v.d;
  s.n.assign(v.n, v.n + v.d);
  s.r.assign(v.r, v.r + v.d + 1);
  if (s.r[0] != 1 || s.r[v.d] != 1) fail(TT_ESHAPE, "boundary ranks must be r_0 = r_d = 1 (PAPER.md:45)");
  for (int k = 0; k < v.d; ++k) {
    if (s.n[k] < 1 || s.r[k] < 1 || s.r[k + 1] < 1) fail(TT_ESHAPE, "mode sizes and ranks must be >= 1");
    if (!v.core[k]) fail(TT_EINVAL, "null core pointer");
  }
  return s;
}

}  // namespace ttb
