// extern "C" boundary of libtt_b200 (include/tt_b200.h).  Every entry point converts
// internal errors into a tt_status plus tt_last_error text; nothing throws across it.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <new>

#include "batch_round.cuh"
#include "comm.cuh"
#include "gram.cuh"
#include "orth.cuh"
#include "round.cuh"
#include "ttops.cuh"

using namespace ttb;

struct tt_batch_s {
  BatchOut res;
};

namespace {

template <typename F>
tt_status guarded(tt_ctx ctx, F f) {
  try {
    f();
    return TT_OK;
  } catch (const Error& e) {
    if (ctx) ctx->last_error = e.msg;
    return e.status;
  } catch (const std::bad_alloc&) {
    if (ctx) ctx->last_error = "host allocation failed";
    return TT_ENOMEM;
  } catch (const std::exception& e) {
    if (ctx) ctx->last_error = e.what();
    return TT_EINVAL;
  }
}

tt_round_opts resolve(const tt_round_opts* o) {
  tt_round_opts r = default_round_opts();
  if (o) r = *o;
  return r;
}

SumInput sum_of(int K, const double* coeff, const tt_view* terms) {
  if (K < 1 || !coeff || !terms) fail(TT_EINVAL, "TT-sum needs K >= 1 terms and coefficients");
  SumInput s;
  for (int l = 0; l < K; ++l) s.add(terms[l], coeff[l]);
  return s;
}

// Pair blocks (i0, j0, bi, bj) of the Gram matrix of A into packed_dev (tt_gram_blocks layout):
// the pair-tiled DMMA kernel for equally shaped sets, else the pair list of the TT-dot kernels.
void gram_blocks_local(tt_ctx ctx, const std::vector<TTRef>& A, int nblk, const int32_t* blk, double* packed_dev) {
  const int m = (int)A.size();
  for (int b = 0; b < nblk; ++b) {
    const int i0 = blk[4 * b], j0 = blk[4 * b + 1], bi = blk[4 * b + 2], bj = blk[4 * b + 3];
    if (i0 < 0 || j0 < 0 || bi < 0 || bj < 0 || i0 + bi > m || j0 + bj > m) fail(TT_EINDEX, "Gram block out of range");
  }
  if (nblk == 0) return;
  bool uniform = true;
  for (int i = 1; i < m; ++i)
    uniform = uniform && A[(size_t)i].d == A[0].d && A[(size_t)i].n == A[0].n && A[(size_t)i].r == A[0].r;
  const char* gt = std::getenv("TT_B200_GRAM_PAIRWISE");  // tests: force the per-pair kernel
  if (uniform && !(gt && gt[0] == '1')) {
    std::vector<const double*> cores;
    for (int i = 0; i < m; ++i) cores.insert(cores.end(), A[(size_t)i].core.begin(), A[(size_t)i].core.end());
    if (gram_tiled_supported(cores, m, A[0].d, A[0].n, A[0].r)) {
      gram_tiled_blocks(ctx, cores, m, A[0].d, A[0].n, A[0].r, nblk, blk, packed_dev);
      return;
    }
  }
  std::vector<std::pair<const TTRef*, const TTRef*>> pr;
  for (int b = 0; b < nblk; ++b) {
    const int i0 = blk[4 * b], j0 = blk[4 * b + 1], bi = blk[4 * b + 2], bj = blk[4 * b + 3];
    for (int s = 0; s < bi; ++s)
      for (int t = 0; t < bj; ++t) pr.push_back({&A[(size_t)(i0 + s)], &A[(size_t)(j0 + t)]});
  }
  dots_device(ctx, pr, packed_dev);
}

// G from the all-gathered pair blocks: tab[5 q] = (i0, j0, bi, bj, offset into recv) for every
// block of every rank; diagonal blocks contribute their lower half only (one value per pair).
__global__ void gram_unpack_blocks_kernel(const double* __restrict__ recv, const int64_t* __restrict__ tab, int m,
                                          double* __restrict__ G) {
  const int64_t* t = tab + 5 * (int64_t)blockIdx.x;
  const int i0 = (int)t[0], j0 = (int)t[1], bi = (int)t[2], bj = (int)t[3];
  const double* src = recv + t[4];
  for (int e = threadIdx.x; e < bi * bj; e += blockDim.x) {
    const int s = e / bj, u = e % bj;
    if (i0 == j0 && u > s) continue;
    const double v = src[e];
    G[(int64_t)(i0 + s) * m + (j0 + u)] = v;
    G[(int64_t)(j0 + u) * m + (i0 + s)] = v;
  }
}

// Sharded Gram (communicator attached): LPT-assigned pair blocks, one all-gather, device unpack.
void gram_sharded(tt_ctx ctx, const std::vector<TTRef>& A, double* G_dev) {
  const int m = (int)A.size(), N = comm_size(ctx), me = comm_rank(ctx);
  static const int bsz = [] {
    const char* e = std::getenv("TT_B200_GRAM_BLOCK");
    return (e && std::atoi(e) > 0) ? std::atoi(e) : 4;
  }();
  const std::vector<int32_t> blk = plan_gram_blocks(m, bsz);
  const int nb = (int)(blk.size() / 4);
  std::vector<double> cost((size_t)nb);
  for (int q = 0; q < nb; ++q) cost[(size_t)q] = (double)blk[(size_t)4 * q + 2] * blk[(size_t)4 * q + 3];
  const std::vector<int> owner = plan_lpt(cost, N);
  std::vector<int64_t> load((size_t)N, 0), tab((size_t)nb * 5);
  std::vector<int32_t> mine;
  for (int q = 0; q < nb; ++q) {
    const int o = owner[(size_t)q];
    for (int c = 0; c < 4; ++c) tab[(size_t)5 * q + c] = blk[(size_t)4 * q + c];
    tab[(size_t)5 * q + 4] = load[(size_t)o];  // offset inside owner o's packed buffer
    load[(size_t)o] += (int64_t)blk[(size_t)4 * q + 2] * blk[(size_t)4 * q + 3];
    if (o == me) mine.insert(mine.end(), blk.begin() + 4 * q, blk.begin() + 4 * q + 4);
  }
  const int64_t cap = std::max<int64_t>(*std::max_element(load.begin(), load.end()), 1);
  for (int q = 0; q < nb; ++q) tab[(size_t)5 * q + 4] += (int64_t)owner[(size_t)q] * cap;
  DBuf send(ctx, (size_t)cap), recv(ctx, (size_t)cap * N);
  gram_blocks_local(ctx, A, (int)(mine.size() / 4), mine.data(), send.p);
  comm_allgather(ctx, send.p, recv.p, sizeof(double) * (size_t)cap);
  BBuf dtab;
  dtab.upload(ctx, tab.data(), tab.size() * sizeof(int64_t));
  TTB_RUN(ctx, "aux", 0, 16.0 * m * m,
          gram_unpack_blocks_kernel<<<nb, 128, 0, ctx->stream>>>(recv.p, static_cast<const int64_t*>(dtab.p), m, G_dev));
}

}  // namespace

extern "C" {

tt_status tt_ctx_create(int device, void* stream, tt_ctx* out) {
  if (!out) return TT_EINVAL;
  *out = nullptr;
  tt_ctx c = new (std::nothrow) tt_ctx_s();
  if (!c) return TT_ENOMEM;
  tt_status st = guarded(c, [&] {
    TTB_CUDA(cudaSetDevice(device));
    c->device = device;
    c->stream = static_cast<cudaStream_t>(stream);
    TTB_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    const char* dbg = std::getenv("TT_B200_DEBUG_SYNC");
    c->debug_sync = dbg && dbg[0] == '1';
    // keep freed pool memory cached across calls (stream-ordered allocator)
    cudaMemPool_t pool;
    TTB_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    TTB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  });
  if (st != TT_OK) {
    delete c;
    return st;
  }
  *out = c;
  return TT_OK;
}

tt_status tt_ctx_destroy(tt_ctx ctx) {
  if (!ctx) return TT_EINVAL;
  if (ctx->h_pinned) cudaFreeHost(ctx->h_pinned);
  if (ctx->up_ring) {
    cudaStreamSynchronize(ctx->stream);
    cudaFreeHost(ctx->up_ring);
    for (auto& pd : ctx->up_pending) cudaEventDestroy(pd.ev);
    for (auto ev : ctx->up_events) cudaEventDestroy(ev);
  }
  if (ctx->scratch) { cudaStreamSynchronize(ctx->stream); cudaFree(ctx->scratch); }
  host_pipe_release(ctx);
  comm_release(ctx);
  for (int i = 0; i < 3; ++i) {
    if (ctx->br_aux[i]) { cudaStreamSynchronize(ctx->br_aux[i]); cudaStreamDestroy(ctx->br_aux[i]); }
    if (ctx->br_join[i]) cudaEventDestroy(ctx->br_join[i]);
  }
  if (ctx->br_fork) cudaEventDestroy(ctx->br_fork);
  delete ctx;
  return TT_OK;
}

tt_status tt_ctx_set_stream(tt_ctx ctx, void* stream) {
  if (!ctx) return TT_EINVAL;
  cudaStream_t ns = static_cast<cudaStream_t>(stream);
  if (ns == ctx->stream) return TT_OK;
  // Work already queued on the old stream may still use the context's scratch, pooled blocks
  // freed with cudaFreeAsync and descriptor uploads: the new stream waits for all of it.
  cudaEvent_t ev;
  if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventRecord(ev, ctx->stream) != cudaSuccess || cudaStreamWaitEvent(ns, ev, 0) != cudaSuccess) {
    ctx->last_error = std::string("tt_ctx_set_stream: ") + cudaGetErrorString(cudaGetLastError());
    return TT_ECUDA;
  }
  cudaEventDestroy(ev);
  ctx->stream = ns;
  return TT_OK;
}

const char* tt_last_error(tt_ctx ctx) { return ctx ? ctx->last_error.c_str() : "null context"; }

const char* tt_status_string(tt_status s) {
  switch (s) {
    case TT_OK: return "TT_OK";
    case TT_EINVAL: return "TT_EINVAL";
    case TT_ESHAPE: return "TT_ESHAPE";
    case TT_EINDEX: return "TT_EINDEX";
    case TT_ENOMEM: return "TT_ENOMEM";
    case TT_ECUDA: return "TT_ECUDA";
    case TT_ENOCONV: return "TT_ENOCONV";
    case TT_ESINGULAR_GRAM: return "TT_ESINGULAR_GRAM";
    case TT_ELINDEP: return "TT_ELINDEP";
    case TT_ENUMDEFECT: return "TT_ENUMDEFECT";
    case TT_ENOTSUP: return "TT_ENOTSUP";
    case TT_ECOMM: return "TT_ECOMM";
  }
  return "unknown";
}

int64_t tt_ctx_launch_count(tt_ctx ctx) { return ctx ? ctx->launches : -1; }

tt_status tt_ctx_sync(tt_ctx ctx) {
  return guarded(ctx, [&] { TTB_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

tt_status tt_ctx_profile(tt_ctx ctx, int32_t enable) {
  if (!ctx) return TT_EINVAL;
  return guarded(ctx, [&] {
    if (enable) prof_reset(ctx);
    else prof_resolve(ctx);
    ctx->prof = enable != 0;
  });
}

tt_status tt_ctx_profile_query(tt_ctx ctx, int32_t idx, char* name_buf, int32_t name_len, int64_t* launches,
                               double* ms, double* flops, double* bytes) {
  if (!ctx) return TT_EINVAL;
  return guarded(ctx, [&] {
    prof_resolve(ctx);
    if (idx < 0 || idx >= (int32_t)ctx->prof_cls.size()) fail(TT_EINDEX, "no such profile class");
    const TTProfEntry& e = ctx->prof_cls[(size_t)idx];
    if (name_buf && name_len > 0) {
      std::strncpy(name_buf, e.name.c_str(), (size_t)name_len - 1);
      name_buf[name_len - 1] = 0;
    }
    if (launches) *launches = e.launches;
    if (ms) *ms = e.ms;
    if (flops) *flops = e.flops;
    if (bytes) *bytes = e.bytes;
  });
}

tt_status tt_tensor_view(tt_tensor t, tt_view* out) {
  if (!t || !out) return TT_EINVAL;
  out->d = t->d;
  out->n = t->n.data();
  out->r = t->r.data();
  out->core = t->core_c.data();
  out->norm = t->norm;
  return TT_OK;
}

tt_status tt_tensor_free(tt_ctx ctx, tt_tensor t) {
  if (!ctx) return TT_EINVAL;
  if (!t) return TT_OK;
  tensor_free(ctx, t);
  return TT_OK;
}

tt_status tt_upload(tt_ctx ctx, const tt_view* host, tt_tensor* out) {
  if (!ctx || !host || !out) return TT_EINVAL;
  return guarded(ctx, [&] {
    TTShape s = view_shape(*host);
    tt_tensor t = tensor_alloc(ctx, s.d, s.n, s.r);
    for (int k = 0; k < s.d; ++k)
      TTB_CUDA(cudaMemcpyAsync(t->core[(size_t)k], host->core[k], sizeof(double) * (size_t)(s.r[k] * s.n[k] * s.r[k + 1]),
                               cudaMemcpyHostToDevice, ctx->stream));
    t->norm = host->norm;
    *out = t;
  });
}

tt_status tt_download(tt_ctx ctx, tt_tensor t, double* const* host_cores) {
  if (!ctx || !t || !host_cores) return TT_EINVAL;
  return guarded(ctx, [&] {
    for (int k = 0; k < t->d; ++k)
      TTB_CUDA(cudaMemcpyAsync(host_cores[k], t->core[(size_t)k],
                               sizeof(double) * (size_t)(t->r[(size_t)k] * t->n[(size_t)k] * t->r[(size_t)k + 1]),
                               cudaMemcpyDeviceToHost, ctx->stream));
    TTB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

tt_status tt_sum(tt_ctx ctx, int32_t K, const double* coeff, const tt_view* terms, tt_tensor* out) {
  if (!ctx || !out) return TT_EINVAL;
  return guarded(ctx, [&] { *out = materialise_sum(ctx, sum_of(K, coeff, terms)); });
}

tt_status tt_axpy(tt_ctx ctx, double alpha, const tt_view* x, const tt_view* y, tt_tensor* out) {
  if (!ctx || !x || !y || !out) return TT_EINVAL;
  tt_view t[2] = {*x, *y};
  double c[2] = {alpha, 1.0};
  return tt_sum(ctx, 2, c, t, out);
}

tt_status tt_matvec(tt_ctx ctx, const tt_view* A, const tt_view* x, tt_tensor* out) {
  if (!ctx || !A || !x || !out) return TT_EINVAL;
  return guarded(ctx, [&] {
    TTShape sa = view_shape(*A), sx = view_shape(*x);
    if (sa.d != sx.d) fail(TT_ESHAPE, "tt_matvec: operator and vector orders differ");
    for (int k = 0; k < sx.d; ++k)
      if (sa.n[(size_t)k] != sx.n[(size_t)k] * sx.n[(size_t)k])
        fail(TT_ESHAPE, "tt_matvec: operator core k must have n_k^2 modes (n_k x n_k blocks)");
    std::vector<const double*> ac(A->core, A->core + A->d), xc(x->core, x->core + x->d);
    *out = matvec(ctx, sx.d, sx.n, sa.r, ac, sx.r, xc);
  });
}

tt_status tt_dot_batch(tt_ctx ctx, int32_t P, const tt_view* x, const tt_view* y, double* out_dev) {
  if (!ctx || P < 0 || (P > 0 && (!x || !y || !out_dev))) return TT_EINVAL;
  return guarded(ctx, [&] {
    std::vector<TTRef> X, Y;
    for (int p = 0; p < P; ++p) { X.push_back(TTRef::of(x[p])); Y.push_back(TTRef::of(y[p])); }
    std::vector<std::pair<const TTRef*, const TTRef*>> pr;
    for (int p = 0; p < P; ++p) pr.push_back({&X[(size_t)p], &Y[(size_t)p]});
    dots_device(ctx, pr, out_dev);
  });
}

tt_status tt_gram_blocks(tt_ctx ctx, int32_t m, const tt_view* a, int32_t nblk, const int32_t* blk, double* packed_dev) {
  if (!ctx || m < 1 || !a || nblk < 0 || (nblk > 0 && (!blk || !packed_dev))) return TT_EINVAL;
  return guarded(ctx, [&] {
    std::vector<TTRef> A;
    for (int i = 0; i < m; ++i) A.push_back(TTRef::of(a[i]));
    gram_blocks_local(ctx, A, nblk, blk, packed_dev);
  });
}

}  // extern "C"

namespace {
__global__ void gram_unpack_kernel(const double* __restrict__ packed, int m, double* G) {
  // packed holds the lower triangle row by row (i >= j)
  const int64_t total = (int64_t)m * (m + 1) / 2;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) / 2.0);
    int ii = i;
    while ((int64_t)ii * (ii + 1) / 2 > t) --ii;
    while ((int64_t)(ii + 1) * (ii + 2) / 2 <= t) ++ii;
    const int j = (int)(t - (int64_t)ii * (ii + 1) / 2);
    const double v = packed[t];
    G[(int64_t)ii * m + j] = v;
    G[(int64_t)j * m + ii] = v;
  }
}
}  // namespace

extern "C" {

tt_status tt_gram(tt_ctx ctx, int32_t m, const tt_view* a, double* G_dev) {
  if (!ctx || m < 1 || !a || !G_dev) return TT_EINVAL;
  return guarded(ctx, [&] {
    std::vector<TTRef> A;
    for (int i = 0; i < m; ++i) A.push_back(TTRef::of(a[i]));
    if (comm_active(ctx)) {
      gram_sharded(ctx, A, G_dev);
      return;
    }
    bool uniform = true;
    for (int i = 1; i < m; ++i)
      uniform = uniform && A[(size_t)i].d == A[0].d && A[(size_t)i].n == A[0].n && A[(size_t)i].r == A[0].r;
    const char* gt = std::getenv("TT_B200_GRAM_PAIRWISE");  // tests: force the per-pair kernel
    if (uniform && !(gt && gt[0] == '1')) {
      std::vector<const double*> cores;
      for (int i = 0; i < m; ++i) cores.insert(cores.end(), A[(size_t)i].core.begin(), A[(size_t)i].core.end());
      if (gram_tiled_supported(cores, m, A[0].d, A[0].n, A[0].r)) {
        gram_tiled(ctx, cores, m, A[0].d, A[0].n, A[0].r, G_dev);
        return;
      }
    }
    std::vector<std::pair<const TTRef*, const TTRef*>> pr;
    for (int i = 0; i < m; ++i)
      for (int j = 0; j <= i; ++j) pr.push_back({&A[(size_t)i], &A[(size_t)j]});
    DBuf packed(ctx, pr.size());
    dots_device(ctx, pr, packed.p);
    const int blocks = (int)std::min<int64_t>(ceil_div((int64_t)pr.size(), 256), 1024);
    TTB_RUN(ctx, "aux", 0, 16.0 * pr.size(), gram_unpack_kernel<<<blocks, 256, 0, ctx->stream>>>(packed.p, m, G_dev));
  });
}

tt_status tt_element(tt_ctx ctx, const tt_view* x, int32_t nidx, const int64_t* lin_idx, double* out_dev) {
  if (!ctx || !x || nidx < 0 || (nidx > 0 && (!lin_idx || !out_dev))) return TT_EINVAL;
  return guarded(ctx, [&] {
    TTRef t = TTRef::of(*x);
    int64_t total = 1;  // prod(n), saturated
    for (int64_t v : t.n) total = (total > INT64_MAX / v) ? INT64_MAX : total * v;
    std::vector<int64_t> idx;
    for (int q = 0; q < nidx; ++q) {
      const int64_t l = lin_idx[q];
      if (l < 1 || l > total) fail(TT_EINDEX, "element index out of range 1..prod(n) (SPEC.md:145)");
      int64_t rem = l - 1;
      for (int k = 0; k < t.d; ++k) { idx.push_back(rem % t.n[(size_t)k]); rem /= t.n[(size_t)k]; }
    }
    elements(ctx, t.d, t.n, t.core, t.r, idx, nidx, out_dev);
  });
}

tt_status tt_norm(tt_ctx ctx, const tt_view* x, double* out_host) {
  if (!ctx || !x || !out_host) return TT_EINVAL;
  return guarded(ctx, [&] {
    double c = 1.0;
    *out_host = sweep_norm(ctx, sum_of(1, &c, x));
  });
}

tt_status tt_round(tt_ctx ctx, int32_t K, const double* coeff, const tt_view* terms, const tt_round_opts* opts,
                   tt_tensor* out, tt_round_info* info) {
  if (!ctx || !out) return TT_EINVAL;
  return guarded(ctx, [&] { *out = round_sum(ctx, sum_of(K, coeff, terms), resolve(opts), info); });
}

tt_status tt_round_batch(tt_ctx ctx, int32_t B, const int32_t* K, const double* const* coeff,
                         const tt_view* const* terms, const tt_round_opts* opts, tt_tensor* out, int64_t* ranks_out) {
  if (!ctx || B < 0 || (B > 0 && (!K || !coeff || !terms || !out))) return TT_EINVAL;
  return guarded(ctx, [&] {
    const tt_round_opts o = resolve(opts);
    std::vector<SumInput> items;
    items.reserve((size_t)B);
    for (int b = 0; b < B; ++b) items.push_back(sum_of(K[b], coeff[b], terms[b]));
    if (B == 0) return;
    // uniform batches (C4) run the one-CTA-per-item batched engine; TT_B200_BATCH_SERIAL=1
    // forces the per-item path (used by the tests to compare the two).
    const char* ser = std::getenv("TT_B200_BATCH_SERIAL");
    if (!(ser && ser[0] == '1') && batch_uniform_supported(B, items, nullptr)) {
      round_batch_uniform(ctx, items, o, out, ranks_out);
      TTB_CUDA(cudaStreamSynchronize(ctx->stream));  // results valid for any stream (header)
      return;
    }
    int done = 0;
    try {
      for (int b = 0; b < B; ++b) {
        out[b] = round_sum(ctx, items[(size_t)b], o, nullptr);
        if (ranks_out) std::memcpy(ranks_out + (size_t)b * (out[b]->d + 1), out[b]->r.data(), sizeof(int64_t) * (out[b]->d + 1));
        ++done;
      }
    } catch (...) {
      for (int b = 0; b < done; ++b) { tensor_free(ctx, out[b]); out[b] = nullptr; }
      throw;
    }
  });
}

tt_status tt_round_batch_strided(tt_ctx ctx, int32_t B, int32_t K, int32_t d, const int64_t* n, const int64_t* r,
                                 const double* const* core, const int64_t* item_stride, const double* coeff,
                                 const double* norms, const tt_round_opts* opts, tt_batch* out) {
  if (!ctx || !out || B < 0 || K < 1 || d < 1 || !n || !r || !core || !item_stride || (B > 0 && !coeff))
    return TT_EINVAL;
  return guarded(ctx, [&] {
    BatchDesc in;
    batch_desc_shape(in, B, K, d, n, r);
    for (int q = 0; q < K * d; ++q)
      if (!core[q]) fail(TT_EINVAL, "null core base pointer");
    in.tab.resize((size_t)B * K * d);
    for (int64_t b = 0; b < B; ++b)
      for (int l = 0; l < K; ++l)
        for (int k = 0; k < d; ++k) {
          const size_t q = (size_t)l * d + k;
          in.tab[((size_t)b * K + l) * d + k] = core[q] + b * item_stride[q];
        }
    in.coef.assign(coeff, coeff + (size_t)B * K);
    if (norms) in.norm.assign(norms, norms + (size_t)B * K);
    else in.norm.assign((size_t)B * K, NAN);
    tt_batch bt = new tt_batch_s();
    try {
      if (B > 0) run_batch(ctx, in, resolve(opts), bt->res);
      else { bt->res.d = d; bt->res.n = in.n; }
      // the result arenas are filled by the compaction queued last: synchronise so the
      // handle's pointers are valid for any stream (include/tt_b200.h)
      TTB_CUDA(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
      delete bt;
      throw;
    }
    *out = bt;
  });
}

tt_status tt_batch_shape(tt_batch bt, int32_t* B, int32_t* d) {
  if (!bt) return TT_EINVAL;
  if (B) *B = bt->res.B;
  if (d) *d = bt->res.d;
  return TT_OK;
}

tt_status tt_batch_ranks(tt_batch bt, int64_t* ranks, double* norms) {
  if (!bt) return TT_EINVAL;
  if (ranks) std::memcpy(ranks, bt->res.ranks.data(), sizeof(int64_t) * bt->res.ranks.size());
  if (norms) std::memcpy(norms, bt->res.norm.data(), sizeof(double) * bt->res.norm.size());
  return TT_OK;
}

tt_status tt_batch_view(tt_batch bt, int32_t b, tt_view* out) {
  if (!bt || !out) return TT_EINVAL;
  if (b < 0 || b >= bt->res.B) return TT_EINDEX;
  const int d = bt->res.d;
  out->d = d;
  out->n = bt->res.n.data();
  out->r = bt->res.ranks.data() + (size_t)b * (d + 1);
  out->core = const_cast<const double* const*>(bt->res.core.data() + (size_t)b * d);
  out->norm = bt->res.norm[(size_t)b];
  return TT_OK;
}

tt_status tt_batch_download(tt_ctx ctx, tt_batch bt, double* host, int64_t capacity, int64_t* count) {
  if (!ctx || !bt || (!host && capacity > 0)) return TT_EINVAL;
  return guarded(ctx, [&] {
    int64_t tot = 0;
    for (int64_t a : bt->res.arena_size) tot += a;
    if (count) *count = tot;
    if (tot > capacity) fail(TT_EINVAL, "tt_batch_download: host buffer too small");
    int64_t off = 0;
    for (size_t w = 0; w < bt->res.arenas.size(); ++w) {
      TTB_CUDA(cudaMemcpyAsync(host + off, bt->res.arenas[w], sizeof(double) * (size_t)bt->res.arena_size[w],
                               cudaMemcpyDeviceToHost, ctx->stream));
      off += bt->res.arena_size[w];
    }
    TTB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

tt_status tt_batch_arena(tt_batch bt, int32_t w, const double** ptr, int64_t* count) {
  if (!bt || !ptr || !count) return TT_EINVAL;
  if (w < 0 || (size_t)w >= bt->res.arenas.size()) return TT_EINDEX;
  *ptr = static_cast<const double*>(bt->res.arenas[(size_t)w]);
  *count = bt->res.arena_size[(size_t)w];
  return TT_OK;
}

tt_status tt_batch_free(tt_ctx ctx, tt_batch bt) {
  if (!ctx) return TT_EINVAL;
  if (!bt) return TT_OK;
  for (void* p : bt->res.arenas) cudaFreeAsync(p, ctx->stream);
  delete bt;
  return TT_OK;
}

tt_status tt_ctx_round_hook(tt_ctx ctx, tt_round_hook fn, void* user) {
  if (!ctx) return TT_EINVAL;
  ctx->round_hook = fn;
  ctx->round_hook_user = user;
  return TT_OK;
}

tt_status tt_orth(tt_ctx ctx, tt_orth_kind kind, int32_t m, const tt_view* a, const tt_orth_opts* opts,
                  tt_tensor* q_out, double* R_host, tt_orth_report* report) {
  if (!ctx) return TT_EINVAL;
  tt_orth_opts o;
  if (opts) o = *opts;
  else { o.round = default_round_opts(); o.hh_beta_literal = 0; o.want_loo = 0; o.hh_mask = 0; }
  return guarded(ctx, [&] { orth_run(ctx, kind, m, a, o, q_out, R_host, report); });
}

}  // extern "C"
