// Context-held communicator for the naturally sharded parts of the hot path (
// north star: "Gram-matrix and CGS projection dot products are split by pair blocks and combined
// with NCCL all-gather over NVLink, and batches of independent roundings are split across GPUs").
//
// Two transports behind one interface:
//   * NCCL, owned by the library: tt_comm_nccl_id on one rank, the 128-byte id passed to every
//     rank (any out-of-band channel), tt_ctx_comm_nccl on every rank.  libnccl.so.2 is loaded with
//     dlopen at that point (the one torch already loaded, when it did), so the library has no
//     link-time NCCL dependency and single-GPU users never load it.
//   * caller-supplied collectives (tt_comm_ops): used by the tests to run two ranks that exchange
//     through the host (gloo), and by callers with their own transport.
// The collectives move only small metadata and dot values, plus one broadcast of each phase-2
// rounding result from its owner; a single rounding sweep never crosses a process.
#include <dlfcn.h>
#include <nccl.h>  // types only: the symbols are resolved from the dlopen'ed library

#include <algorithm>
#include <cstring>
#include <mutex>

#include "comm.cuh"

namespace ttb {

namespace {

struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) {
      const char* e = dlerror();
      api.err = std::string("cannot load libnccl.so.2: ") + (e ? e : "unknown");
      return;
    }
    auto sym = [&](const char* s) { return dlsym(h, s); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather && api.Broadcast &&
             api.GroupStart && api.GroupEnd && api.GetErrorString;
    if (!api.ok) api.err = "libnccl.so.2 lacks an expected symbol";
  });
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  fail(TT_ECOMM, std::string(what) + " failed: " + nccl_api().GetErrorString(r));
}

}  // namespace

bool comm_active(tt_ctx ctx) { return ctx->comm != nullptr; }
int comm_rank(tt_ctx ctx) { return ctx->comm ? ctx->comm->rank : 0; }
int comm_size(tt_ctx ctx) { return ctx->comm ? ctx->comm->nranks : 1; }

void comm_allgather(tt_ctx ctx, const void* send_dev, void* recv_dev, size_t bytes) {
  TTComm* c = ctx->comm;
  if (!c || (c->nranks == 1 && !c->nccl)) {
    if (send_dev != recv_dev && bytes)
      TTB_CUDA(cudaMemcpyAsync(recv_dev, send_dev, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
    return;
  }
  if (c->nccl) {
    nccl_check(nccl_api().AllGather(send_dev, recv_dev, bytes, ncclUint8, static_cast<ncclComm_t>(c->nccl), ctx->stream),
               "ncclAllGather");
    return;
  }
  TTB_CUDA(cudaStreamSynchronize(ctx->stream));
  if (c->ops.allgather(c->ops.user, send_dev, recv_dev, bytes, ctx->stream) != 0)
    fail(TT_ECOMM, "caller-supplied all-gather failed");
}

void comm_broadcast_many(tt_ctx ctx, const std::vector<void*>& bufs, const std::vector<size_t>& bytes,
                         const std::vector<int>& root) {
  TTComm* c = ctx->comm;
  if (!c || (c->nranks == 1 && !c->nccl) || bufs.empty()) return;
  if (c->nccl) {
    NcclApi& api = nccl_api();
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (size_t q = 0; q < bufs.size(); ++q)
      nccl_check(api.Broadcast(bufs[q], bufs[q], bytes[q], ncclUint8, root[q], static_cast<ncclComm_t>(c->nccl),
                               ctx->stream),
                 "ncclBroadcast");
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
    return;
  }
  TTB_CUDA(cudaStreamSynchronize(ctx->stream));
  for (size_t q = 0; q < bufs.size(); ++q)
    if (c->ops.broadcast(c->ops.user, bufs[q], bytes[q], root[q], ctx->stream) != 0)
      fail(TT_ECOMM, "caller-supplied broadcast failed");
}

void comm_release(tt_ctx ctx) {
  if (!ctx->comm) return;
  if (ctx->comm->nccl && nccl_api().ok) nccl_api().CommDestroy(static_cast<ncclComm_t>(ctx->comm->nccl));
  delete ctx->comm;
  ctx->comm = nullptr;
}

void plan_slice(int64_t P, int nranks, int rank, int64_t* s, int64_t* e) {
  const int64_t base = P / nranks, rem = P % nranks;
  *s = rank * base + std::min<int64_t>(rank, rem);
  *e = *s + base + (rank < rem ? 1 : 0);
}

std::vector<int> plan_lpt(const std::vector<double>& cost, int nranks) {
  std::vector<int> order(cost.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[(size_t)a] > cost[(size_t)b]; });
  std::vector<double> load((size_t)nranks, 0.0);
  std::vector<int> owner(cost.size(), 0);
  for (int i : order) {
    int best = 0;
    for (int q = 1; q < nranks; ++q)
      if (load[(size_t)q] < load[(size_t)best]) best = q;
    owner[(size_t)i] = best;
    load[(size_t)best] += cost[(size_t)i];
  }
  return owner;
}

std::vector<int32_t> plan_gram_blocks(int m, int b) {
  std::vector<int32_t> blk;
  if (b < 1) b = 1;
  for (int I = 0; I < m; I += b)
    for (int J = 0; J <= I; J += b) blk.insert(blk.end(), {I, J, std::min(b, m - I), std::min(b, m - J)});
  return blk;
}

}  // namespace ttb

using namespace ttb;

namespace {
template <typename F>
tt_status guard(tt_ctx ctx, F f) {
  try {
    f();
    return TT_OK;
  } catch (const Error& e) {
    if (ctx) ctx->last_error = e.msg;
    return e.status;
  } catch (const std::exception& e) {
    if (ctx) ctx->last_error = e.what();
    return TT_EINVAL;
  }
}
}  // namespace

extern "C" {

tt_status tt_comm_nccl_id(uint8_t* id) {
  if (!id) return TT_EINVAL;
  NcclApi& api = nccl_api();
  if (!api.ok) return TT_ECOMM;
  ncclUniqueId u;
  if (api.GetUniqueId(&u) != ncclSuccess) return TT_ECOMM;
  static_assert(sizeof(ncclUniqueId) == TT_COMM_ID_BYTES, "ncclUniqueId size");
  std::memcpy(id, &u, sizeof(u));
  return TT_OK;
}

tt_status tt_ctx_comm_nccl(tt_ctx ctx, int32_t nranks, int32_t rank, const uint8_t* id) {
  if (!ctx || nranks < 1 || rank < 0 || rank >= nranks || !id) return TT_EINVAL;
  return guard(ctx, [&] {
    NcclApi& api = nccl_api();
    if (!api.ok) fail(TT_ECOMM, api.err);
    comm_release(ctx);
    TTB_CUDA(cudaSetDevice(ctx->device));
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    ncclComm_t comm = nullptr;
    nccl_check(api.CommInitRank(&comm, nranks, u, rank), "ncclCommInitRank");
    ctx->comm = new TTComm();
    ctx->comm->nranks = nranks;
    ctx->comm->rank = rank;
    ctx->comm->nccl = comm;
  });
}

tt_status tt_ctx_comm_ops(tt_ctx ctx, int32_t nranks, int32_t rank, const tt_comm_ops* ops) {
  if (!ctx || nranks < 1 || rank < 0 || rank >= nranks || !ops || !ops->allgather || !ops->broadcast) return TT_EINVAL;
  return guard(ctx, [&] {
    comm_release(ctx);
    ctx->comm = new TTComm();
    ctx->comm->nranks = nranks;
    ctx->comm->rank = rank;
    ctx->comm->ops = *ops;
  });
}

tt_status tt_ctx_comm_detach(tt_ctx ctx) {
  if (!ctx) return TT_EINVAL;
  return guard(ctx, [&] {
    TTB_CUDA(cudaStreamSynchronize(ctx->stream));
    comm_release(ctx);
  });
}

tt_status tt_ctx_comm_info(tt_ctx ctx, int32_t* nranks, int32_t* rank) {
  if (!ctx) return TT_EINVAL;
  if (nranks) *nranks = comm_size(ctx);
  if (rank) *rank = comm_rank(ctx);
  return TT_OK;
}

tt_status tt_plan_slice(int64_t P, int32_t nranks, int32_t rank, int64_t* start, int64_t* end) {
  if (P < 0 || nranks < 1 || rank < 0 || rank >= nranks || !start || !end) return TT_EINVAL;
  plan_slice(P, nranks, rank, start, end);
  return TT_OK;
}

tt_status tt_plan_lpt(int32_t P, const double* cost, int32_t nranks, int32_t* owner) {
  if (P < 0 || nranks < 1 || (P > 0 && (!cost || !owner))) return TT_EINVAL;
  std::vector<int> o = plan_lpt(std::vector<double>(cost, cost + P), nranks);
  for (int i = 0; i < P; ++i) owner[i] = o[(size_t)i];
  return TT_OK;
}

tt_status tt_plan_gram_blocks(int32_t m, int32_t b, int32_t nranks, int32_t cap, int32_t* blk, int32_t* owner,
                              int32_t* nblk) {
  if (m < 1 || b < 1 || nranks < 1 || !nblk || cap < 0 || (cap > 0 && (!blk || !owner))) return TT_EINVAL;
  std::vector<int32_t> bl = plan_gram_blocks(m, b);
  const int nb = (int)(bl.size() / 4);
  *nblk = nb;
  if (nb > cap) return cap == 0 ? TT_OK : TT_EINVAL;
  std::vector<double> cost((size_t)nb);
  for (int q = 0; q < nb; ++q) cost[(size_t)q] = (double)bl[(size_t)4 * q + 2] * bl[(size_t)4 * q + 3];
  std::vector<int> o = plan_lpt(cost, nranks);
  std::memcpy(blk, bl.data(), sizeof(int32_t) * bl.size());
  for (int q = 0; q < nb; ++q) owner[q] = o[(size_t)q];
  return TT_OK;
}

}  // extern "C"
