// Communicator held by a context (comm.cu) and the host-side shard plans.
#pragma once
#include <vector>

#include "common.cuh"

struct TTComm {
  int nranks = 1, rank = 0;
  void* nccl = nullptr;  // ncclComm_t (NCCL loaded with dlopen at attach time)
  tt_comm_ops ops{};     // caller-supplied collectives (when nccl is null)
};

namespace ttb {

// true when a communicator is attached (of any size: one rank runs the sharded code path too)
bool comm_active(tt_ctx ctx);
int comm_rank(tt_ctx ctx);
int comm_size(tt_ctx ctx);
// All-gather `bytes` from every rank: recv (DEVICE, nranks * bytes) in rank order.  Ordered on the
// ctx stream (NCCL) or complete on return (caller-supplied ops; the ctx stream is synchronised
// before the callback runs).
void comm_allgather(tt_ctx ctx, const void* send_dev, void* recv_dev, size_t bytes);
// Broadcasts of several device buffers, buffer q from rank root[q] (grouped into one NCCL launch).
void comm_broadcast_many(tt_ctx ctx, const std::vector<void*>& bufs, const std::vector<size_t>& bytes,
                         const std::vector<int>& root);
void comm_release(tt_ctx ctx);

// ---------------------------------------------------------------- plans (host only, no device)
// Contiguous balanced slice [*s, *e) of P items for `rank` of `nranks`.
void plan_slice(int64_t P, int nranks, int rank, int64_t* s, int64_t* e);
// Longest-processing-time assignment: items in decreasing cost (ties: lower index first) go to
// the least-loaded rank (ties: lower rank).  Deterministic, so every rank computes the same map.
std::vector<int> plan_lpt(const std::vector<double>& cost, int nranks);
// b x b blocks (i0, j0, bi, bj) covering every pair i >= j of an m x m Gram matrix exactly once
// (diagonal blocks are full squares; their upper half is redundant and ignored on unpack).
std::vector<int32_t> plan_gram_blocks(int m, int b);

}  // namespace ttb
