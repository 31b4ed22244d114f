// Orthogonalization drivers (PAPER.md Algs. 1-8) on top of the GPU TT-rounding and
// TT-dot kernels.  Running TT-sums are kept as coefficients over stored tensors and
// materialised (rounded) only at the paper's rounding points; the counts are exactly
// Table 1's (m, m, 2m, 2m, m, 4m-1).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>

#include "comm.cuh"
#include "gram.cuh"
#include "orth.cuh"
#include "ttops.cuh"

namespace ttb {

TTRef TTRef::of(const tt_view& v) {
  TTShape s = view_shape(v);
  TTRef t;
  t.d = s.d;
  t.n = s.n;
  t.r = s.r;
  t.core.assign(v.core, v.core + v.d);
  t.norm = v.norm;
  return t;
}

TTRef TTRef::of(tt_tensor x) {
  TTRef t;
  t.d = x->d;
  t.n = x->n;
  t.r = x->r;
  t.core = x->core_c;
  t.norm = x->norm;
  return t;
}

namespace {

// Operands with one rank profile per side (all first operands alike, all second operands alike;
// 16-byte aligned cores): the pairs become row / column blocks of a Gram matrix between the
// distinct first and the distinct second operands and run on the pair-tiled DMMA Gram kernel
// (gram.cu), which stages each mode slice once per tile -- the drivers' dot batches are one
// vector against a set (CGS/CGS2 projections, MGS rows).  Output in pair order.
bool dots_gram(tt_ctx ctx, const std::vector<std::pair<const TTRef*, const TTRef*>>& pairs, double* out_dev) {
  const TTRef& fa = *pairs[0].first;
  const TTRef& fb = *pairs[0].second;
  std::vector<const TTRef*> ua, ub;  // distinct first / second operands
  std::vector<int> ix(pairs.size()), iy(pairs.size());
  auto id_of = [](std::vector<const TTRef*>& u, const TTRef* t) -> int {
    for (size_t k = 0; k < u.size(); ++k)
      if (u[k] == t || u[k]->core == t->core) return (int)k;
    u.push_back(t);
    return (int)u.size() - 1;
  };
  for (size_t q = 0; q < pairs.size(); ++q) {
    const TTRef* a = pairs[q].first;
    const TTRef* b = pairs[q].second;
    if (a->d != fa.d || a->n != fa.n || a->r != fa.r) return false;
    if (b->d != fb.d || b->n != fb.n || b->r != fb.r) return false;
    ix[q] = id_of(ua, a);
    iy[q] = id_of(ub, b);
  }
  if (fa.d != fb.d || fa.n != fb.n) return false;
  std::vector<const double*> cores;
  for (const TTRef* t : ua) cores.insert(cores.end(), t->core.begin(), t->core.end());
  for (const TTRef* t : ub) cores.insert(cores.end(), t->core.begin(), t->core.end());
  const int na = (int)ua.size(), m = na + (int)ub.size();
  std::vector<int64_t> rmax(fa.r.size());
  for (size_t k = 0; k < rmax.size(); ++k) rmax[k] = std::max(fa.r[k], fb.r[k]);
  if (!gram_tiled_supported(cores, m, fa.d, fa.n, rmax)) return false;
  std::vector<int32_t> blk;
  for (size_t q = 0; q < pairs.size();) {
    size_t e = q + 1;
    while (e < pairs.size() && ix[e] == ix[q] && iy[e] == iy[e - 1] + 1) ++e;  // row block
    if (e - q > 1) {
      blk.insert(blk.end(), {ix[q], na + iy[q], 1, (int32_t)(e - q)});
    } else {
      while (e < pairs.size() && iy[e] == iy[q] && ix[e] == ix[e - 1] + 1) ++e;  // column block
      blk.insert(blk.end(), {ix[q], na + iy[q], (int32_t)(e - q), 1});
    }
    q = e;
  }
  gram_tiled_blocks(ctx, cores, m, fa.d, fa.n, fa.r, (int)(blk.size() / 4), blk.data(), out_dev, &fb.r);
  return true;
}

}  // namespace

void dots_device(tt_ctx ctx, const std::vector<std::pair<const TTRef*, const TTRef*>>& pairs, double* out_dev) {
  if (pairs.empty()) return;
  static const bool pairwise = std::getenv("TT_B200_DOT_PAIRWISE") != nullptr;
  if (!pairwise && dots_gram(ctx, pairs, out_dev)) return;
  DotBatch b;
  b.d = pairs[0].first->d;
  b.n = pairs[0].first->n;
  b.P = (int)pairs.size();
  for (auto& pr : pairs) {
    const TTRef& x = *pr.first;
    const TTRef& y = *pr.second;
    if (x.d != b.d || y.d != b.d || x.n != b.n || y.n != b.n) fail(TT_ESHAPE, "TT-dot operands differ in shape");
    b.xc.insert(b.xc.end(), x.core.begin(), x.core.end());
    b.yc.insert(b.yc.end(), y.core.begin(), y.core.end());
    b.xr.insert(b.xr.end(), x.r.begin(), x.r.end());
    b.yr.insert(b.yr.end(), y.r.begin(), y.r.end());
  }
  dot_batch(ctx, b, out_dev);  // ranks > 32: grouped DMMA GEMMs per core
}

std::vector<double> dots_host(tt_ctx ctx, const std::vector<std::pair<const TTRef*, const TTRef*>>& pairs) {
  std::vector<double> h(pairs.size(), 0.0);
  if (pairs.empty()) return h;
  if (comm_active(ctx) && pairs.size() >= 2) {
    // split into contiguous slices (one per rank), one all-gather of equal-sized buffers
    // (north star: "CGS projection dot products are split ... and combined with all-gather")
    const int N = comm_size(ctx), me = comm_rank(ctx);
    const int64_t P = (int64_t)pairs.size(), cap = ceil_div(P, N);
    int64_t s = 0, e = 0;
    plan_slice(P, N, me, &s, &e);
    DBuf send(ctx, (size_t)cap), recv(ctx, (size_t)cap * N);
    if (e > s)
      dots_device(ctx, std::vector<std::pair<const TTRef*, const TTRef*>>(pairs.begin() + s, pairs.begin() + e), send.p);
    comm_allgather(ctx, send.p, recv.p, sizeof(double) * (size_t)cap);
    std::vector<double> all((size_t)cap * N);
    d2h_small(ctx, all.data(), recv.p, all.size());
    for (int q = 0; q < N; ++q) {
      int64_t a = 0, b = 0;
      plan_slice(P, N, q, &a, &b);
      for (int64_t t = a; t < b; ++t) h[(size_t)t] = all[(size_t)q * cap + (t - a)];
    }
    return h;
  }
  DBuf o(ctx, pairs.size());
  dots_device(ctx, pairs, o.p);
  d2h_small(ctx, h.data(), o.p, pairs.size());
  return h;
}

int cholesky_host(std::vector<double>& G, int m) {
  // symmetrise, then L in the lower triangle (row-major)
  std::vector<double> L((size_t)m * m, 0.0);
  for (int j = 0; j < m; ++j) {
    double s = 0.5 * (G[(size_t)j * m + j] + G[(size_t)j * m + j]);
    for (int k = 0; k < j; ++k) s -= L[(size_t)j * m + k] * L[(size_t)j * m + k];
    if (!(s > 0.0)) return j;
    L[(size_t)j * m + j] = std::sqrt(s);
    for (int i = j + 1; i < m; ++i) {
      double t = 0.5 * (G[(size_t)i * m + j] + G[(size_t)j * m + i]);
      for (int k = 0; k < j; ++k) t -= L[(size_t)i * m + k] * L[(size_t)j * m + k];
      L[(size_t)i * m + j] = t / L[(size_t)j * m + j];
    }
  }
  G = L;
  return -1;
}

// eigenvalues of a small symmetric matrix by cyclic Jacobi (host)
static std::vector<double> sym_eig(std::vector<double> A, int n) {
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        tot += A[(size_t)i * n + j] * A[(size_t)i * n + j];
        if (i != j) off += A[(size_t)i * n + j] * A[(size_t)i * n + j];
      }
    if (off <= 1e-36 * tot || off == 0.0) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A[(size_t)p * n + q];
        if (apq == 0.0) continue;
        const double app = A[(size_t)p * n + p], aqq = A[(size_t)q * n + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::hypot(1.0, theta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double akp = A[(size_t)k * n + p], akq = A[(size_t)k * n + q];
          A[(size_t)k * n + p] = c * akp - s * akq;
          A[(size_t)k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = A[(size_t)p * n + k], aqk = A[(size_t)q * n + k];
          A[(size_t)p * n + k] = c * apk - s * aqk;
          A[(size_t)q * n + k] = s * apk + c * aqk;
        }
      }
  }
  std::vector<double> ev((size_t)n);
  for (int i = 0; i < n; ++i) ev[(size_t)i] = A[(size_t)i * n + i];
  return ev;
}

double loo_host(const std::vector<double>& Gq, int m, int k) {
  // ||I_k - Q_k^T Q_k||_2, Eq. (9): largest |eigenvalue| of the symmetrised defect
  std::vector<double> D((size_t)k * k);
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j)
      D[(size_t)i * k + j] = (i == j ? 1.0 : 0.0) - 0.5 * (Gq[(size_t)i * m + j] + Gq[(size_t)j * m + i]);
  std::vector<double> ev = sym_eig(D, k);
  double mx = 0.0;
  for (double v : ev) mx = std::max(mx, std::fabs(v));
  return mx;
}

tt_tensor make_canonical(tt_ctx ctx, const std::vector<int64_t>& n, int64_t lin1) {
  const int d = (int)n.size();
  int64_t total = 1;  // prod(n), saturated (16^50 overflows int64)
  for (int64_t v : n) total = (total > INT64_MAX / v) ? INT64_MAX : total * v;
  if (lin1 < 1 || lin1 > total) fail(TT_EINDEX, "canonical index out of range (PAPER.md:337)");
  tt_tensor t = tensor_alloc(ctx, d, n, std::vector<int64_t>((size_t)d + 1, 1));
  int64_t sz = 0;
  for (int64_t v : n) sz += v;
  std::vector<double> h((size_t)sz, 0.0);
  int64_t rem = lin1 - 1, off = 0;
  for (int k = 0; k < d; ++k) {
    h[(size_t)(off + rem % n[(size_t)k])] = 1.0;
    rem /= n[(size_t)k];
    off += n[(size_t)k];
  }
  TTB_CUDA(cudaMemcpyAsync(t->block, h.data(), sizeof(double) * (size_t)sz, cudaMemcpyHostToDevice, ctx->stream));
  t->norm = 1.0;
  return t;
}

namespace {

struct Owned {  // RAII for library tensors produced inside a driver
  tt_ctx ctx;
  tt_tensor t = nullptr;
  explicit Owned(tt_ctx c, tt_tensor x = nullptr) : ctx(c), t(x) {}
  ~Owned() { if (t) tensor_free(ctx, t); }
  tt_tensor release() { tt_tensor x = t; t = nullptr; return x; }
  void reset(tt_tensor x) { if (t) tensor_free(ctx, t); t = x; }
};

double last_core_norm(tt_ctx ctx, tt_tensor t) {
  const int d = t->d;
  const int64_t n = t->r[(size_t)d - 1] * t->n[(size_t)d - 1] * t->r[(size_t)d];
  DBuf s(ctx, 1);
  sumsq(ctx, t->core[(size_t)d - 1], n, s.p);
  double h = 0.0;
  d2h_small(ctx, &h, s.p, 1);
  return std::sqrt(h);
}

void scale_last_core(tt_ctx ctx, tt_tensor t, double a) {
  const int d = t->d;
  scale_inplace(ctx, t->core[(size_t)d - 1], t->r[(size_t)d - 1] * t->n[(size_t)d - 1] * t->r[(size_t)d], a);
}

int64_t max_rank(tt_tensor t) {
  int64_t m = 1;
  for (int64_t v : t->r) m = std::max(m, v);
  return m;
}

// tt_ctx_round_hook: hand the rounding call's TT-sum to the observer (ctx stream synchronised).
void notify_round(tt_ctx ctx, int64_t call, const SumInput& in, const tt_round_opts& o) {
  if (!ctx->round_hook) return;
  TTB_CUDA(cudaStreamSynchronize(ctx->stream));
  const int K = in.K();
  std::vector<tt_view> v((size_t)K);
  for (int l = 0; l < K; ++l) {
    v[(size_t)l].d = in.d;
    v[(size_t)l].n = in.n.data();
    v[(size_t)l].r = in.r[(size_t)l].data();
    v[(size_t)l].core = in.core[(size_t)l].data();
    v[(size_t)l].norm = in.norm[(size_t)l];
  }
  ctx->round_hook(ctx->round_hook_user, call, K, in.coef.data(), v.data(), &o);
}

struct Ledger {
  int64_t calls = 0;
  std::vector<int64_t> max_ranks;
  tt_tensor round(tt_ctx ctx, const SumInput& in, const tt_round_opts& o) {
    notify_round(ctx, calls, in, o);
    tt_tensor t = round_sum(ctx, in, o, nullptr);
    ++calls;
    max_ranks.push_back(max_rank(t));
    return t;
  }
};

// Modelled flops of rounding `in` (right-to-left QR + explicit Q of the
// formal-rank panels, capped by the structural ranks): the LPT cost of a phase-2 rounding.
double round_cost_model(const SumInput& in) {
  const int d = in.d;
  std::vector<double> R((size_t)d + 1, 0.0), Rp((size_t)d + 1, 1.0);
  for (int k = 0; k <= d; ++k)
    for (const auto& r : in.r) R[(size_t)k] += (double)r[(size_t)k];
  R[0] = R[(size_t)d] = 1.0;
  for (int k = d; k >= 1; --k) Rp[(size_t)k - 1] = std::min(R[(size_t)k - 1], (double)in.n[(size_t)k - 1] * Rp[(size_t)k]);
  double f = 0.0;
  for (int k = d - 1; k >= 1; --k) {
    const double m = (double)in.n[(size_t)k] * Rp[(size_t)k + 1], c = R[(size_t)k];
    f += (m >= c) ? 4.0 * m * c * c - 4.0 * c * c * c / 3.0 : 4.0 * c * m * m - 4.0 * m * m * m / 3.0;
  }
  return f;
}

// The independent roundings of a driver's phase 2 (TT-Gram q_i; TT-Householder
// q_i).  Without a communicator they run in order.  With one, the LPT plan on
// round_cost_model assigns each to a rank; the owner rounds it and takes its norm, one all-gather
// shares every output's ranks and norm, and each q_i is broadcast from its owner (grouped), so
// every rank returns every q_i.  The ledger records the calls in index order (Table 1 counts).
std::vector<tt_tensor> round_independent(tt_ctx ctx, const std::vector<SumInput>& sums, const tt_round_opts& o,
                                         Ledger& led) {
  TTB_RANGE("tt_orth: phase-2 independent roundings");
  const int m = (int)sums.size();
  std::vector<tt_tensor> Q((size_t)m, nullptr);
  auto free_all = [&] {
    for (tt_tensor& t : Q)
      if (t) { tensor_free(ctx, t); t = nullptr; }
  };
  if (!comm_active(ctx)) {
    try {
      for (int i = 0; i < m; ++i) {
        Q[(size_t)i] = led.round(ctx, sums[(size_t)i], o);
        Q[(size_t)i]->norm = last_core_norm(ctx, Q[(size_t)i]);
      }
    } catch (...) {
      free_all();
      throw;
    }
    return Q;
  }
  const int N = comm_size(ctx), me = comm_rank(ctx), d = sums[0].d;
  std::vector<double> cost((size_t)m);
  for (int i = 0; i < m; ++i) cost[(size_t)i] = round_cost_model(sums[(size_t)i]);
  const std::vector<int> owner = plan_lpt(cost, N);
  const size_t row = (size_t)d + 2;  // ranks r_0..r_d (exact in a double) and the norm
  std::vector<double> info((size_t)m * row, 0.0);
  try {
    for (int i = 0; i < m; ++i) {
      if (owner[(size_t)i] != me) continue;
      notify_round(ctx, led.calls + i, sums[(size_t)i], o);
      tt_tensor t = round_sum(ctx, sums[(size_t)i], o, nullptr);
      Q[(size_t)i] = t;
      t->norm = last_core_norm(ctx, t);
      for (int k = 0; k <= d; ++k) info[(size_t)i * row + k] = (double)t->r[(size_t)k];
      info[(size_t)i * row + d + 1] = t->norm;
    }
    DBuf send(ctx, info.size()), recv(ctx, info.size() * N);
    TTB_CUDA(cudaMemcpyAsync(send.p, info.data(), sizeof(double) * info.size(), cudaMemcpyHostToDevice, ctx->stream));
    comm_allgather(ctx, send.p, recv.p, sizeof(double) * info.size());
    std::vector<double> all(info.size() * N);
    d2h_small(ctx, all.data(), recv.p, all.size());
    std::vector<void*> bufs;
    std::vector<size_t> bytes;
    std::vector<int> roots;
    for (int i = 0; i < m; ++i) {
      const double* g = all.data() + (size_t)owner[(size_t)i] * info.size() + (size_t)i * row;
      std::vector<int64_t> rk((size_t)d + 1);
      for (int k = 0; k <= d; ++k) rk[(size_t)k] = (int64_t)g[k];
      if (!Q[(size_t)i]) {
        Q[(size_t)i] = tensor_alloc(ctx, d, sums[(size_t)i].n, rk);
        Q[(size_t)i]->norm = g[d + 1];
      }
      size_t total = 0;
      for (int k = 0; k < d; ++k) total += (size_t)(rk[(size_t)k] * sums[(size_t)i].n[(size_t)k] * rk[(size_t)k + 1]);
      bufs.push_back(Q[(size_t)i]->block ? Q[(size_t)i]->block : Q[(size_t)i]->core[0]);  // arena items: cores contiguous
      bytes.push_back(total * sizeof(double));
      roots.push_back(owner[(size_t)i]);
      led.calls++;
      led.max_ranks.push_back(*std::max_element(rk.begin(), rk.end()));
    }
    comm_broadcast_many(ctx, bufs, bytes, roots);
  } catch (...) {
    free_all();
    throw;
  }
  return Q;
}

void add_ref(SumInput& s, const TTRef& x, double c) {
  tt_view v;
  v.d = x.d;
  v.n = x.n.data();
  v.r = x.r.data();
  v.core = x.core.data();
  v.norm = x.norm;
  s.add(v, c);
}

// TT of the indicator "psi-order linear index >= L" (0-based index, mode 1 fastest): ranks <= 2,
// states 0 = digits equal so far (from mode d down), 1 = already greater; core k's right index is
// the state before its digit, its left index the state after; core 1 accepts both states.
tt_tensor mask_geq_tt(tt_ctx ctx, const std::vector<int64_t>& n, int64_t L) {
  const int d = (int)n.size();
  std::vector<int64_t> dig((size_t)d), r((size_t)d + 1, 2);
  int64_t rem = L;
  for (int k = 0; k < d; ++k) { dig[(size_t)k] = rem % n[(size_t)k]; rem /= n[(size_t)k]; }
  r[0] = r[(size_t)d] = 1;
  tt_tensor t = tensor_alloc(ctx, d, n, r);
  std::vector<double> h;
  for (int k = 0; k < d; ++k) {
    const int64_t left = r[(size_t)k], right = r[(size_t)k + 1], nk = n[(size_t)k];
    std::vector<double> c((size_t)(left * nk * right), 0.0);
    for (int64_t sin = 0; sin < right; ++sin) {
      const int64_t state = (k == d - 1) ? 0 : sin;  // mode d starts "equal"
      for (int64_t x = 0; x < nk; ++x) {
        int64_t sout;
        if (state == 1 || x > dig[(size_t)k]) sout = 1;
        else if (x == dig[(size_t)k]) sout = 0;
        else continue;  // smaller at the most significant differing digit
        const int64_t row = (k == 0) ? 0 : sout;
        c[(size_t)((row * nk + x) * right + sin)] = 1.0;
      }
    }
    h.insert(h.end(), c.begin(), c.end());
  }
  TTB_CUDA(cudaMemcpyAsync(t->block, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, ctx->stream));
  TTB_CUDA(cudaStreamSynchronize(ctx->stream));  // h is a host temporary
  return t;
}

std::vector<int64_t> phi0(const std::vector<int64_t>& n, int64_t lin1) {
  std::vector<int64_t> idx(n.size());
  int64_t rem = lin1 - 1;
  for (size_t k = 0; k < n.size(); ++k) {
    idx[k] = rem % n[k];
    rem /= n[k];
  }
  return idx;
}

std::vector<double> elements_host(tt_ctx ctx, const TTRef& x, const std::vector<int64_t>& lins) {
  std::vector<int64_t> idx;
  for (int64_t l : lins) {
    std::vector<int64_t> v = phi0(x.n, l);
    idx.insert(idx.end(), v.begin(), v.end());
  }
  DBuf o(ctx, lins.size());
  elements(ctx, x.d, x.n, x.core, x.r, idx, (int)lins.size(), o.p);
  std::vector<double> h(lins.size());
  d2h_small(ctx, h.data(), o.p, lins.size());
  return h;
}

// ----------------------------------------------------------------- Gram-Schmidt family
void run_gs(tt_ctx ctx, tt_orth_kind kind, int m, const std::vector<TTRef>& A, const std::vector<double>& an,
            const tt_orth_opts& o, std::vector<tt_tensor>& Q, std::vector<double>& R, std::vector<double>& GQ,
            Ledger& led, int* fail_index) {
  const int passes = (kind == TT_CGS2 || kind == TT_MGS2) ? 2 : 1;
  const bool modified = (kind == TT_MGS || kind == TT_MGS2);
  std::vector<TTRef> QR;  // refs of finished q's
  for (int i = 0; i < m; ++i) {
    const std::string step_name = "tt_orth: Gram-Schmidt step " + std::to_string(i + 1);
    TTB_RANGE(step_name.c_str());
    TTRef base = A[(size_t)i];
    base.norm = an[(size_t)i];
    Owned prev(ctx);
    for (int ps = 0; ps < passes; ++ps) {
      std::vector<std::pair<const TTRef*, const TTRef*>> pr;
      for (int j = 0; j < i; ++j) pr.push_back({&base, &QR[(size_t)j]});
      std::vector<double> dbq = dots_host(ctx, pr);
      std::vector<double> c((size_t)i, 0.0);
      for (int j = 0; j < i; ++j) {
        double v = dbq[(size_t)j];
        if (modified)
          for (int l = 0; l < j; ++l) v -= c[(size_t)l] * GQ[(size_t)l * m + j];
        c[(size_t)j] = v;
        R[(size_t)j * m + i] += v;  // R = R_1 + R_2 (Algs. 3-4, last line)
      }
      SumInput s;
      add_ref(s, base, 1.0);
      for (int j = 0; j < i; ++j) add_ref(s, QR[(size_t)j], -c[(size_t)j]);
      tt_tensor p = led.round(ctx, s, o.round);
      const double pn = last_core_norm(ctx, p);
      p->norm = pn;
      prev.reset(p);
      base = TTRef::of(p);
    }
    const double nrm = base.norm;
    if (nrm <= 1e3 * U_ROUND * an[(size_t)i]) {
      *fail_index = i;
      fail(TT_ELINDEP, "linear dependence at step " + std::to_string(i) + " (SPEC.md:473)");
    }
    R[(size_t)i * m + i] = nrm;
    tt_tensor q = prev.release();
    scale_last_core(ctx, q, 1.0 / nrm);  // q_i = p / R(i,i)
    q->norm = 1.0;
    Q.push_back(q);
    QR.push_back(TTRef::of(q));
    if (modified || o.want_loo) {
      std::vector<std::pair<const TTRef*, const TTRef*>> pr;
      for (int j = 0; j <= i; ++j) pr.push_back({&QR[(size_t)j], &QR[(size_t)i]});
      std::vector<double> g = dots_host(ctx, pr);
      for (int j = 0; j <= i; ++j) GQ[(size_t)j * m + i] = GQ[(size_t)i * m + j] = g[(size_t)j];
    }
  }
}

// ----------------------------------------------------------------- Gram (Alg. 5)
void run_gram(tt_ctx ctx, int m, const std::vector<TTRef>& A, const std::vector<double>& an, const tt_orth_opts& o,
              std::vector<tt_tensor>& Q, std::vector<double>& R, Ledger& led, int* fail_index) {
  TTB_RANGE("tt_orth: TT-Gram");
  std::vector<std::pair<const TTRef*, const TTRef*>> pr;
  for (int i = 0; i < m; ++i)
    for (int j = 0; j <= i; ++j) pr.push_back({&A[(size_t)i], &A[(size_t)j]});
  std::vector<double> g;
  {
    TTB_RANGE("tt_orth: Gram matrix");
    g = dots_host(ctx, pr);
  }
  std::vector<double> G((size_t)m * m);
  size_t t = 0;
  for (int i = 0; i < m; ++i)
    for (int j = 0; j <= i; ++j, ++t) G[(size_t)i * m + j] = G[(size_t)j * m + i] = g[t];
  int piv = cholesky_host(G, m);
  if (piv >= 0) {
    *fail_index = piv;
    fail(TT_ESINGULAR_GRAM, "Cholesky of the Gram matrix failed at pivot " + std::to_string(piv) +
                                " (numerically singular, PAPER.md:224-226)");
  }
  // R = L^T, R^{-1} by back substitution (Remark 3)
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) R[(size_t)i * m + j] = (j >= i) ? G[(size_t)j * m + i] : 0.0;
  std::vector<double> X((size_t)m * m, 0.0);
  for (int j = 0; j < m; ++j) {
    X[(size_t)j * m + j] = 1.0 / R[(size_t)j * m + j];
    for (int i = j - 1; i >= 0; --i) {
      double s = 0.0;
      for (int k = i + 1; k <= j; ++k) s += R[(size_t)i * m + k] * X[(size_t)k * m + j];
      X[(size_t)i * m + j] = -s / R[(size_t)i * m + i];
    }
  }
  std::vector<SumInput> sums((size_t)m);
  for (int i = 0; i < m; ++i)
    for (int k = 0; k <= i; ++k) {
      TTRef a = A[(size_t)k];
      a.norm = an[(size_t)k];
      add_ref(sums[(size_t)i], a, X[(size_t)k * m + i]);  // q_i = sum_k R^{-1}(k,i) a_k (A5)
    }
  std::vector<tt_tensor> q = round_independent(ctx, sums, o.round, led);
  Q.insert(Q.end(), q.begin(), q.end());
}

// ----------------------------------------------------------------- Householder (Algs. 6-8)
void run_householder(tt_ctx ctx, int m, const std::vector<TTRef>& A, const std::vector<double>& an,
                     const tt_orth_opts& o, std::vector<tt_tensor>& Q, std::vector<double>& R, Ledger& led,
                     std::vector<tt_tensor>& Uout, int* fail_index) {
  const std::vector<int64_t>& n = A[0].n;
  std::vector<std::unique_ptr<Owned>> E;  // canonical e_1..e_m
  std::vector<TTRef> ER;
  for (int j = 1; j <= m; ++j) {
    E.emplace_back(new Owned(ctx, make_canonical(ctx, n, j)));
    ER.push_back(TTRef::of(E.back()->t));
  }
  std::vector<tt_tensor> U((size_t)m, nullptr);
  std::vector<TTRef> UR((size_t)m);
  std::vector<double> GU((size_t)m * m, 0.0), gamma((size_t)m * m, 0.0);
  Owned wown(ctx);
  TTRef w = A[0];
  w.norm = an[0];
  for (int i = 1; i <= m; ++i) {
    const std::string step_name = "tt_orth: Householder step " + std::to_string(i);
    TTB_RANGE(step_name.c_str());
    // TTH-vec(w, {e_1..e_i}) with element reads <w, e_j> = w(phi(j))
    std::vector<int64_t> lins;
    for (int j = 1; j <= i; ++j) lins.push_back(j);
    std::vector<double> ew = elements_host(ctx, w, lins);
    std::vector<double> r((size_t)i, 0.0);
    double s = 0.0;
    for (int j = 0; j < i - 1; ++j) { r[(size_t)j] = ew[(size_t)j]; s += r[(size_t)j] * r[(size_t)j]; }
    SumInput s1;
    Owned masked(ctx);
    if (o.hh_mask && i > 1) {
      // SURVEY.md §8(f) 3 (departure from Alg. 6 lines 4-9): w with the entries phi(1..i-1) set to
      // zero exactly, as w (.) mask(lin >= i-1), instead of the cancelling w - sum_{j<i} r(j) e_j
      Owned mk(ctx, mask_geq_tt(ctx, n, i - 1));
      masked.reset(hadamard(ctx, w.d, w.n, w.r, w.core, mk.t->r, mk.t->core_c));
      TTRef mr = TTRef::of(masked.t);
      add_ref(s1, mr, 1.0);  // norm NaN: s(x) = its own norm, computed (no cancellation)
    } else {
      add_ref(s1, w, 1.0);
      for (int j = 0; j < i - 1; ++j) add_ref(s1, ER[(size_t)j], -r[(size_t)j]);
    }
    Owned w1(ctx, led.round(ctx, s1, o.round));                 // Alg. 6 line 9
    const double w1n = last_core_norm(ctx, w1.t);
    w1.t->norm = w1n;
    const double sg = (ew[(size_t)i - 1] >= 0.0) ? 1.0 : -1.0;  // sign(0) = +1 (A8)
    double beta;
    if (o.hh_beta_literal) {
      const double d2 = w.norm * w.norm - s;
      if (d2 < -1e-12 * w.norm * w.norm) {
        *fail_index = i - 1;
        fail(TT_ENUMDEFECT, "||a||^2 - s < 0 in TTH-vec (SPEC.md:436)");
      }
      beta = std::sqrt(std::max(d2, 0.0));
    } else {
      beta = w1n;  // A9
    }
    r[(size_t)i - 1] = sg * beta;
    SumInput s2;
    add_ref(s2, TTRef::of(w1.t), 1.0);
    add_ref(s2, ER[(size_t)i - 1], -r[(size_t)i - 1]);
    Owned w2(ctx, led.round(ctx, s2, o.round));                 // Alg. 6 line 12
    const double nw = last_core_norm(ctx, w2.t);
    for (int j = 0; j < i; ++j) R[(size_t)j * m + (i - 1)] = r[(size_t)j];
    if (nw > 0.0) {
      scale_last_core(ctx, w2.t, 1.0 / nw);                     // u = w / ||w|| (A7)
      w2.t->norm = 1.0;
      U[(size_t)i - 1] = w2.release();
      UR[(size_t)i - 1] = TTRef::of(U[(size_t)i - 1]);
      std::vector<std::pair<const TTRef*, const TTRef*>> pr;
      for (int p = 0; p < i; ++p)
        if (U[(size_t)p]) pr.push_back({&UR[(size_t)p], &UR[(size_t)i - 1]});
      std::vector<double> g = dots_host(ctx, pr);
      size_t t = 0;
      for (int p = 0; p < i; ++p)
        if (U[(size_t)p]) { GU[(size_t)p * m + i - 1] = GU[(size_t)(i - 1) * m + p] = g[t++]; }
      // gamma_{j,i} = 2(<a_j, u_i> - sum_{p<i} gamma_{j,p} <u_p, u_i>) for j > i
      std::vector<std::pair<const TTRef*, const TTRef*>> pa;
      for (int j = i + 1; j <= m; ++j) pa.push_back({&A[(size_t)j - 1], &UR[(size_t)i - 1]});
      std::vector<double> da = dots_host(ctx, pa);
      for (int j = i + 1; j <= m; ++j) {
        double v = da[(size_t)(j - i - 1)];
        for (int p = 0; p < i - 1; ++p) v -= gamma[(size_t)(j - 1) * m + p] * GU[(size_t)p * m + i - 1];
        gamma[(size_t)(j - 1) * m + i - 1] = 2.0 * v;
      }
    }
    if (i < m) {                                                 // Alg. 8 lines 9-11
      SumInput sw;
      TTRef a = A[(size_t)i];
      a.norm = an[(size_t)i];
      add_ref(sw, a, 1.0);
      for (int l = 0; l < i; ++l)
        if (U[(size_t)l]) add_ref(sw, UR[(size_t)l], -gamma[(size_t)i * m + l]);
      wown.reset(led.round(ctx, sw, o.round));
      wown.t->norm = last_core_norm(ctx, wown.t);
      w = TTRef::of(wown.t);
    }
  }
  // phase 2: q_i = round(e_i - sum_{j<=i} beta_ij u_j) (Alg. 8 lines 13-19)
  std::vector<double> EU((size_t)m * m, 0.0);  // EU[j*m + i] = u_j(phi(i))
  for (int j = 0; j < m; ++j) {
    if (!U[(size_t)j]) continue;
    std::vector<int64_t> lins;
    for (int i = j; i < m; ++i) lins.push_back(i + 1);
    std::vector<double> e = elements_host(ctx, UR[(size_t)j], lins);
    for (int i = j; i < m; ++i) EU[(size_t)j * m + i] = e[(size_t)(i - j)];
  }
  std::vector<SumInput> sums((size_t)m);
  for (int i = 1; i <= m; ++i) {
    std::vector<double> bt((size_t)m, 0.0);
    for (int j = i; j >= 1; --j) {
      if (!U[(size_t)j - 1]) continue;
      double v = EU[(size_t)(j - 1) * m + (i - 1)];
      for (int l = j + 1; l <= i; ++l) v -= bt[(size_t)l - 1] * GU[(size_t)(l - 1) * m + (j - 1)];
      bt[(size_t)j - 1] = 2.0 * v;
    }
    SumInput& sq = sums[(size_t)i - 1];
    add_ref(sq, ER[(size_t)i - 1], 1.0);
    for (int j = i; j >= 1; --j)
      if (U[(size_t)j - 1]) add_ref(sq, UR[(size_t)j - 1], -bt[(size_t)j - 1]);
  }
  std::vector<tt_tensor> q = round_independent(ctx, sums, o.round, led);
  Q.insert(Q.end(), q.begin(), q.end());
  Uout = U;
  (void)fail_index;
}

}  // namespace

tt_status orth_run(tt_ctx ctx, tt_orth_kind kind, int m, const tt_view* a, const tt_orth_opts& o, tt_tensor* q_out,
                   double* R_host, tt_orth_report* rep) {
  if (m < 1 || !a || !q_out || !R_host) fail(TT_EINVAL, "tt_orth: bad arguments");
  std::vector<TTRef> A;
  for (int i = 0; i < m; ++i) {
    A.push_back(TTRef::of(a[i]));
    if (A.back().d != A[0].d || A.back().n != A[0].n) fail(TT_ESHAPE, "tt_orth: inputs differ in shape");
  }
  // ||a_i|| from one batched TT-dot
  std::vector<std::pair<const TTRef*, const TTRef*>> pr;
  for (int i = 0; i < m; ++i) pr.push_back({&A[(size_t)i], &A[(size_t)i]});
  std::vector<double> an2 = dots_host(ctx, pr);
  std::vector<double> an((size_t)m);
  for (int i = 0; i < m; ++i) an[(size_t)i] = std::sqrt(std::max(an2[(size_t)i], 0.0));
  std::vector<tt_tensor> Q, U;
  std::vector<double> R((size_t)m * m, 0.0), GQ((size_t)m * m, 0.0);
  Ledger led;
  int fidx = -1;
  if (rep) rep->fail_index = -1;
  try {
    switch (kind) {
      case TT_CGS: case TT_MGS: case TT_CGS2: case TT_MGS2:
        run_gs(ctx, kind, m, A, an, o, Q, R, GQ, led, &fidx);
        break;
      case TT_GRAM:
        run_gram(ctx, m, A, an, o, Q, R, led, &fidx);
        break;
      case TT_HOUSEHOLDER:
        run_householder(ctx, m, A, an, o, Q, R, led, U, &fidx);
        break;
      default:
        fail(TT_EINVAL, "unknown orthogonalization kind");
    }
  } catch (...) {
    for (tt_tensor t : Q) tensor_free(ctx, t);
    for (tt_tensor t : U) if (t) tensor_free(ctx, t);
    if (rep) { rep->fail_index = fidx; rep->rounding_calls = led.calls; }
    throw;
  }
  std::memcpy(R_host, R.data(), sizeof(double) * (size_t)m * m);
  for (int i = 0; i < m; ++i) q_out[i] = Q[(size_t)i];
  if (rep) {
    rep->rounding_calls = led.calls;
    if (rep->max_rank_per_call)
      std::memcpy(rep->max_rank_per_call, led.max_ranks.data(), sizeof(int64_t) * led.max_ranks.size());
    if (rep->loo_per_step) {
      bool have = (kind == TT_MGS || kind == TT_MGS2 || ((kind == TT_CGS || kind == TT_CGS2) && o.want_loo));
      if (!have) {
        std::vector<TTRef> QR;
        for (tt_tensor t : Q) QR.push_back(TTRef::of(t));
        std::vector<std::pair<const TTRef*, const TTRef*>> pq;
        for (int i = 0; i < m; ++i)
          for (int j = 0; j <= i; ++j) pq.push_back({&QR[(size_t)i], &QR[(size_t)j]});
        std::vector<double> g = dots_host(ctx, pq);
        size_t t = 0;
        for (int i = 0; i < m; ++i)
          for (int j = 0; j <= i; ++j, ++t) GQ[(size_t)i * m + j] = GQ[(size_t)j * m + i] = g[t];
      }
      for (int k = 1; k <= m; ++k) rep->loo_per_step[k - 1] = loo_host(GQ, m, k);
    }
    if (rep->householder_u) {
      for (int i = 0; i < m; ++i) rep->householder_u[i] = (i < (int)U.size()) ? U[(size_t)i] : nullptr;
    } else {
      for (tt_tensor t : U) if (t) tensor_free(ctx, t);
    }
  } else {
    for (tt_tensor t : U) if (t) tensor_free(ctx, t);
  }
  return TT_OK;
}

}  // namespace ttb
