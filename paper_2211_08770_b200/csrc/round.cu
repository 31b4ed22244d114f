// TT-rounding pipeline (host orchestration of the sm_100a kernels).
//
//   right-to-left (k = d..2): panel A_k = (X_k x_3 R_{k+1})^T assembled straight from the
//     terms' cores (block-diagonal TT-sum read in-kernel; one grouped DMMA GEMM over terms),
//     blocked Householder QR (TSQR panels + compact WY), core k <- Q (its column-major
//     layout IS the (R'_{k-1}, n_k, R'_k) core layout), R passed left;
//   norm ||x|| = ||C_1||_F, tau = max(delta ||x|| / sqrt(d-1), floor_c u s(x));
//   left-to-right (k = 1..d-1): truncated SVD of the unfolding, core k <- U_rho,
//     core k+1 <- (S V^T) x_1 core k+1 (DMMA GEMM).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <numeric>

#include "batch_round.cuh"
#include "gemm.cuh"
#include "qr.cuh"
#include "round.cuh"
#include "svd.cuh"
#include "ttops.cuh"

namespace ttb {

void SumInput::add(const tt_view& v, double c) {
  TTShape s = view_shape(v);
  if (coef.empty()) {
    d = s.d;
    n = s.n;
  } else {
    if (s.d != d) fail(TT_ESHAPE, "TT-sum terms differ in order d");
    for (int k = 0; k < d; ++k)
      if (s.n[k] != n[k]) fail(TT_ESHAPE, "TT-sum terms differ in mode sizes");
  }
  r.push_back(s.r);
  core.emplace_back(v.core, v.core + v.d);
  coef.push_back(c);
  norm.push_back(v.norm);
}

void SumInput::add_tensor(tt_tensor t, double c) {
  tt_view v;
  v.d = t->d;
  v.n = t->n.data();
  v.r = t->r.data();
  v.core = t->core_c.data();
  v.norm = t->norm;
  add(v, c);
}

tt_round_opts default_round_opts() {
  tt_round_opts o;
  o.rel_tol = 0.0;
  o.max_rank = 0;
  o.floor_c = 2048.0;
  o.qrcp_theta = 0.5;
  o.rank_revealing = 1;
  return o;
}

namespace {

constexpr double QRCP_EPS = 1e-12;

struct Sweep {
  std::vector<int64_t> R;     // formal ranks R_0..R_d
  std::vector<int64_t> Rp;    // ranks after the right-to-left sweep
  DBuf C1;                    // C_1 (1, n_1, R'_1)
  // Householder factors of core k's QR (k = 2..d): the right-orthonormal core k is Q_k^T,
  // never formed; the left-to-right sweep applies Q_k to the thin S V^T.  Either blocked
  // compact-WY factors (F) or, for the rank-revealing sweep, the unblocked column-pivoted
  // reflectors (P: m x c matrix with the reflectors in columns 0..k-1, tau).
  std::vector<QRFactors> F;
  std::vector<DBuf> P, Ptau;
  std::vector<int64_t> Pm;
  std::vector<char> rr;
};

// Rank-revealing sweep: the column-pivoted QR of a right-to-left panel A_k stops once the
// trailing block R_22 satisfies ||X_{<k}||_F ||R_22||_F <= RR_EPS s(x): the tensor x =
// X_{<k} A_k^T Q_{>k}^T with X_{<k} = [X^(1)_{<k} .. X^(K)_{<k}] (block columns), so dropping
// R_22 perturbs x by at most ||X_{<k}||_F ||R_22||_F in the Frobenius norm -- independent of
// how the terms distribute their scale over the cores (gauge).  Summed over the d-1 panels the
// perturbation stays below (d-1) RR_EPS s(x), orders of magnitude under the noise floor
// floor_c u s(x).  ||X^(l)_{<k}||_F^2 = trace of the TT-dot recursion's W after core k-1
// (x = y = term l).  DESIGN.md section 8.
constexpr double RR_EPS = 16.0 * U_ROUND;

struct RRBound {
  double s = 0.0;               // s(x) = sum_l |c_l| ||y_l||
  std::vector<double> left;     // left[j] = ||X_{<=j}||_F (cores 1..j of all terms), j = 0..d
};

std::vector<std::vector<int64_t>> offsets(const SumInput& in, std::vector<int64_t>& R) {
  const int d = in.d, K = in.K();
  std::vector<std::vector<int64_t>> off((size_t)d + 1, std::vector<int64_t>((size_t)K, 0));
  R.assign((size_t)d + 1, 1);
  for (int k = 1; k < d; ++k) {
    int64_t s = 0;
    for (int l = 0; l < K; ++l) {
      off[(size_t)k][(size_t)l] = s;
      s += in.r[(size_t)l][(size_t)k];
    }
    R[(size_t)k] = s;
  }
  return off;
}

// Right-to-left orthogonalisation of the (never materialised) TT-sum.
double norm_of(tt_ctx ctx, const double* x, int64_t n);

// Left-part norms of all terms after every core (one batched self-dot launch) and s(x).
RRBound rr_bound(tt_ctx ctx, const SumInput& in) {
  const int d = in.d, K = in.K();
  DotBatch b;
  b.d = d;
  b.n = in.n;
  b.P = K;
  for (int l = 0; l < K; ++l) {
    for (int k = 0; k < d; ++k) {
      b.xc.push_back(in.core[(size_t)l][(size_t)k]);
      b.yc.push_back(in.core[(size_t)l][(size_t)k]);
    }
    for (int k = 0; k <= d; ++k) {
      b.xr.push_back(in.r[(size_t)l][(size_t)k]);
      b.yr.push_back(in.r[(size_t)l][(size_t)k]);
    }
  }
  DBuf out(ctx, (size_t)K), tr(ctx, (size_t)K * (d + 1));
  dot_batch(ctx, b, out.p, tr.p);
  std::vector<double> h((size_t)K * (d + 1));
  d2h_small(ctx, h.data(), tr.p, h.size());
  RRBound rb;
  rb.left.assign((size_t)d + 1, 0.0);
  for (int l = 0; l < K; ++l) {
    for (int j = 0; j <= d; ++j) rb.left[(size_t)j] += std::max(h[(size_t)l * (d + 1) + j], 0.0);
    double nl = in.norm[(size_t)l];
    if (!(nl == nl)) nl = std::sqrt(std::max(h[(size_t)l * (d + 1) + d], 0.0));
    rb.s += std::fabs(in.coef[(size_t)l]) * nl;
  }
  for (double& v : rb.left) v = std::sqrt(v);
  return rb;
}

void right_to_left(tt_ctx ctx, const SumInput& in, Sweep& sw, const RRBound* rrb) {
  TTB_RANGE("tt_round: right-to-left orthogonalisation");
  const bool rank_revealing = rrb != nullptr;
  const int d = in.d, K = in.K();
  std::vector<std::vector<int64_t>> off = offsets(in, sw.R);
  sw.Rp.assign((size_t)d + 1, 1);
  sw.F.clear();
  sw.F.resize((size_t)d);
  sw.P.clear();
  sw.P.resize((size_t)d);
  sw.Ptau.clear();
  sw.Ptau.resize((size_t)d);
  sw.Pm.assign((size_t)d, 0);
  sw.rr.assign((size_t)d, 0);
  // panel of the last core: A_d (n_d x R_{d-1}).  The coefficients c_l are applied to the
  // terms' LAST cores here (same tensor: c_l may scale any core of term l), so every column
  // block of every panel carries its term's real magnitude -- what the rank-revealing stop
  // criterion needs (rounding outputs, the usual terms, are left-orthonormal in cores 1..d-1).
  int64_t m = in.n[(size_t)d - 1], c = sw.R[(size_t)d - 1];
  DBuf A(ctx, (size_t)m * c);
  {
    std::vector<TermCore> tc;
    for (int l = 0; l < K; ++l)
      tc.push_back({in.core[(size_t)l][(size_t)d - 1], in.r[(size_t)l][(size_t)d - 1], 1, off[(size_t)d - 1][(size_t)l], 0, in.coef[(size_t)l]});
    gather_last(ctx, tc, in.n[(size_t)d - 1], A.p, m);
  }
  // The rank-revealing QRCP pays off when the sum's numerical rank is below its structural
  // rank; once a panel keeps every column (e.g. sums of independently rounded vectors, whose
  // perturbations sit far above the 16 u s(x) cut), the rest of the sweep uses the blocked
  // Householder QR, which is cheaper per column than the pivoted one.
  bool rr_on = rank_revealing;
  for (int k = d; k >= 2; --k) {
    const int64_t nk = in.n[(size_t)k - 1];
    m = nk * sw.Rp[(size_t)k];
    c = sw.R[(size_t)k - 1];
    int64_t kq = std::min(m, c);
    DBuf Rk;
    bool done = false;
    if (rr_on) {  // cluster-resident QRCP when it fits, the grid / single-CTA QRCP otherwise
      // Tall panels beyond L2 (m >= 2c, > 64 MB): blocked Householder QR first (DMMA, one pass
      // over A), then the pivoted QR of its c x c triangle R, which stays in L2.  A P = Q (R P)
      // = Q Q' R', so the pivots, the trailing masses and hence the stopping test are those of
      // the QRCP of A itself (Frobenius norms are invariant under Q); the column-by-column pivoted
      // sweep never streams the m x c panel.  Q_k = Q diag(Q', I).
      static const char* pre_env = std::getenv("TT_B200_RR_PRE");
      const bool dbg = std::getenv("TT_B200_RR_DEBUG") != nullptr;
      // (only past L2: an L2-resident panel is cheaper to pivot directly, measured in DESIGN.md)
      bool pre = !qrcp_cluster_fits(m, c) && m >= 2 * c && (double)m * c * sizeof(double) > 64e6;
      if (pre_env && pre_env[0] == '0') pre = false;
      if (pre_env && pre_env[0] == '1') pre = !qrcp_cluster_fits(m, c) && m >= 2 * c;
      cudaEvent_t ev0 = nullptr, ev1 = nullptr;
      if (dbg) {
        cudaEventCreate(&ev0);
        cudaEventCreate(&ev1);
        cudaEventRecord(ev0, ctx->stream);
      }
      DBuf Rsq;
      double* Y = A.p;
      int64_t my = m;
      if (pre) {
        geqrf(ctx, A.p, m, m, c, sw.F[(size_t)k - 1]);
        Rsq.alloc(ctx, (size_t)c * c);
        copy_upper(ctx, A.p, m, c, c, Rsq.p, c);
        Y = Rsq.p;
        my = c;
      }
      QRCPState st;
      qrcp_init(ctx, st, Y, my, my, c);
      const double lk = rrb->left[(size_t)k - 1];
      const double stop = lk > 0.0 ? RR_EPS * rrb->s / lk : 0.0;
      qrcp_run(ctx, st, Y, my, stop * stop, (int)kq);
      if (st.k == 0) qrcp_run(ctx, st, Y, my, -1.0, 1);  // keep rank >= 1
      if (dbg) {
        float ms = 0.f;
        cudaEventRecord(ev1, ctx->stream);
        cudaEventSynchronize(ev1);
        cudaEventElapsedTime(&ms, ev0, ev1);
        cudaEventDestroy(ev0);
        cudaEventDestroy(ev1);
        std::fprintf(stderr, "[rr] core %d panel %lld x %lld kept %d of %lld %.3f ms%s\n", k, (long long)m, (long long)c,
                     st.k, (long long)kq, ms, pre ? " (qr+qrcp)" : qrcp_cluster_fits(m, c) ? " (cluster)" : "");
      }
      if (st.k >= kq && !qrcp_cluster_fits(m, c)) rr_on = false;  // no rank drop: full QR from here
      kq = st.k;
      // L_k^T = R_1 P^T (kq x c): R_1 in pivoted order, columns put back in original order
      DBuf R1(ctx, (size_t)kq * c);
      copy_upper(ctx, Y, my, kq, c, R1.p, kq);
      Rk.alloc(ctx, (size_t)kq * c);
      unpermute_cols(ctx, R1.p, kq, kq, c, st.perm.p, Rk.p, kq);
      sw.rr[(size_t)k - 1] = pre ? 2 : 1;
      sw.Pm[(size_t)k - 1] = my;
      sw.Ptau[(size_t)k - 1] = std::move(st.tau);
      sw.P[(size_t)k - 1] = pre ? std::move(Rsq) : std::move(A);  // keeps the reflectors (columns 0..kq-1)
      if (pre) A = DBuf();
      done = true;
    }
    if (!done) {
      QRFactors& f = sw.F[(size_t)k - 1];
      geqrf(ctx, A.p, m, m, c, f);
      Rk.alloc(ctx, (size_t)kq * c);
      copy_upper(ctx, A.p, m, kq, c, Rk.p, kq);
    }
    sw.Rp[(size_t)k - 1] = kq;
    const int64_t nkm1 = in.n[(size_t)k - 2];
    if (k - 1 >= 2) {
      // A_{k-1}[(i kq + b'), off_{k-2,l} + a] = sum_{b in block l} R(b', b) X_{k-1}^(l)(a, i, b)
      const int64_t m2 = nkm1 * kq, c2 = sw.R[(size_t)k - 2];
      DBuf A2(ctx, (size_t)m2 * c2);
      std::vector<GemmDesc> gs;
      for (int l = 0; l < K; ++l) {
        GemmDesc g;
        g.M = kq;
        g.K = in.r[(size_t)l][(size_t)k - 1];
        g.N = in.r[(size_t)l][(size_t)k - 2] * nkm1;
        g.A = Rk.p + off[(size_t)k - 1][(size_t)l] * kq;
        g.lda = kq;
        g.B = in.core[(size_t)l][(size_t)k - 2];
        g.ldb = in.r[(size_t)l][(size_t)k - 1];
        g.C = A2.p + off[(size_t)k - 2][(size_t)l] * m2;
        g.ldc = kq;
        g.ncol_split = nkm1;
        g.ldc_hi = m2;
        gs.push_back(g);
      }
      gemm_grouped(ctx, gs);
      A = std::move(A2);
    } else {
      // first core: C_1 (1, n_1, kq) = R_2 (kq x R_1) * M1 (R_1 x n_1), M1 = [c_l X_1^(l)]
      const int64_t R1 = sw.R[1];
      DBuf M1(ctx, (size_t)R1 * nkm1);
      std::vector<TermCore> tc;
      for (int l = 0; l < K; ++l)
        tc.push_back({in.core[(size_t)l][0], 1, in.r[(size_t)l][1], 0, off[1][(size_t)l], 1.0});
      gather_first(ctx, tc, nkm1, M1.p, R1);
      sw.C1.alloc(ctx, (size_t)kq * nkm1);
      GemmDesc g;
      g.M = kq; g.N = nkm1; g.K = R1; g.A = Rk.p; g.lda = kq; g.B = M1.p; g.ldb = R1; g.C = sw.C1.p; g.ldc = kq;
      gemm(ctx, g);
    }
  }
}

double norm_of(tt_ctx ctx, const double* x, int64_t n) {
  DBuf s(ctx, 1);
  sumsq(ctx, x, n, s.p);
  double h = 0.0;
  d2h_small(ctx, &h, s.p, 1);
  return std::sqrt(h);
}

double term_norm(tt_ctx ctx, const SumInput& in, int l) {
  SumInput one;
  one.d = in.d;
  one.n = in.n;
  one.r.push_back(in.r[(size_t)l]);
  one.core.push_back(in.core[(size_t)l]);
  one.coef.push_back(1.0);
  one.norm.push_back(NAN);
  return sweep_norm(ctx, one);
}

}  // namespace

double sweep_norm(tt_ctx ctx, const SumInput& in) {
  if (in.d == 1) {
    std::vector<const double*> xs;
    for (int l = 0; l < in.K(); ++l) xs.push_back(in.core[(size_t)l][0]);
    DBuf o(ctx, (size_t)in.n[0]);
    lincomb(ctx, xs, in.coef, in.n[0], o.p);
    return norm_of(ctx, o.p, in.n[0]);
  }
  Sweep sw;
  right_to_left(ctx, in, sw, nullptr);
  return norm_of(ctx, sw.C1.p, sw.Rp[1] * in.n[0]);
}

tt_tensor materialise_sum(tt_ctx ctx, const SumInput& in) {
  const int d = in.d, K = in.K();
  std::vector<int64_t> R;
  std::vector<std::vector<int64_t>> off = offsets(in, R);
  tt_tensor t = tensor_alloc(ctx, d, in.n, R);
  for (int k = 0; k < d; ++k) {
    std::vector<TermCore> tc;
    for (int l = 0; l < K; ++l) {
      const int64_t o0 = (k == 0) ? 0 : off[(size_t)k][(size_t)l];
      const int64_t o1 = (k == d - 1) ? 0 : off[(size_t)k + 1][(size_t)l];
      tc.push_back({in.core[(size_t)l][(size_t)k], in.r[(size_t)l][(size_t)k], in.r[(size_t)l][(size_t)k + 1], o0, o1,
                    in.coef[(size_t)l]});
    }
    if (d == 1) {
      std::vector<const double*> xs;
      for (int l = 0; l < K; ++l) xs.push_back(in.core[(size_t)l][0]);
      lincomb(ctx, xs, in.coef, in.n[0], t->core[0]);
    } else {
      materialise_core(ctx, tc, in.n[(size_t)k], R[(size_t)k], R[(size_t)k + 1], k == 0, k == d - 1, t->core[(size_t)k]);
    }
  }
  return t;
}

tt_tensor round_sum(tt_ctx ctx, const SumInput& in, const tt_round_opts& o, tt_round_info* info) {
  TTB_RANGE("tt_round");
  const int d = in.d, K = in.K();
  if (K < 1) fail(TT_EINVAL, "TT-round needs at least one term");
  if (o.rel_tol < 0.0 || !(o.rel_tol == o.rel_tol)) fail(TT_EINVAL, "rel_tol must be >= 0");
  const double theta = (o.qrcp_theta > 0.0 && o.qrcp_theta <= 1.0) ? o.qrcp_theta : 0.5;
  const bool keep_all = (o.rel_tol == 0.0);
  tt_round_info inf{};
  if (d == 1) {
    tt_tensor t = tensor_alloc(ctx, 1, in.n, {1, 1});
    std::vector<const double*> xs;
    for (int l = 0; l < K; ++l) xs.push_back(in.core[(size_t)l][0]);
    lincomb(ctx, xs, in.coef, in.n[0], t->core[0]);
    inf.norm = norm_of(ctx, t->core[0], in.n[0]);
    inf.scale = inf.norm;
    t->norm = inf.norm;
    if (info) *info = inf;
    return t;
  }
  // Sums inside the batched engine's shapes (d <= 64, K <= 16, formal ranks <= 64: C1, the Krylov
  // sets, short Householder sums) run as a one-item batch: the whole rounding is a handful of
  // one-CTA launches with on-device decisions and a single ranks read-back, where this sweep pays
  // several launches and host round trips per core.  Same rounding (SURVEY A2/A12
  // threshold), parity-tested against the oracle like the sweep.  TT_B200_SERIAL_BATCH=0 keeps the
  // sweep.  Exact rounding (rel_tol = 0) stays on the sweep: the batched engine forms the output
  // cores as Y V S^-1, which leaves a zero column (not an orthonormal completion) for an exactly
  // zero singular value that keep_all retains.
  static const char* sb_env = std::getenv("TT_B200_SERIAL_BATCH");
  if (!(sb_env && sb_env[0] == '0') && !keep_all && batch_shape_supported(d, K, in.r, nullptr)) {
    tt_tensor t = nullptr;
    round_batch_uniform(ctx, std::vector<SumInput>{in}, o, &t, nullptr, &inf);
    if (info) *info = inf;
    return t;
  }
  // pre-cancellation scale s(x) = sum_l |c_l| ||y_l||
  double s = 0.0;
  const bool rank_revealing = !keep_all && o.rank_revealing;
  RRBound rrb;
  if (rank_revealing) {
    rrb = rr_bound(ctx, in);
    s = rrb.s;
  } else if (!keep_all && o.floor_c > 0.0) {
    for (int l = 0; l < K; ++l) {
      double nl = in.norm[(size_t)l];
      if (!(nl == nl)) nl = term_norm(ctx, in, l);
      s += std::fabs(in.coef[(size_t)l]) * nl;
    }
  }
  Sweep sw;
  right_to_left(ctx, in, sw, rank_revealing ? &rrb : nullptr);
  const double nrm = norm_of(ctx, sw.C1.p, sw.Rp[1] * in.n[0]);
  if (keep_all || o.floor_c <= 0.0) s = nrm;
  double tau = 0.0;
  if (!keep_all) tau = std::max(o.rel_tol * nrm / std::sqrt((double)(d - 1)), o.floor_c * U_ROUND * s);
  // QRCP stop: below theta*tau (decision stays exact, see svd.cu) and below QRCP_EPS s(x)
  // so the kept subspace equals the exact truncated SVD's to the parity tolerance.
  const double stop_abs = std::min(theta * tau, QRCP_EPS * std::max(s, nrm));
  inf.norm = nrm;
  inf.scale = s;
  inf.tau = tau;
  if (nrm == 0.0) {
    tt_tensor t = tensor_alloc(ctx, d, in.n, std::vector<int64_t>((size_t)d + 1, 1));
    TTB_CUDA(cudaMemsetAsync(t->block, 0, sizeof(double) * (size_t)std::accumulate(in.n.begin(), in.n.end(), (int64_t)0), ctx->stream));
    t->norm = 0.0;
    if (info) *info = inf;
    return t;
  }
  // left-to-right truncation
  TTB_RANGE("tt_round: left-to-right truncation");
  std::vector<int64_t> ranks((size_t)d + 1, 1);
  std::vector<DBuf> outc((size_t)d);
  DBuf Z = std::move(sw.C1);
  for (int k = 1; k <= d - 1; ++k) {
    const int64_t m = ranks[(size_t)k - 1] * in.n[(size_t)k - 1], c = sw.Rp[(size_t)k];
    DBuf U, SV;
    TruncResult tr = truncated_svd(ctx, Z.p, m, c, tau, keep_all, o.max_rank, stop_abs, U, SV);
    inf.qrcp_steps += tr.qrcp_steps;
    inf.resumes += tr.resumes;
    ranks[(size_t)k] = tr.rho;
    outc[(size_t)k - 1] = std::move(U);
    // core k+1 <- (S V^T) x_1 Q_{k+1}^T, i.e. Z_{k+1}^T = Q_{k+1} (S V^T)^T = H [ (SV)^T ; 0 ]
    const int64_t N = in.n[(size_t)k] * sw.Rp[(size_t)k + 1];
    DBuf Zn(ctx, (size_t)N * tr.rho);
    TTB_CUDA(cudaMemsetAsync(Zn.p, 0, sizeof(double) * (size_t)N * tr.rho, ctx->stream));
    TTB_CUDA(cudaMemcpy2DAsync(Zn.p, sizeof(double) * N, SV.p, sizeof(double) * c, sizeof(double) * c, (size_t)tr.rho,
                               cudaMemcpyDeviceToDevice, ctx->stream));
    if (sw.rr[(size_t)k] == 2) {  // Q_k = Q diag(Q', I): Q' on the top c rows, then the blocked Q
      apply_reflectors_left(ctx, sw.P[(size_t)k].p, sw.Pm[(size_t)k], sw.Ptau[(size_t)k].p, sw.Pm[(size_t)k], (int)c,
                            Zn.p, N, tr.rho);
      sw.P[(size_t)k].release();
      sw.Ptau[(size_t)k].release();
      ormqr_left(ctx, sw.F[(size_t)k], Zn.p, N, tr.rho);
      sw.F[(size_t)k] = QRFactors();
    } else if (sw.rr[(size_t)k]) {
      apply_reflectors_left(ctx, sw.P[(size_t)k].p, sw.Pm[(size_t)k], sw.Ptau[(size_t)k].p, N, (int)c, Zn.p, N,
                            tr.rho);
      sw.P[(size_t)k].release();
      sw.Ptau[(size_t)k].release();
    } else {
      ormqr_left(ctx, sw.F[(size_t)k], Zn.p, N, tr.rho);
      sw.F[(size_t)k] = QRFactors();
    }
    Z = std::move(Zn);
  }
  outc[(size_t)d - 1] = std::move(Z);
  tt_tensor t = tensor_alloc(ctx, d, in.n, ranks);
  for (int k = 0; k < d; ++k)
    copy_d2d(ctx, t->core[(size_t)k], outc[(size_t)k].p, ranks[(size_t)k] * in.n[(size_t)k] * ranks[(size_t)k + 1]);
  t->norm = nrm;
  if (info) *info = inf;
  return t;
}

}  // namespace ttb
