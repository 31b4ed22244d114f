// Debug harness: cluster QRCP vs the single-CTA QRCP on random matrices (prints mismatches).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I include tools/qrcp_check.cu
//        paper_2211_08770_b200/_lib/obj/*.o -o tools/qrcp_check
#include <cstdio>
#include <random>
#include <vector>

#include "../paper_2211_08770_b200/csrc/qr.cuh"

using namespace ttb;

int main(int argc, char** argv) {
  tt_ctx ctx = nullptr;
  if (tt_ctx_create(0, nullptr, &ctx) != TT_OK) { printf("ctx failed\n"); return 1; }
  ctx->debug_sync = true;
  int shapes[][2] = {{32, 64}, {1024, 64}, {320, 300}, {64, 16}, {500, 37}};
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd;
  for (auto& sh : shapes) {
    const int m = sh[0], c = sh[1];
    std::vector<double> h((size_t)m * c);
    // low-rank + noise so the stop criterion triggers
    const int r = std::min(10, std::min(m, c));
    std::vector<double> U((size_t)m * r), V((size_t)r * c);
    for (auto& x : U) x = nd(rng);
    for (auto& x : V) x = nd(rng);
    for (int j = 0; j < c; ++j)
      for (int i = 0; i < m; ++i) {
        double s = 1e-13 * nd(rng);
        for (int q = 0; q < r; ++q) s += U[(size_t)i + (size_t)q * m] * V[(size_t)q + (size_t)j * r];
        h[(size_t)i + (size_t)j * m] = s;
      }
    for (int mode = 0; mode < 2; ++mode) {
      try {
        DBuf Y(ctx, (size_t)m * c);
        cudaMemcpy(Y.p, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
        QRCPState st;
        qrcp_init(ctx, st, Y.p, m, m, c);
        if (mode == 1) st.cluster = 0;  // force the single-CTA kernel
        qrcp_run(ctx, st, Y.p, m, 1e-18 * m * c, std::min(m, c));
        std::vector<int> perm(c);
        std::vector<double> out(h.size()), tau(c);
        cudaMemcpy(perm.data(), st.perm.p, sizeof(int) * c, cudaMemcpyDeviceToHost);
        cudaMemcpy(out.data(), Y.p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost);
        cudaMemcpy(tau.data(), st.tau.p, sizeof(double) * c, cudaMemcpyDeviceToHost);
        bool ok = true;
        std::vector<int> seen(c, 0);
        for (int j = 0; j < c; ++j) {
          if (perm[j] < 0 || perm[j] >= c) ok = false;
          else seen[perm[j]]++;
        }
        for (int j = 0; j < c; ++j) ok = ok && seen[j] == 1;
        printf("m=%d c=%d mode=%s k=%d e2=%.3e perm_ok=%d R00=%.6e R11=%.6e tau0=%.6e perm[0..3]=%d %d %d %d\n", m, c,
               mode ? "single" : "cluster", st.k, st.e2, (int)ok, out[0], out[(size_t)m + 1], tau[0], perm[0],
               c > 1 ? perm[1] : -1, c > 2 ? perm[2] : -1, c > 3 ? perm[3] : -1);
      } catch (const Error& e) {
        printf("m=%d c=%d mode=%d error: %s\n", m, c, mode, e.msg.c_str());
        return 1;
      }
    }
  }
  return 0;
}
