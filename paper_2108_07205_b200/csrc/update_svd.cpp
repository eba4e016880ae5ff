// svd_optimal update compression (reference lowrank.cpp:329-362,
// CompressionMode::SvdOptimal): each off-diagonal block of Q (kc, kp, pk)
// densely evaluated and truncated by its SVD at eps, stacked as in
// assemble_stacked (lowrank.cpp:240-251), then L1 re-truncated by its own
// SVD: L = U_fin, R = diag(s_fin) V_fin^T R1.  A diagnostic mode (dense
// blocks, O(rows cols min(rows, cols)) SVDs), like the reference's.
#include "dense.hpp"
#include "entries.hpp"
#include "svd.hpp"
#include "update.hpp"

namespace sbx {

namespace {
std::vector<i64> scalars(const std::vector<i64>& nodes) {
  std::vector<i64> o;
  o.reserve(2 * nodes.size());
  for (i64 n : nodes) {
    o.push_back(2 * n);
    o.push_back(2 * n + 1);
  }
  return o;
}

TruncSvd block_svd(const EntryOracle& eo, const std::vector<i64>& rows, const std::vector<i64>& cols, double eps,
                   cudaStream_t s) {
  const i64 nr = i64(rows.size()), nc = i64(cols.size());
  if (nr == 0 || nc == 0) {
    TruncSvd t;
    t.m = nr;
    t.n = nc;
    return t;
  }
  DevBuf<i64> dr, dc;
  dr.upload(rows, s);
  dc.upload(cols, s);
  DevBuf<double> B(static_cast<size_t>(nr * nc));
  eo.submatrix(dr.get(), nr, dc.get(), nc, B.get(), nr, s);
  return truncated_svd_device(B.get(), nr, nc, nr, eps, s);
}
}  // namespace

std::unique_ptr<Update> update_svd_optimal_device(const Geom& old_g, const Geom& new_g, const Plan& plan, int form,
                                                  double mu, double eps, cudaStream_t s) {
  require(eps > 0.0 && eps <= 0.1, "compression tolerance out of range");
  auto u = std::make_unique<Update>();
  const auto kept_old_s = scalars(plan.kept_old), cut_s = scalars(plan.cut_old);
  const auto kept_new_s = scalars(plan.kept_new), added_s = scalars(plan.added_new);
  u->nk2 = i64(kept_old_s.size());
  u->nc2 = i64(cut_s.size());
  u->np2 = i64(added_s.size());
  const i64 n_ext = u->n_ext(), nk2 = u->nk2, nc2 = u->nc2, np2 = u->np2;
  EntryOracle eold(old_g, form, mu, s), enew(new_g, form, mu, s);
  // BlockSource blocks (nystrom.cpp:271-358): kc on the old mesh, kp / pk on the new one
  const TruncSvd kc = block_svd(eold, kept_old_s, cut_s, eps, s);
  const TruncSvd kp = block_svd(enew, kept_new_s, added_s, eps, s);
  const TruncSvd pk = block_svd(enew, added_s, kept_new_s, eps, s);
  u->k_kc = kc.k;
  u->k_kp = kp.k;
  u->k_pk = pk.k;
  const i64 k1 = pk.k + kc.k + kp.k;
  u->k1 = k1;
  u->notes.push_back("svd_optimal");
  if (k1 == 0) {
    u->k = 0;
    SBX_CUDA(cudaStreamSynchronize(s));
    return u;
  }
  // assemble_stacked: L1 = [pk.L | -kc.L | kp.L] by row group, R1 = block rows
  const i64 ckc = pk.k, ckp = pk.k + kc.k;
  DevBuf<double> L1(static_cast<size_t>(n_ext * k1)), R1(static_cast<size_t>(k1 * n_ext));
  L1.zero(s);
  R1.zero(s);
  std::vector<ScatterJob> sj;
  if (kc.k) sj.push_back({kc.U.get(), L1.get() + ckc * n_ext, nullptr, int(nk2), int(kc.k), int(nk2), int(n_ext), 0, 0, -1.0});
  if (kp.k) sj.push_back({kp.U.get(), L1.get() + ckp * n_ext, nullptr, int(nk2), int(kp.k), int(nk2), int(n_ext), 0, 0, 1.0});
  if (pk.k)
    sj.push_back({pk.U.get(), L1.get() + (nk2 + nc2), nullptr, int(np2), int(pk.k), int(np2), int(n_ext), 0, 0, 1.0});
  scatter_batched(sj, s);
  if (pk.k) svd_sv_vt(pk, R1.get(), k1, s);                          // rows [0, pk.k), cols [0, nk2)
  if (kc.k) svd_sv_vt(kc, R1.get() + ckc + nk2 * k1, k1, s);         // cols [nk2, nk2 + nc2)
  if (kp.k) svd_sv_vt(kp, R1.get() + ckp + (nk2 + nc2) * k1, k1, s);  // cols [nk2 + nc2, n_ext)
  // final truncation of L1 (lowrank.cpp:355-360)
  const TruncSvd fin = truncated_svd_device(L1.get(), n_ext, k1, n_ext, eps, s);
  const i64 k = fin.k;
  u->k = k;
  if (k > 0) {
    u->L->resize(size_t(n_ext * k));
    SBX_CUDA(cudaMemcpyAsync(u->L->get(), fin.U.get(), size_t(n_ext * k) * 8, cudaMemcpyDeviceToDevice, s));
    DevBuf<double> SVt(static_cast<size_t>(k * k1));
    svd_sv_vt(fin, SVt.get(), k, s);
    u->R.resize(size_t(k * n_ext));
    gemm_batched({{SVt.get(), R1.get(), u->R.get(), int(k), int(n_ext), int(k1), int(k), int(k1), int(k), 0, 0, 1.0,
                   0.0}},
                 s);
  }
  SBX_CUDA(cudaStreamSynchronize(s));
  return u;
}

}  // namespace sbx
