// HBS arena layout and HBS1 interchange (reference hbs.cpp:681-808).
#include <algorithm>
#include <cstring>
#include <fstream>

#include "hbs.hpp"

namespace sbx {

i64 HbsOp::solve_factor_doubles() const {
  i64 t = 0;
  for (size_t i = 1; i < nodes.size(); ++i) {
    const auto& nd = nodes[i];
    t += (nd.k + nd.c) * nd.c + nd.c * nd.k;  // f, g, e
  }
  return t + nodes[0].c * nodes[0].c;  // root_g
}

i64 HbsOp::apply_factor_doubles() const {
  i64 t = 0;
  for (size_t i = 0; i < nodes.size(); ++i) {
    const auto& nd = nodes[i];
    if (i == 0 && nodes.size() > 1) continue;
    t += nd.k * nd.c + nd.c * nd.k;                  // v^T, u
    if (nd.is_leaf()) t += nd.c * nd.c;              // d
    if (i > 0) t += nd.k * nodes[size_t(sib(i64(i)))].k;  // b_sib
  }
  return t;
}

void hbs_layout(HbsOp& op) {
  require(!op.nodes.empty(), "hbs: empty operator");
  op.max_depth = 0;
  for (auto& nd : op.nodes) op.max_depth = std::max(op.max_depth, nd.depth);
  // candidate sizes, bottom-up
  for (int d = op.max_depth; d >= 0; --d)
    for (auto& nd : op.nodes) {
      if (nd.depth != d) continue;
      nd.c = nd.is_leaf() ? 2 * (nd.end - nd.begin)
                          : op.nodes[size_t(nd.left)].k + op.nodes[size_t(nd.right)].k;
    }
  i64 off = 0;
  auto place = [&](i64 sz) {
    i64 o = off;
    off += (sz + 31) / 32 * 32;  // 256-byte aligned blocks
    return o;
  };
  const size_t nn = op.nodes.size();
  // level-major per factor kind so each sweep level streams one range
  for (int kind = 0; kind < 7; ++kind)
    for (int d = op.max_depth; d >= 0; --d)
      for (size_t i = 0; i < nn; ++i) {
        auto& nd = op.nodes[i];
        if (nd.depth != d || !op.has(i)) continue;  // sharded: this rank's nodes only
        const bool root = i == 0;
        const i64 k = nd.k, c = nd.c;
        switch (kind) {
          case 0:  // fg (solve up)
            if (!root) nd.o_fg = place((k + c) * c);
            break;
          case 1:  // e (solve down)
            if (!root) nd.o_e = place(c * k);
            break;
          case 2:  // vd (apply up)
            if (!root || nd.is_leaf()) nd.o_vd = place((k + (nd.is_leaf() ? c : 0)) * c);
            break;
          case 3:  // u (apply down)
            if (!root) nd.o_u = place(c * k);
            break;
          case 4:  // b_sib
            if (!root) nd.o_b = place(k * op.nodes[size_t(op.sib(i64(i)))].k);
            break;
          case 5:  // v (invert)
            if (!root) nd.o_v = place(c * k);
            break;
          case 6:  // dhat (invert)
            if (!root) nd.o_dhat = place(k * k);
            break;
        }
      }
  op.o_root_g = place(op.nodes[0].c * op.nodes[0].c);
  op.arena_used = off;
  op.arena.resize(size_t(std::max<i64>(off, 32)));
  op.top_L = 0;
  op.o_top = -1;
  op.top_K = op.top_cap = 0;
  op.node_rcond.clear();
  op.solve_plan.built = false;
  op.apply_plan.built = false;
}

namespace {

void rbytes(std::istream& is, void* p, size_t n) {
  is.read(static_cast<char*>(p), std::streamsize(n));
  if (!is) throw Error(7, "hbs_load: truncated file");
}
template <class T>
T rpod(std::istream& is) {
  T v;
  rbytes(is, &v, sizeof(T));
  return v;
}
HMat rmat(std::istream& is) {
  const auto r = rpod<std::int64_t>(is);
  const auto c = rpod<std::int64_t>(is);
  if (r < 0 || c < 0) throw Error(7, "hbs_load: corrupt matrix header");
  HMat m(r, c);
  if (m.size()) rbytes(is, m.a.data(), size_t(8 * m.size()));
  return m;
}
std::vector<i64> ridx(std::istream& is) {
  const auto n = rpod<std::int64_t>(is);
  if (n < 0) throw Error(7, "hbs_load: corrupt index header");
  std::vector<i64> v(static_cast<size_t>(n));
  if (n) rbytes(is, v.data(), size_t(8 * n));
  return v;
}
template <class T>
void wpod(std::ostream& os, T v) {
  os.write(reinterpret_cast<const char*>(&v), sizeof(T));
}
void wmat(std::ostream& os, i64 r, i64 c, const double* p) {
  wpod<std::int64_t>(os, r);
  wpod<std::int64_t>(os, c);
  if (r * c) os.write(reinterpret_cast<const char*>(p), std::streamsize(8 * r * c));
}
void widx(std::ostream& os, const std::vector<i64>& v) {
  wpod<std::int64_t>(os, std::int64_t(v.size()));
  if (!v.empty()) os.write(reinterpret_cast<const char*>(v.data()), std::streamsize(8 * v.size()));
}

// copy a column-major (r x c) block into rows [r0, r0+r) of a column-major
// destination with leading dimension ld
void put_rows(double* dst, i64 ld, i64 r0, const HMat& m) {
  for (i64 j = 0; j < m.c; ++j)
    std::memcpy(dst + r0 + j * ld, m.a.data() + j * m.r, size_t(8 * m.r));
}
void get_rows(const double* src, i64 ld, i64 r0, i64 r, i64 c, std::vector<double>& out) {
  out.resize(size_t(r * c));
  for (i64 j = 0; j < c; ++j) std::memcpy(out.data() + j * r, src + r0 + j * ld, size_t(8 * r));
}
HMat transpose(const HMat& m) {
  HMat t(m.c, m.r);
  for (i64 j = 0; j < m.c; ++j)
    for (i64 i = 0; i < m.r; ++i) t.a[size_t(j + i * m.c)] = m.a[size_t(i + j * m.r)];
  return t;
}
void check_shape(const HMat& m, i64 r, i64 c, const char* what) {
  if (m.size() == 0 && r * c == 0) return;
  if (m.r != r || m.c != c)
    throw Error(7, std::string("hbs_load: inconsistent shape for ") + what);
}

}  // namespace

std::unique_ptr<HbsOp> hbs_load_hbs1(const std::string& path, cudaStream_t s) {
  std::ifstream is(path, std::ios::binary);
  require(bool(is), "hbs_load: cannot open " + path);
  char magic[4];
  rbytes(is, magic, 4);
  if (std::memcmp(magic, "HBS1", 4) != 0) throw Error(7, "hbs_load: bad magic bytes");
  if (rpod<std::uint32_t>(is) != 1) throw Error(7, "hbs_load: unsupported version");
  auto op = std::make_unique<HbsOp>();
  op->has_inverse = rpod<std::uint8_t>(is) != 0;
  op->n = rpod<std::int64_t>(is);
  op->leaf_nodes = rpod<std::int64_t>(is);
  op->eps = rpod<double>(is);
  op->max_block_drawn = rpod<std::int64_t>(is);
  const auto count = rpod<std::int64_t>(is);
  require(count > 0 && count < (1 << 26), "hbs_load: bad node count");
  op->nodes.resize(size_t(count));
  struct Mats {
    HMat u, v, d, b, dhat, e, f, g;
  };
  std::vector<Mats> mats(static_cast<size_t>(count));
  for (size_t i = 0; i < size_t(count); ++i) {
    auto& nd = op->nodes[i];
    nd.begin = rpod<std::int64_t>(is);
    nd.end = rpod<std::int64_t>(is);
    nd.parent = rpod<std::int64_t>(is);
    nd.left = rpod<std::int64_t>(is);
    nd.right = rpod<std::int64_t>(is);
    nd.depth = rpod<std::int32_t>(is);
    nd.k = rpod<std::int64_t>(is);
    nd.row_skel = ridx(is);
    nd.col_skel = ridx(is);
    auto& m = mats[i];
    for (HMat* p : {&m.u, &m.v, &m.d, &m.b, &m.dhat, &m.e, &m.f, &m.g}) *p = rmat(is);
  }
  HMat root_g = rmat(is);
  const auto nnotes = rpod<std::int64_t>(is);
  for (i64 i = 0; i < nnotes; ++i) {
    const auto len = rpod<std::int64_t>(is);
    std::string str(size_t(std::max<std::int64_t>(len, 0)), '\0');
    if (len > 0) rbytes(is, str.data(), size_t(len));
    op->notes.push_back(std::move(str));
  }
  hbs_layout(*op);
  std::vector<double> host(static_cast<size_t>(op->arena.size()), 0.0);
  double* H = host.data();
  const size_t nn = op->nodes.size();
  for (size_t i = 0; i < nn; ++i) {
    const auto& nd = op->nodes[i];
    const auto& m = mats[i];
    const i64 k = nd.k, c = nd.c;
    if (i == 0) {
      if (nd.is_leaf()) {
        check_shape(m.d, c, c, "root d");
        put_rows(H + nd.o_vd, c, 0, m.d);
      }
      continue;
    }
    check_shape(m.u, c, k, "u");
    check_shape(m.v, c, k, "v");
    put_rows(H + nd.o_u, c, 0, m.u);
    put_rows(H + nd.o_v, c, 0, m.v);
    const i64 vd_ld = k + (nd.is_leaf() ? c : 0);
    put_rows(H + nd.o_vd, vd_ld, 0, transpose(m.v));
    if (nd.is_leaf()) {
      check_shape(m.d, c, c, "d");
      put_rows(H + nd.o_vd, vd_ld, k, m.d);
    }
    const i64 ks = op->nodes[size_t(op->sib(i64(i)))].k;
    check_shape(m.b, k, ks, "b_sib");
    put_rows(H + nd.o_b, k, 0, m.b);
    if (op->has_inverse) {
      check_shape(m.dhat, k, k, "dhat");
      check_shape(m.e, c, k, "e");
      check_shape(m.f, k, c, "f");
      check_shape(m.g, c, c, "g");
      put_rows(H + nd.o_dhat, k, 0, m.dhat);
      put_rows(H + nd.o_e, c, 0, m.e);
      put_rows(H + nd.o_fg, k + c, 0, m.f);
      put_rows(H + nd.o_fg, k + c, k, m.g);
    }
  }
  if (op->has_inverse) {
    check_shape(root_g, op->nodes[0].c, op->nodes[0].c, "root_g");
    put_rows(H + op->o_root_g, op->nodes[0].c, 0, root_g);
  }
  op->has_apply = true;
  op->arena.upload(host, s);
  SBX_CUDA(cudaStreamSynchronize(s));
  return op;
}

void hbs_save_hbs1(const HbsOp& op, const std::string& path, cudaStream_t s) {
  require(!op.sharded(), "hbs_save: a subtree-sharded operator holds only its subtree's factors");
  std::vector<double> host(op.arena.size());
  op.arena.download(host.data(), host.size(), s);
  SBX_CUDA(cudaStreamSynchronize(s));
  const double* H = host.data();
  std::ofstream os(path, std::ios::binary);
  require(bool(os), "hbs_save: cannot open " + path);
  os.write("HBS1", 4);
  wpod<std::uint32_t>(os, 1);
  wpod<std::uint8_t>(os, op.has_inverse ? 1 : 0);
  wpod<std::int64_t>(os, op.n);
  wpod<std::int64_t>(os, op.leaf_nodes);
  wpod<double>(os, op.eps);
  wpod<std::int64_t>(os, op.max_block_drawn);
  wpod<std::int64_t>(os, std::int64_t(op.nodes.size()));
  std::vector<double> tmp;
  for (size_t i = 0; i < op.nodes.size(); ++i) {
    const auto& nd = op.nodes[i];
    wpod<std::int64_t>(os, nd.begin);
    wpod<std::int64_t>(os, nd.end);
    wpod<std::int64_t>(os, nd.parent);
    wpod<std::int64_t>(os, nd.left);
    wpod<std::int64_t>(os, nd.right);
    wpod<std::int32_t>(os, nd.depth);
    wpod<std::int64_t>(os, nd.k);
    widx(os, nd.row_skel);
    widx(os, nd.col_skel);
    const i64 k = nd.k, c = nd.c;
    if (i == 0) {
      // root keeps no u, v, b_sib or inverse factors (hbs.cpp:411,450-458)
      wmat(os, 0, 0, nullptr);  // u
      wmat(os, 0, 0, nullptr);  // v
      if (nd.is_leaf())
        wmat(os, c, c, H + nd.o_vd);
      else
        wmat(os, 0, 0, nullptr);
      for (int z = 0; z < 5; ++z) wmat(os, 0, 0, nullptr);  // b, dhat, e, f, g
      continue;
    }
    wmat(os, c, k, H + nd.o_u);
    wmat(os, c, k, H + nd.o_v);
    const i64 vd_ld = k + (nd.is_leaf() ? c : 0);
    if (nd.is_leaf()) {
      get_rows(H + nd.o_vd, vd_ld, k, c, c, tmp);
      wmat(os, c, c, tmp.data());
    } else {
      wmat(os, 0, 0, nullptr);
    }
    const i64 ks = op.nodes[size_t(op.sib(i64(i)))].k;
    wmat(os, k, ks, H + nd.o_b);
    if (op.has_inverse) {
      wmat(os, k, k, H + nd.o_dhat);
      wmat(os, c, k, H + nd.o_e);
      get_rows(H + nd.o_fg, k + c, 0, k, c, tmp);
      wmat(os, k, c, tmp.data());
      get_rows(H + nd.o_fg, k + c, k, c, c, tmp);
      wmat(os, c, c, tmp.data());
    } else {
      for (int z = 0; z < 4; ++z) wmat(os, 0, 0, nullptr);
    }
  }
  if (op.has_inverse)
    wmat(os, op.nodes[0].c, op.nodes[0].c, H + op.o_root_g);
  else
    wmat(os, 0, 0, nullptr);
  wpod<std::int64_t>(os, std::int64_t(op.notes.size()));
  for (const auto& str : op.notes) {
    wpod<std::int64_t>(os, std::int64_t(str.size()));
    os.write(str.data(), std::streamsize(str.size()));
  }
  require(bool(os), "hbs_save: write failed");
}

}  // namespace sbx
