// Kernel-block assembly on sm_100a (north-star subsystem 1).
// Compiled with --fmad=false so the interior (double-layer + completion)
// entries round exactly like the reference's scalar code (nystrom.cpp:80-172):
// no FMA contraction, IEEE division.  Stores are coalesced along the
// leading dimension of the column-major destination.
#include <algorithm>
#include <cstdint>
#include <vector>

#include "entries.hpp"
#include "logquad.hpp"

namespace sbx {

namespace {

__device__ __forceinline__ i64 node_of(const EntryView& v, i64 local) {
  return v.map ? v.map[local] : local;
}

__device__ __forceinline__ bool in_null(const EntryView& v, int comp) {
  return v.form == SBX_INTERIOR_DIRICHLET || (v.form == SBX_MIXED && comp == 0);
}
__device__ __forceinline__ bool single_layer(const EntryView& v, int comp) {
  return v.form == SBX_EXTERIOR_COMBINED || (v.form == SBX_MIXED && comp != 0);
}

// One scalar entry A(2i+a, 2j+b) of the completed BIE (nystrom.cpp:80-172):
// double layer + completion bit-for-bit in the reference's operation order;
// on single-layer components the Stokeslet with the product-integration log
// correction on the self and neighbouring panels (tables from logquad.cpp).
__device__ double entry(const EntryView& v, i64 rs, i64 cs) {
  const i64 i = node_of(v, rs >> 1), j = node_of(v, cs >> 1);
  const int a = int(rs & 1), b = int(cs & 1);
  const int ci = v.comp[i];
  const double c4 = 1.0 / (4.0 * kPi * v.mu);
  if (i == j) {
    const double wi = v.w[i];
    const double dl = -v.kappa[i] / (2.0 * kPi) * wi;
    // out[2] = out[1] in the reference: both off-diagonal slots are (dl*tx)*ty
    const double ta = (a == 0 || a != b) ? v.tx[i] : v.ty[i];
    const double tb = (b == 1 || a != b) ? v.ty[i] : v.tx[i];
    double out = dl * ta * tb;
    if (a == b) out = v.jump + out;
    if (single_layer(v, ci)) {
      const double sm = wi * c4;
      out += sm * ta * tb;
      if (a == b) {
        const i64 n = v.sl_n;
        const int loc = v.sl_i[i], q = v.sl_i[n + i];
        const double jac = v.sl_d[n + i];
        const double lam = v.sl_tab[v.sl_i[4 * n + i] + loc * q + loc];
        out += c4 * (-lam * jac - wi * log(jac));
      }
    }
    if (in_null(v, ci)) {
      const double na = a == 0 ? v.nx[i] : v.ny[i];
      const double nb = b == 0 ? v.nx[i] : v.ny[i];
      out += wi * na * nb;
    }
    return out;
  }
  const int cj = v.comp[j];
  const double rx = v.x[i] - v.x[j];
  const double ry = v.y[i] - v.y[j];
  const double r2 = rx * rx + ry * ry;
  const double wj = v.w[j];
  const double dn = (rx * v.nx[j] + ry * v.ny[j]) / (kPi * r2 * r2);
  const double c = wj * dn;
  const double ra = (a == 0 || a != b) ? rx : ry;  // out[2] = out[1] = (c*rx)*ry
  const double rb = (b == 1 || a != b) ? ry : rx;
  double out = c * ra * rb;
  if (single_layer(v, cj)) {
    const double sc = wj * c4 / r2;
    out += sc * ra * rb;
    if (a == b) {
      double lg = 0.0;
      bool corrected = false;
      if (ci == cj) {
        const i64 n = v.sl_n;
        const int np = v.sl_i[3 * n + i];
        int diff = v.sl_i[2 * n + i] - v.sl_i[2 * n + j];
        if (diff < 0) diff += np;
        const int locj = v.sl_i[j];
        const double xj = v.sl_d[j], jacj = v.sl_d[n + j];
        double lam = 0.0, xi = 0.0;
        if (diff == 0) {
          const int q = v.sl_i[n + i];
          lam = v.sl_tab[v.sl_i[4 * n + i] + v.sl_i[i] * q + locj];
          xi = v.sl_d[i];
          corrected = true;
        } else if (diff == 1 || diff == np - 1) {
          const int dir = diff == 1 ? 0 : 1;  // previous / next panel of i
          lam = v.sl_lam[(dir * n + i) * v.sl_qmax + locj];
          xi = v.sl_d[(2 + dir) * n + i];
          corrected = true;
        }
        if (corrected) lg = c4 * (-lam * jacj - wj * (0.5 * log(r2) - log(fabs(xj - xi))));
      }
      if (!corrected) lg = c4 * wj * (-0.5 * log(r2));
      out += lg;
    }
  }
  if (in_null(v, ci) && in_null(v, cj)) {
    const double na = a == 0 ? v.nx[i] : v.ny[i];
    const double nb = b == 0 ? v.nx[j] : v.ny[j];
    out += wj * na * nb;
  }
  return out;
}

// The whole 2 x 2 block A(2i + a, 2j + b) of `entry` with the geometry,
// the division and the logarithms formed once: every output is
// produced by exactly the operations entry() uses for it, so the bits agree.
__device__ void entry_block(const EntryView& v, i64 i, i64 j, double (&o)[2][2]) {
  const int ci = v.comp[i];
  const double c4 = 1.0 / (4.0 * kPi * v.mu);
  if (i == j) {
    const double wi = v.w[i];
    const double dl = -v.kappa[i] / (2.0 * kPi) * wi;
    const double tx = v.tx[i], ty = v.ty[i];
    const bool sl = single_layer(v, ci), nul = in_null(v, ci);
    double corr = 0.0;
    if (sl) {
      const i64 n = v.sl_n;
      const int loc = v.sl_i[i], q = v.sl_i[n + i];
      const double jac = v.sl_d[n + i];
      const double lam = v.sl_tab[v.sl_i[4 * n + i] + loc * q + loc];
      corr = c4 * (-lam * jac - wi * log(jac));
    }
    const double sm = wi * c4;
    const double nx = v.nx[i], ny = v.ny[i];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const double ta = (a == 0 || a != b) ? tx : ty;
        const double tb = (b == 1 || a != b) ? ty : tx;
        double out = dl * ta * tb;
        if (a == b) out = v.jump + out;
        if (sl) {
          out += sm * ta * tb;
          if (a == b) out += corr;
        }
        if (nul) {
          const double na = a == 0 ? nx : ny;
          const double nb = b == 0 ? nx : ny;
          out += wi * na * nb;
        }
        o[a][b] = out;
      }
    return;
  }
  const int cj = v.comp[j];
  const double rx = v.x[i] - v.x[j];
  const double ry = v.y[i] - v.y[j];
  const double r2 = rx * rx + ry * ry;
  const double wj = v.w[j];
  const double dn = (rx * v.nx[j] + ry * v.ny[j]) / (kPi * r2 * r2);
  const double c = wj * dn;
  const bool slj = single_layer(v, cj), nul = in_null(v, ci) && in_null(v, cj);
  double sc = 0.0, lg = 0.0;
  if (slj) {
    sc = wj * c4 / r2;
    bool corrected = false;
    if (ci == cj) {
      const i64 n = v.sl_n;
      const int np = v.sl_i[3 * n + i];
      int diff = v.sl_i[2 * n + i] - v.sl_i[2 * n + j];
      if (diff < 0) diff += np;
      const int locj = v.sl_i[j];
      const double xj = v.sl_d[j], jacj = v.sl_d[n + j];
      double lam = 0.0, xi = 0.0;
      if (diff == 0) {
        const int q = v.sl_i[n + i];
        lam = v.sl_tab[v.sl_i[4 * n + i] + v.sl_i[i] * q + locj];
        xi = v.sl_d[i];
        corrected = true;
      } else if (diff == 1 || diff == np - 1) {
        const int dir = diff == 1 ? 0 : 1;
        lam = v.sl_lam[(dir * n + i) * v.sl_qmax + locj];
        xi = v.sl_d[(2 + dir) * n + i];
        corrected = true;
      }
      if (corrected) lg = c4 * (-lam * jacj - wj * (0.5 * log(r2) - log(fabs(xj - xi))));
    }
    if (!corrected) lg = c4 * wj * (-0.5 * log(r2));
  }
  const double nxi = v.nx[i], nyi = v.ny[i], nxj = v.nx[j], nyj = v.ny[j];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const double ra = (a == 0 || a != b) ? rx : ry;
      const double rb = (b == 1 || a != b) ? ry : rx;
      double out = c * ra * rb;
      if (slj) {
        out += sc * ra * rb;
        if (a == b) out += lg;
      }
      if (nul) {
        const double na = a == 0 ? nxi : nyi;
        const double nb = b == 0 ? nxj : nyj;
        out += wj * na * nb;
      }
      o[a][b] = out;
    }
}

// A 2 x 2 output tile (rows r, r + 1 of columns c, c + 1 of a column-major
// block with leading dimension ld): when both index pairs are the two
// components of one node each, one entry_block; otherwise entry by entry.
// Adjacent rows leave as one 16-byte store when aligned.
__device__ __forceinline__ void tile_2x2(const EntryView& v, const i64* rl, const i64* cl, int r, int c, int nr,
                                         int nc, bool transpose, double* col0, double* col1) {
  const bool r2ok = r + 1 < nr, c2ok = c + 1 < nc;
  const i64 ra = rl[r], rb = r2ok ? rl[r + 1] : -1;
  const i64 ca = cl[c], cb = c2ok ? cl[c + 1] : -1;
  double o[2][2];
  const bool rpair = r2ok && (ra & 1) == 0 && rb == ra + 1;
  const bool cpair = c2ok && (ca & 1) == 0 && cb == ca + 1;
  if (rpair && cpair) {
    double e[2][2];
    if (!transpose) {
      entry_block(v, node_of(v, ra >> 1), node_of(v, ca >> 1), e);
      o[0][0] = e[0][0], o[0][1] = e[0][1], o[1][0] = e[1][0], o[1][1] = e[1][1];
    } else {  // tile (r, c) of A(cols, rows)^T: o[x][y] = A(cl[c + y], rl[r + x])
      entry_block(v, node_of(v, ca >> 1), node_of(v, ra >> 1), e);
      o[0][0] = e[0][0], o[0][1] = e[1][0], o[1][0] = e[0][1], o[1][1] = e[1][1];
    }
  } else {
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y) {
        const i64 ri = x ? rb : ra, cj = y ? cb : ca;
        o[x][y] = (ri >= 0 && cj >= 0) ? (transpose ? entry(v, cj, ri) : entry(v, ri, cj)) : 0.0;
      }
  }
#pragma unroll
  for (int y = 0; y < 2; ++y) {
    if (y == 1 && !c2ok) break;
    double* dst = (y ? col1 : col0) + r;
    if (r2ok && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
      *reinterpret_cast<double2*>(dst) = make_double2(o[0][y], o[1][y]);
    } else {
      dst[0] = o[0][y];
      if (r2ok) dst[1] = o[1][y];
    }
  }
}

struct M2d {
  double a00, a01, a10, a11;
  __device__ double at(int i, int j) const {
    return i == 0 ? (j == 0 ? a00 : a01) : (j == 0 ? a10 : a11);
  }
};

// kernels.cpp:13-31 (target x, source y)
__device__ M2d stokeslet(double x0, double x1, double y0, double y1, double mu) {
  const double rx = x0 - y0, ry = x1 - y1;
  const double r2 = rx * rx + ry * ry;
  const double c = 1.0 / (4.0 * kPi * mu);
  const double s = c / r2;
  const double lg = -0.5 * log(r2) * c;
  return {rx * rx * s + lg, rx * ry * s, ry * rx * s, ry * ry * s + lg};
}
__device__ M2d double_layer(double x0, double x1, double y0, double y1, double n0, double n1) {
  const double rx = x0 - y0, ry = x1 - y1;
  const double r2 = rx * rx + ry * ry;
  const double c = (rx * n0 + ry * n1) / (kPi * r2 * r2);
  return {rx * rx * c, rx * ry * c, ry * rx * c, ry * ry * c};
}
// kernels.cpp:50-72
__device__ M2d stokeslet_gradient(double x0, double x1, double y0, double y1, double mu, double d0,
                                  double d1) {
  const double rx = x0 - y0, ry = x1 - y1;
  const double r2 = rx * rx + ry * ry;
  const double rd = rx * d0 + ry * d1;
  const double c2 = 2.0 * rd / (r2 * r2);
  const double s = 4.0 * kPi * mu;
  return {((d0 * rx + rx * d0) / r2 - rx * rx * c2 - rd / r2) / s,
          ((d0 * ry + rx * d1) / r2 - rx * ry * c2) / s,
          ((d1 * rx + ry * d0) / r2 - ry * rx * c2) / s,
          ((d1 * ry + ry * d1) / r2 - ry * ry * c2 - rd / r2) / s};
}
__device__ M2d double_layer_gradient(double x0, double x1, double y0, double y1, double n0,
                                     double n1, double d0, double d1) {
  const double rx = x0 - y0, ry = x1 - y1;
  const double r2 = rx * rx + ry * ry, r4 = r2 * r2;
  const double rn = rx * n0 + ry * n1, rd = rx * d0 + ry * d1;
  const double a = rn / r4;
  const double b = (n0 * d0 + n1 * d1) / r4 - 4.0 * rn * rd / (r4 * r2);
  return {((d0 * rx + rx * d0) * a + rx * rx * b) / kPi, ((d0 * ry + rx * d1) * a + rx * ry * b) / kPi,
          ((d1 * rx + ry * d0) * a + ry * rx * b) / kPi, ((d1 * ry + ry * d1) * a + ry * ry * b) / kPi};
}

__global__ void block_jobs_kernel(EntryView v, const BlockJob* __restrict__ jobs,
                                  const i64* __restrict__ rows, const i64* __restrict__ cols,
                                  double* __restrict__ out, const i64* __restrict__ dst_cols) {
  const BlockJob jb = jobs[blockIdx.y];
  const int tr = (jb.nr + 1) / 2, tc = (jb.nc + 1) / 2;  // 2 x 2 tiles
  const i64 total = i64(tr) * tc;
  for (i64 idx = blockIdx.x * i64(blockDim.x) + threadIdx.x; idx < total;
       idx += i64(gridDim.x) * blockDim.x) {
    const int r = 2 * int(idx % tr), c = 2 * int(idx / tr);
    const i64 oc0 = jb.dst_col_off >= 0 ? dst_cols[jb.dst_col_off + c] : c;
    const i64 oc1 = c + 1 < jb.nc ? (jb.dst_col_off >= 0 ? dst_cols[jb.dst_col_off + c + 1] : c + 1) : oc0;
    tile_2x2(v, rows + jb.row_off, cols + jb.col_off, r, c, jb.nr, jb.nc, false, out + jb.out_off + oc0 * jb.ld,
             out + jb.out_off + oc1 * jb.ld);
  }
}

__global__ void submatrix_kernel(EntryView v, const i64* __restrict__ rows, i64 nr,
                                 const i64* __restrict__ cols, i64 nc, double* __restrict__ out,
                                 i64 ld) {
  const i64 total = nr * nc;
  for (i64 idx = blockIdx.x * i64(blockDim.x) + threadIdx.x; idx < total;
       idx += i64(gridDim.x) * blockDim.x) {
    const i64 r = idx % nr, c = idx / nr;
    out[r + c * ld] = entry(v, rows[r], cols[c]);
  }
}

// The four proxy functionals of one candidate node for both of its
// components (q[a][.] for component a): the kernel matrices formed once.
__device__ __forceinline__ void proxy_node(const EntryView& v, const ProxyJob& jb, i64 node, double d0, double d1,
                                           double p0, double p1, double (&q)[2][4]) {
  if (jb.kind != 1) {  // outgoing: fields at the candidate from circle sources
    const double mu = jb.kind == 2 ? 1.0 : v.mu;
    const M2d sl = stokeslet(v.x[node], v.y[node], p0, p1, mu);
    const M2d dl = double_layer(v.x[node], v.y[node], p0, p1, d0, d1);
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      q[a][0] = sl.at(a, 0);
      q[a][1] = sl.at(a, 1);
      q[a][2] = dl.at(a, 0);
      q[a][3] = dl.at(a, 1);
    }
  } else {  // incoming: candidate source evaluated on the circle
    const double nj0 = v.nx[node], nj1 = v.ny[node], wj = v.w[node];
    M2d val = double_layer(p0, p1, v.x[node], v.y[node], nj0, nj1);
    M2d grad = double_layer_gradient(p0, p1, v.x[node], v.y[node], nj0, nj1, d0, d1);
    if (single_layer(v, v.comp[node])) {
      const M2d s1 = stokeslet(p0, p1, v.x[node], v.y[node], v.mu);
      const M2d g1 = stokeslet_gradient(p0, p1, v.x[node], v.y[node], v.mu, d0, d1);
      val = {val.a00 + s1.a00, val.a01 + s1.a01, val.a10 + s1.a10, val.a11 + s1.a11};
      grad = {grad.a00 + g1.a00, grad.a01 + g1.a01, grad.a10 + g1.a10, grad.a11 + g1.a11};
    }
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      q[a][0] = wj * val.at(0, a);
      q[a][1] = wj * val.at(1, a);
      q[a][2] = wj * grad.at(0, a);
      q[a][3] = wj * grad.at(1, a);
    }
  }
}

__device__ __forceinline__ void proxy_store(const EntryView& v, const ProxyJob& jb, double* col, int s, i64 node,
                                            int a, const double (&q)[4]) {
  double* dst = col + 4 * s;
  if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    reinterpret_cast<double2*>(dst)[0] = make_double2(q[0], q[1]);
    reinterpret_cast<double2*>(dst)[1] = make_double2(q[2], q[3]);
  } else {
    dst[0] = q[0];
    dst[1] = q[1];
    dst[2] = q[2];
    dst[3] = q[3];
  }
  if (s == 0 && jb.with_null) {
    const bool nul = in_null(v, v.comp[node]);
    const double nn = a == 0 ? v.nx[node] : v.ny[node];
    col[4 * jb.ns] = nul ? (jb.kind == 1 ? v.w[node] * nn : nn) : 0.0;
  }
}

// One thread per (proxy point, candidate pair): when the two candidates are
// the components of one node, its kernel matrices serve both columns.
__global__ void proxy_jobs_kernel(EntryView v, const ProxyJob* __restrict__ jobs,
                                  const i64* __restrict__ cand, double* __restrict__ out) {
  const ProxyJob jb = jobs[blockIdx.y];
  const int np = (jb.n + 1) / 2;
  const i64 total = i64(jb.ns) * np;
  for (i64 idx = blockIdx.x * i64(blockDim.x) + threadIdx.x; idx < total;
       idx += i64(gridDim.x) * blockDim.x) {
    const int s = int(idx % jb.ns), c = 2 * int(idx / jb.ns);
    const double t = 2.0 * kPi * double(s) / double(jb.ns);
    double d0, d1;
    sincos(t, &d1, &d0);  // bitwise equal to sin(t), cos(t) (scripts/sincos_check.cu), one reduction
    const double p0 = jb.cx + jb.rad * d0, p1 = jb.cy + jb.rad * d1;
    const i64 cs0 = cand[jb.cand_off + c];
    const bool two = c + 1 < jb.n;
    const i64 cs1 = two ? cand[jb.cand_off + c + 1] : -1;
    const i64 node0 = node_of(v, cs0 >> 1);
    double q[2][4];
    proxy_node(v, jb, node0, d0, d1, p0, p1, q);
    const int a0 = int(cs0 & 1);
    proxy_store(v, jb, out + jb.out_off + i64(c) * jb.ld, s, node0, a0, q[a0]);
    if (two) {
      const i64 node1 = node_of(v, cs1 >> 1);
      const int a1 = int(cs1 & 1);
      if (node1 != node0) proxy_node(v, jb, node1, d0, d1, p0, p1, q);
      proxy_store(v, jb, out + jb.out_off + i64(c + 1) * jb.ld, s, node1, a1, q[a1]);
    }
  }
}

__global__ void near_jobs_kernel(EntryView v, const NearJob* __restrict__ jobs,
                                 const i64* __restrict__ cand, const i64* __restrict__ nearv,
                                 double* __restrict__ out) {
  const NearJob jb = jobs[blockIdx.y];
  const int tr = (jb.n_near + 1) / 2, tc = (jb.n + 1) / 2;  // 2 x 2 tiles
  const i64 total = i64(tr) * tc;
  for (i64 idx = blockIdx.x * i64(blockDim.x) + threadIdx.x; idx < total;
       idx += i64(gridDim.x) * blockDim.x) {
    const int r = 2 * int(idx % tr), c = 2 * int(idx / tr);
    // output (r, c) = transpose ? A(near_r, cand_c) : A(cand_c, near_r)
    double* base = out + jb.out_off;
    tile_2x2(v, nearv + jb.near_off, cand + jb.cand_off, r, c, jb.n_near, jb.n, !jb.transpose,
             base + i64(c) * jb.ld, base + i64(c + 1 < jb.n ? c + 1 : c) * jb.ld);
  }
}

__global__ void boundary_data_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                     i64 n, const double* __restrict__ src, i64 n_src, double mu,
                                     double* __restrict__ out) {
  for (i64 i = blockIdx.x * i64(blockDim.x) + threadIdx.x; i < n; i += i64(gridDim.x) * blockDim.x) {
    double u0 = 0, u1 = 0;  // field_velocity (nystrom.cpp:394-398)
    for (i64 s = 0; s < n_src; ++s) {
      const M2d k = stokeslet(x[i], y[i], src[4 * s], src[4 * s + 1], mu);
      u0 += k.a00 * src[4 * s + 2] + k.a01 * src[4 * s + 3];
      u1 += k.a10 * src[4 * s + 2] + k.a11 * src[4 * s + 3];
    }
    out[2 * i] = u0;
    out[2 * i + 1] = u1;
  }
}


// evaluate_solution (nystrom.cpp:408-448): velocity (and pressure) at
// targets from nrhs densities; one CTA per (target, block of up to 8
// densities), nodes strided over the threads, kernel matrices formed once
// per node and applied to every density; block reduction at the end.  Also
// the closest node (first minimum) for the near-boundary flag.
constexpr int kEvalR = 8;

__global__ void __launch_bounds__(256) evaluate_kernel(EntryView v, i64 n, const double* __restrict__ tau, i64 ldt,
                                                       int nrhs, const double* __restrict__ tgt, int with_p,
                                                       double* __restrict__ vel, double* __restrict__ pre,
                                                       double* __restrict__ cdist, i64* __restrict__ cnode) {
  const int t = blockIdx.x;
  const int r0 = blockIdx.y * kEvalR;
  const int nr = min(kEvalR, nrhs - r0);
  const double px = tgt[2 * t], py = tgt[2 * t + 1];
  double u0[kEvalR], u1[kEvalR], pp[kEvalR];
#pragma unroll
  for (int q = 0; q < kEvalR; ++q) u0[q] = u1[q] = pp[q] = 0.0;
  double best = INFINITY;
  i64 bestj = 0x7fffffffffffffffLL;
  const double c4 = 1.0 / (4.0 * kPi * v.mu);
  for (i64 j = threadIdx.x; j < n; j += blockDim.x) {
    const double rx = px - v.x[j], ry = py - v.y[j];
    const double r2 = rx * rx + ry * ry;
    const double dist = sqrt(r2);
    if (dist < best) {
      best = dist;
      bestj = j;
    }
    const double wj = v.w[j], nx = v.nx[j], ny = v.ny[j];
    const double dn = (rx * nx + ry * ny) / (kPi * r2 * r2);
    double k00 = rx * rx * dn, k01 = rx * ry * dn, k11 = ry * ry * dn;
    const bool sl = single_layer(v, v.comp[j]);
    double s00 = 0, s01 = 0, s11 = 0;
    if (sl) {
      const double lg = -0.5 * log(r2) * c4, sc = c4 / r2;
      s00 = rx * rx * sc + lg;
      s01 = rx * ry * sc;
      s11 = ry * ry * sc + lg;
    }
    double pd0 = 0, pd1 = 0, ps0 = 0, ps1 = 0;
    if (with_p) {
      const double rn = rx * nx + ry * ny;
      pd0 = (v.mu / kPi) * (-nx / r2 + rx * (2.0 * rn / (r2 * r2)));
      pd1 = (v.mu / kPi) * (-ny / r2 + ry * (2.0 * rn / (r2 * r2)));
      if (sl) {
        ps0 = rx / (2.0 * kPi * r2);
        ps1 = ry / (2.0 * kPi * r2);
      }
    }
#pragma unroll
    for (int q = 0; q < kEvalR; ++q) {
      if (q >= nr) break;
      const double t0 = tau[2 * j + size_t(r0 + q) * ldt], t1 = tau[2 * j + 1 + size_t(r0 + q) * ldt];
      u0[q] += wj * (k00 * t0 + k01 * t1) + (sl ? wj * (s00 * t0 + s01 * t1) : 0.0);
      u1[q] += wj * (k01 * t0 + k11 * t1) + (sl ? wj * (s01 * t0 + s11 * t1) : 0.0);
      if (with_p) pp[q] += wj * (pd0 * t0 + pd1 * t1) + (sl ? wj * (ps0 * t0 + ps1 * t1) : 0.0);
    }
  }
  __shared__ double red[3 * kEvalR][8];
  __shared__ double rb[8];
  __shared__ long long rj[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < kEvalR; ++q) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      u0[q] += __shfl_xor_sync(0xffffffffu, u0[q], o);
      u1[q] += __shfl_xor_sync(0xffffffffu, u1[q], o);
      pp[q] += __shfl_xor_sync(0xffffffffu, pp[q], o);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const long long oj = __shfl_xor_sync(0xffffffffu, (long long)bestj, o);
    if (ob < best || (ob == best && oj < bestj)) {
      best = ob;
      bestj = oj;
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < kEvalR; ++q) {
      red[q][warp] = u0[q];
      red[kEvalR + q][warp] = u1[q];
      red[2 * kEvalR + q][warp] = pp[q];
    }
    rb[warp] = best;
    rj[warp] = bestj;
  }
  __syncthreads();
  if (threadIdx.x < nr) {
    const int q = threadIdx.x;
    double a = 0, b = 0, c = 0;
    for (int w = 0; w < 8; ++w) {
      a += red[q][w];
      b += red[kEvalR + q][w];
      c += red[2 * kEvalR + q][w];
    }
    vel[2 * (size_t(r0 + q) * gridDim.x + t)] = a;
    vel[2 * (size_t(r0 + q) * gridDim.x + t) + 1] = b;
    if (with_p) pre[size_t(r0 + q) * gridDim.x + t] = c;
  }
  if (threadIdx.x == 0 && blockIdx.y == 0) {
    double bb = rb[0];
    long long bj = rj[0];
    for (int w = 1; w < 8; ++w)
      if (rb[w] < bb || (rb[w] == bb && rj[w] < bj)) {
        bb = rb[w];
        bj = rj[w];
      }
    cdist[t] = bb;
    cnode[t] = bj;
  }
}

unsigned grid_x(i64 total, unsigned cap = 4096) {
  return unsigned(std::max<i64>(1, std::min<i64>((total + 255) / 256, cap)));
}

}  // namespace

EntryOracle::EntryOracle(const Geom& g, int formulation, double mu, cudaStream_t s,
                         const i64* d_map)
    : form_(formulation) {
  require(formulation >= 0 && formulation <= 2, "unknown formulation");
  require(mu > 0, "assembler: viscosity must be positive");
  if (formulation == SBX_INTERIOR_DIRICHLET)
    require(g.comps.size() == 1, "interior formulation expects a single curve");
  if (formulation == SBX_MIXED) require(!g.comps[0].is_hole, "mixed formulation expects wall first");
  const GeomDev& d = g.dev;
  v_.x = d.x();
  v_.y = d.y();
  v_.nx = d.nx();
  v_.ny = d.ny();
  v_.w = d.w();
  v_.kappa = d.kappa();
  v_.tx = d.tx();
  v_.ty = d.ty();
  v_.comp = d.comp.get();
  v_.map = d_map;
  v_.jump = formulation == SBX_EXTERIOR_COMBINED ? 0.5 : -0.5;
  v_.mu = mu;
  v_.form = formulation;
  std::vector<char> sl(g.comps.size(), 0);
  bool any_sl = false;
  for (size_t c = 0; c < g.comps.size(); ++c) {
    sl[c] = formulation == SBX_EXTERIOR_COMBINED || (formulation == SBX_MIXED && g.comps[c].is_hole);
    any_sl |= sl[c] != 0;
  }
  if (any_sl) {
    const SlTables& T = single_layer_tables(g, sl, s);
    v_.sl_i = T.ints.get();
    v_.sl_d = T.dbl.get();
    v_.sl_lam = T.lam.get();
    v_.sl_tab = T.tab.get();
    v_.sl_n = T.n;
    v_.sl_qmax = T.qmax;
  }
}

void EntryOracle::submatrix(const i64* d_rows, i64 nr, const i64* d_cols, i64 nc, double* d_out,
                            i64 ld, cudaStream_t s) const {
  if (nr * nc == 0) return;
  submatrix_kernel<<<grid_x(nr * nc), 256, 0, s>>>(v_, d_rows, nr, d_cols, nc, d_out, ld);
  SBX_LAUNCHED();
}

void EntryOracle::submatrix_host(const i64* rows, i64 nr, const i64* cols, i64 nc, double* out,
                                 cudaStream_t s) const {
  DevBuf<i64> dr, dc;
  DevBuf<double> dout(size_t(std::max<i64>(nr * nc, 1)));
  dr.upload(rows, size_t(nr), s);
  dc.upload(cols, size_t(nc), s);
  submatrix(dr.get(), nr, dc.get(), nc, dout.get(), nr, s);
  dout.download(out, size_t(nr * nc), s);
  SBX_CUDA(cudaStreamSynchronize(s));
}

void boundary_data_host(const Geom& g, i64 n_src, const double* src_xyf, double mu, double* out,
                        cudaStream_t s) {
  const i64 n = g.n_nodes();
  DevBuf<double> ds, dout(size_t(2 * n));
  ds.upload(src_xyf, size_t(4 * n_src), s);
  boundary_data_kernel<<<grid_x(n), 256, 0, s>>>(g.dev.x(), g.dev.y(), n, ds.get(), n_src, mu,
                                                 dout.get());
  SBX_LAUNCHED();
  dout.download(out, size_t(2 * n), s);
  SBX_CUDA(cudaStreamSynchronize(s));
}


void evaluate_solution_host(const Geom& g, int formulation, double mu, const double* tau, i64 ldt, i64 nrhs,
                            const double* targets, i64 n_targets, bool with_pressure, double* velocity,
                            double* pressure, unsigned char* near, cudaStream_t s) {
  require(ldt >= 2 * g.n_nodes(), "evaluate_solution: density size mismatch");
  if (n_targets == 0 || nrhs == 0) return;
  EntryOracle eo(g, formulation, mu, s);
  const i64 n = g.n_nodes();
  DevBuf<double> dt, dg, dv(static_cast<size_t>(2 * n_targets * nrhs)),
      dp(static_cast<size_t>(std::max<i64>(1, n_targets * nrhs))), dd(static_cast<size_t>(n_targets));
  DevBuf<i64> dj(static_cast<size_t>(n_targets));
  dt.resize(size_t(ldt * nrhs));
  SBX_CUDA(cudaMemcpyAsync(dt.get(), tau, size_t(ldt * nrhs) * 8, cudaMemcpyHostToDevice, s));
  dg.upload(targets, size_t(2 * n_targets), s);
  dim3 grid(unsigned(n_targets), unsigned((nrhs + kEvalR - 1) / kEvalR));
  evaluate_kernel<<<grid, 256, 0, s>>>(eo.view(), n, dt.get(), ldt, int(nrhs), dg.get(), with_pressure ? 1 : 0,
                                       dv.get(), dp.get(), dd.get(), dj.get());
  SBX_LAUNCHED();
  dv.download(velocity, size_t(2 * n_targets * nrhs), s);
  if (with_pressure && pressure) dp.download(pressure, size_t(n_targets * nrhs), s);
  std::vector<double> cd(static_cast<size_t>(n_targets));
  std::vector<i64> cj(static_cast<size_t>(n_targets));
  dd.download(cd.data(), cd.size(), s);
  dj.download(cj.data(), cj.size(), s);
  SBX_CUDA(cudaStreamSynchronize(s));
  if (near)  // within one local panel length of the curve (nystrom.cpp:444-445)
    for (i64 t = 0; t < n_targets; ++t)
      near[t] = cd[size_t(t)] < g.panel_arclength(g.panel_of[size_t(cj[size_t(t)])]) ? 1 : 0;
}

void launch_block_jobs(const EntryView& v, const BlockJob* d_jobs, int n_jobs, i64 max_entries,
                       const i64* d_rows, const i64* d_cols, double* out, cudaStream_t s,
                       const i64* d_dst_cols) {
  if (n_jobs == 0 || max_entries == 0) return;
  dim3 grid(grid_x(max_entries, 64), unsigned(n_jobs));
  block_jobs_kernel<<<grid, 256, 0, s>>>(v, d_jobs, d_rows, d_cols, out, d_dst_cols);
  SBX_LAUNCHED();
}

void launch_proxy_jobs(const EntryView& v, const ProxyJob* d_jobs, int n_jobs, int max_rows,
                       int max_n, const i64* d_cand, double* out, cudaStream_t s) {
  if (n_jobs == 0) return;
  dim3 grid(grid_x(i64(max_rows) * max_n, 64), unsigned(n_jobs));
  proxy_jobs_kernel<<<grid, 256, 0, s>>>(v, d_jobs, d_cand, out);
  SBX_LAUNCHED();
}

void launch_near_jobs(const EntryView& v, const NearJob* d_jobs, int n_jobs, i64 max_entries,
                      const i64* d_cand, const i64* d_near, double* out, cudaStream_t s) {
  if (n_jobs == 0 || max_entries == 0) return;
  dim3 grid(grid_x(max_entries, 64), unsigned(n_jobs));
  near_jobs_kernel<<<grid, 256, 0, s>>>(v, d_jobs, d_cand, d_near, out);
  SBX_LAUNCHED();
}

std::vector<double> HostEntries::block(const i64* rows, i64 nr, const i64* cols, i64 nc) const {
  std::vector<double> b(static_cast<size_t>(nr * nc), 0.0);
  if (nr > 0 && nc > 0) fn(ctx, rows, nr, cols, nc, b.data());
  return b;
}

void host_block_jobs(const HostEntries& h, const std::vector<BlockJob>& jobs, const std::vector<i64>& rows,
                     const std::vector<i64>& cols, double* out, cudaStream_t s) {
  for (const auto& j : jobs) {
    require(j.dst_col_off < 0, "custom entries: scattered block columns are not supported");
    if (j.nr == 0 || j.nc == 0) continue;
    const auto b = h.block(rows.data() + j.row_off, j.nr, cols.data() + j.col_off, j.nc);
    SBX_CUDA(cudaMemcpy2DAsync(out + j.out_off, size_t(j.ld) * 8, b.data(), size_t(j.nr) * 8, size_t(j.nr) * 8,
                               size_t(j.nc), cudaMemcpyHostToDevice, s));
    SBX_CUDA(cudaStreamSynchronize(s));  // b is a temporary
  }
}

void host_near_jobs(const HostEntries& h, const std::vector<NearJob>& jobs, const std::vector<i64>& cand,
                    const std::vector<i64>& near, double* out, cudaStream_t s) {
  for (const auto& j : jobs) {
    if (j.n == 0 || j.n_near == 0) continue;
    const i64* c = cand.data() + j.cand_off;
    const i64* nv = near.data() + j.near_off;
    // W^T rows [out_off, out_off + n_near) x the n candidate columns:
    // row ID (transpose 0): A(cand, near)^T; column ID: A(near, cand)
    std::vector<double> wt(static_cast<size_t>(j.n_near) * j.n);
    if (j.transpose == 0) {
      const auto b = h.block(c, j.n, nv, j.n_near);  // n x n_near
      for (int r = 0; r < j.n_near; ++r)
        for (int q = 0; q < j.n; ++q) wt[size_t(r) + size_t(q) * j.n_near] = b[size_t(q) + size_t(r) * j.n];
    } else {
      wt = h.block(nv, j.n_near, c, j.n);
    }
    SBX_CUDA(cudaMemcpy2DAsync(out + j.out_off, size_t(j.ld) * 8, wt.data(), size_t(j.n_near) * 8,
                               size_t(j.n_near) * 8, size_t(j.n), cudaMemcpyHostToDevice, s));
    SBX_CUDA(cudaStreamSynchronize(s));
  }
}

}  // namespace sbx
