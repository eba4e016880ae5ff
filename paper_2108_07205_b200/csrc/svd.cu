// Dense SVD on the device: one-sided (Hestenes) Jacobi with the round-robin
// tournament ordering, for the diagnostic paths of the reference that call
// Eigen::BDCSVD -- truncated_svd (idlib.cpp:134-154) behind svd_optimal
// (lowrank.cpp:329-362) and dense_cond / factor_cond of
// conditioning_report (els.cpp:205-270).
//
// Each sweep is n-1 steps; a step rotates n/2 disjoint column pairs, one CTA
// per pair (three column dot products over the rows, the Jacobi rotation
// that orthogonalises the pair, applied to both columns of the working
// matrix and of V).  Sweeps repeat until no pair needed a rotation
// (|a_i . a_j| <= tol sqrt(|a_i|^2 |a_j|^2), tol = 4 eps).  One-sided
// Jacobi is accurate to working precision relative to each singular value,
// so the eps-rank rule s_k > eps s_0 counts the same values BDCSVD does up
// to rounding.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <numeric>

#include "dense.hpp"
#include "svd.hpp"

namespace sbx {

namespace {

constexpr int kJT = 256;

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  return red[0];
}

__global__ void __launch_bounds__(kJT) jacobi_step_kernel(double* __restrict__ W, int m, int ldw,
                                                         double* __restrict__ V, int nv, int ldv,
                                                         const int2* __restrict__ pairs, int* __restrict__ rotated) {
  __shared__ double red[kJT / 32];
  __shared__ double cs[2];
  const int2 pr = pairs[blockIdx.x];
  double* ai = W + size_t(pr.x) * ldw;
  double* aj = W + size_t(pr.y) * ldw;
  double a = 0.0, b = 0.0, g = 0.0;
  for (int r = threadIdx.x; r < m; r += kJT) {
    const double x = ai[r], y = aj[r];
    a = fma(x, x, a);
    b = fma(y, y, b);
    g = fma(x, y, g);
  }
  a = block_sum(a, red);
  b = block_sum(b, red);
  g = block_sum(g, red);
  if (threadIdx.x == 0) {
    double c = 1.0, s = 0.0;
    if (a > 0.0 && b > 0.0 && fabs(g) > 4.0 * DBL_EPSILON * sqrt(a) * sqrt(b)) {
      const double zeta = (b - a) / (2.0 * g);
      const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
      c = 1.0 / sqrt(1.0 + t * t);
      s = c * t;
      *rotated = 1;
    }
    cs[0] = c;
    cs[1] = s;
  }
  __syncthreads();
  const double c = cs[0], s = cs[1];
  if (s == 0.0) return;
  // [a_i a_j] <- [a_i a_j] [[c, s], [-s, c]]  (makes a_i . a_j vanish)
  for (int r = threadIdx.x; r < m; r += kJT) {
    const double x = ai[r], y = aj[r];
    ai[r] = c * x - s * y;
    aj[r] = s * x + c * y;
  }
  if (V) {
    double* vi = V + size_t(pr.x) * ldv;
    double* vj = V + size_t(pr.y) * ldv;
    for (int r = threadIdx.x; r < nv; r += kJT) {
      const double x = vi[r], y = vj[r];
      vi[r] = c * x - s * y;
      vj[r] = s * x + c * y;
    }
  }
}

__global__ void col_norms_kernel(const double* __restrict__ W, int m, int ldw, double* __restrict__ out) {
  __shared__ double red[kJT / 32];
  const double* a = W + size_t(blockIdx.x) * ldw;
  double s = 0.0;
  for (int r = threadIdx.x; r < m; r += kJT) s = fma(a[r], a[r], s);
  s = block_sum(s, red);
  if (threadIdx.x == 0) out[blockIdx.x] = sqrt(s);
}

// dst(:, q) = src(:, ord[q]) * (scale ? 1 / sv[q] : 1)
__global__ void gather_cols_kernel(const double* __restrict__ src, int rows, int lds, const int* __restrict__ ord,
                                   const double* __restrict__ sv, double* __restrict__ dst, int ldd) {
  const int q = blockIdx.x;
  const double f = sv ? 1.0 / sv[q] : 1.0;
  const double* a = src + size_t(ord[q]) * lds;
  for (int r = threadIdx.x; r < rows; r += blockDim.x) dst[r + size_t(q) * ldd] = a[r] * f;
}

__global__ void identity_kernel(double* V, int n, int ldv) {
  for (int c = blockIdx.x; c < n; c += gridDim.x)
    for (int r = threadIdx.x; r < n; r += blockDim.x) V[r + size_t(c) * ldv] = r == c ? 1.0 : 0.0;
}

// Round-robin tournament: n (even) players, n-1 rounds of n/2 disjoint pairs.
std::vector<int2> tournament(int n) {
  std::vector<int2> out;
  out.reserve(size_t(n - 1) * size_t(n / 2));
  std::vector<int> p(static_cast<size_t>(n));
  std::iota(p.begin(), p.end(), 0);
  for (int r = 0; r < n - 1; ++r) {
    for (int i = 0; i < n / 2; ++i) {
      const int x = p[size_t(i)], y = p[size_t(n - 1 - i)];
      out.push_back(make_int2(std::min(x, y), std::max(x, y)));
    }
    std::rotate(p.begin() + 1, p.end() - 1, p.end());  // keep p[0], rotate the rest
  }
  return out;
}

// Orthogonalises the columns of W (m x n, n even, ld m) in place; V (n x n)
// accumulates the rotations when non-null.
void jacobi_sweeps(double* W, int m, int n, double* V, cudaStream_t s) {
  if (n < 2) return;
  const std::vector<int2> pairs = tournament(n);
  DevBuf<int2> d_pairs;
  d_pairs.upload(pairs, s);
  DevBuf<int> flag(1);
  const int half = n / 2;
  for (int sweep = 0; sweep < 60; ++sweep) {
    SBX_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), s));
    for (int r = 0; r < n - 1; ++r) {
      jacobi_step_kernel<<<half, kJT, 0, s>>>(W, m, m, V, n, n, d_pairs.get() + size_t(r) * half, flag.get());
      SBX_LAUNCHED();
    }
    int h = 0;
    flag.download(&h, 1, s);
    SBX_CUDA(cudaStreamSynchronize(s));
    if (!h) return;
  }
  throw Error(2, "jacobi svd: no convergence after 60 sweeps");
}

// Tall working copy (rows >= cols, cols padded to even) of A or A^T.
struct Work {
  DevBuf<double> W;
  int m = 0, n = 0, npad = 0;
  bool transposed = false;
};

Work make_work(const double* A, i64 m, i64 n, i64 lda, cudaStream_t s) {
  require(m <= i64(INT32_MAX) && n <= i64(INT32_MAX), "svd: matrix too large");
  Work w;
  w.transposed = m < n;
  w.m = int(w.transposed ? n : m);
  w.n = int(w.transposed ? m : n);
  w.npad = w.n + (w.n & 1);
  w.W.resize(size_t(w.m) * size_t(std::max(w.npad, 1)));
  w.W.zero(s);
  if (w.n > 0)
    copy_batched({{A, w.W.get(), w.m, w.n, int(lda), w.m, w.transposed ? 1 : 0, 0}}, s);
  return w;
}

std::vector<double> norms_of(const Work& w, cudaStream_t s) {
  std::vector<double> h(size_t(w.npad));
  if (w.npad == 0) return h;
  DevBuf<double> d(static_cast<size_t>(w.npad));
  col_norms_kernel<<<w.npad, kJT, 0, s>>>(w.W.get(), w.m, w.m, d.get());
  SBX_LAUNCHED();
  d.download(h.data(), h.size(), s);
  SBX_CUDA(cudaStreamSynchronize(s));
  return h;
}

std::vector<int> descending(const std::vector<double>& v) {
  std::vector<int> ord(v.size());
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return v[size_t(a)] > v[size_t(b)]; });
  return ord;
}

}  // namespace

std::vector<double> singular_values_device(const double* A, i64 m, i64 n, i64 lda, cudaStream_t s) {
  if (m == 0 || n == 0) return {};
  Work w = make_work(A, m, n, lda, s);
  jacobi_sweeps(w.W.get(), w.m, w.npad, nullptr, s);
  const std::vector<double> nv = norms_of(w, s);
  const std::vector<int> ord = descending(nv);
  std::vector<double> out(size_t(std::min(m, n)));
  for (size_t q = 0; q < out.size(); ++q) out[q] = nv[size_t(ord[q])];
  return out;
}

TruncSvd truncated_svd_device(const double* A, i64 m, i64 n, i64 lda, double eps, cudaStream_t s) {
  TruncSvd t;
  t.m = m;
  t.n = n;
  if (m == 0 || n == 0) return t;
  Work w = make_work(A, m, n, lda, s);
  DevBuf<double> V(static_cast<size_t>(w.npad) * size_t(w.npad));
  identity_kernel<<<std::min(w.npad, 1024), 128, 0, s>>>(V.get(), w.npad, w.npad);
  SBX_LAUNCHED();
  jacobi_sweeps(w.W.get(), w.m, w.npad, V.get(), s);
  const std::vector<double> nv = norms_of(w, s);
  std::vector<int> ord = descending(nv);
  // idlib.cpp:145-148: k = #{ s_k > eps s_0 }
  i64 k = 0;
  const double s0 = nv[size_t(ord[0])];
  if (s0 > 0.0)
    while (k < i64(std::min(m, n)) && nv[size_t(ord[size_t(k)])] > eps * s0) ++k;
  t.k = k;
  t.sv.resize(size_t(k));
  for (i64 q = 0; q < k; ++q) t.sv[size_t(q)] = nv[size_t(ord[size_t(q)])];
  if (k == 0) return t;
  ord.resize(size_t(k));
  DevBuf<int> d_ord;
  d_ord.upload(ord, s);
  DevBuf<double> d_sv;
  d_sv.upload(t.sv, s);
  // tall side: left vectors = W(:, ord) / s; short side: V(:, ord)
  DevBuf<double> left(static_cast<size_t>(w.m) * size_t(k)), right(static_cast<size_t>(w.n) * size_t(k));
  gather_cols_kernel<<<unsigned(k), 256, 0, s>>>(w.W.get(), w.m, w.m, d_ord.get(), d_sv.get(), left.get(), w.m);
  SBX_LAUNCHED();
  gather_cols_kernel<<<unsigned(k), 256, 0, s>>>(V.get(), w.n, w.npad, d_ord.get(), nullptr, right.get(), w.n);
  SBX_LAUNCHED();
  if (w.transposed) {  // A^T = L S R^T  =>  A = R S L^T
    t.U = std::move(right);
    t.V = std::move(left);
  } else {
    t.U = std::move(left);
    t.V = std::move(right);
  }
  SBX_CUDA(cudaStreamSynchronize(s));
  return t;
}

__global__ void sv_vt_kernel(const double* __restrict__ V, int n, int k, const double* __restrict__ sv,
                             double* __restrict__ R, i64 ldr) {
  const i64 total = i64(n) * k;
  for (i64 e = blockIdx.x * i64(blockDim.x) + threadIdx.x; e < total; e += i64(gridDim.x) * blockDim.x) {
    const int q = int(e % k), j = int(e / k);  // R(q, j): consecutive threads along a column of R
    R[q + size_t(j) * ldr] = sv[q] * V[j + size_t(q) * n];
  }
}

void svd_sv_vt(const TruncSvd& t, double* R, i64 ldr, cudaStream_t s) {
  if (t.k == 0 || t.n == 0) return;
  DevBuf<double> d_sv;
  d_sv.upload(t.sv, s);
  const i64 total = t.n * t.k;
  sv_vt_kernel<<<unsigned(std::min<i64>((total + 255) / 256, 4096)), 256, 0, s>>>(t.V.get(), int(t.n), int(t.k),
                                                                                 d_sv.get(), R, ldr);
  SBX_LAUNCHED();
  SBX_CUDA(cudaStreamSynchronize(s));
}

}  // namespace sbx
