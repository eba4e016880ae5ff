// Batched small dense linear algebra on sm_100a (see dense.hpp).
// One CTA per problem; matrices are staged in shared memory when they fit
// and otherwise factored in place in global memory (L2 resident for the
// sizes of this workload).  GEMM tiles use FP64 tensor cores
// (mma.sync.m8n8k4.f64 -> SASS DMMA).
#include <cfloat>
#include <cstdlib>

#include <algorithm>
#include <memory>
#include <mutex>

#include "dense.hpp"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace sbx {

namespace {

constexpr int kT = 512;
constexpr int kWarps = kT / 32;
constexpr size_t kSmemCap = 200 * 1024;

template <class T>
struct JobTable {
  DevBuf<T> d;
  const T* upload(const std::vector<T>& h, cudaStream_t s) {
    d.reserve(h.size());
    SBX_CUDA(cudaMemcpyAsync(d.get(), h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, s));
    return d.get();
  }
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum; all threads get the result. red: >= kWarps doubles.
__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = l < kWarps ? red[l] : 0.0;
  t = warp_sum(t);
  return t;
}

// Block-wide first-max (largest value, smallest index on ties).
__device__ void block_argmax(double v, int idx, double* rv, int* ri, double& out_v, int& out_i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > v || (ov == v && oi < idx)) {
      v = ov;
      idx = oi;
    }
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) {
    rv[w] = v;
    ri[w] = idx;
  }
  __syncthreads();
  v = l < kWarps ? rv[l] : -1.0;
  idx = l < kWarps ? ri[l] : 0x7fffffff;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > v || (ov == v && oi < idx)) {
      v = ov;
      idx = oi;
    }
  }
  out_v = v;
  out_i = idx;
}

// Applies the Householder reflector (1, v[j+1..M)) with tau to U columns at
// once (U independent load streams per lane), then the xGEQPF norm
// downdate of ColPivHouseholderQR for each.  col[u] == nullptr skips a slot.
template <int U>
__device__ __forceinline__ void reflect_cols(double* const (&col)[U], const int (&slot)[U],
                                             const double* v, int j, int M, double tau, bool pivot,
                                             double* upd, double* dir, double thr, int lane) {
  if (M - j > 1 && tau != 0.0) {
    double d[U];
#pragma unroll
    for (int u = 0; u < U; ++u) d[u] = 0.0;
    for (int i = j + 1 + lane; i < M; i += 32) {
      const double vi = v[i];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (col[u]) d[u] += vi * col[u][i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int u = 0; u < U; ++u) d[u] += __shfl_xor_sync(0xffffffffu, d[u], o);
    double tw[U];
#pragma unroll
    for (int u = 0; u < U; ++u) tw[u] = col[u] ? tau * (d[u] + col[u][j]) : 0.0;
    for (int i = j + 1 + lane; i < M; i += 32) {
      const double vi = v[i];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (col[u]) col[u][i] -= vi * tw[u];
    }
    __syncwarp();
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (col[u]) col[u][j] -= tw[u];
    }
    __syncwarp();
  }
  if (!pivot) return;
  // lane u downdates slot u (same arithmetic as one column at a time); the
  // rare recomputations from the remaining rows take the whole warp
  const double* mc = nullptr;
  int ms = 0;
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (lane == u) {
      mc = col[u];
      ms = slot[u];
    }
  bool rec = false;
  if (lane < U && mc) {
    const double uu = upd[ms];
    if (uu != 0.0) {
      double t = fabs(mc[j]) / uu;
      t = (1.0 + t) * (1.0 - t);
      t = t < 0.0 ? 0.0 : t;
      const double rr = uu / dir[ms];
      if (t * rr * rr <= thr)
        rec = true;
      else
        upd[ms] = uu * sqrt(t);
    }
  }
  unsigned todo = __ballot_sync(0xffffffffu, rec);
  while (todo) {
    const int u = __ffs(todo) - 1;
    todo &= todo - 1;
    const double* cu = nullptr;
    int su = 0;
#pragma unroll
    for (int q = 0; q < U; ++q)
      if (q == u) {
        cu = col[q];
        su = slot[q];
      }
    double sacc = 0.0;
    for (int i = j + 1 + lane; i < M; i += 32) sacc += cu[i] * cu[i];
    sacc = warp_sum(sacc);
    if (lane == 0) upd[su] = dir[su] = sqrt(sacc);
  }
  __syncwarp();
}

// ---------------------------------------------------------------- QR / CPQR
// Householder QR of A (M x n, ld lda) by one CTA; with `pivot` it is
// Eigen's ColPivHouseholderQR.  Columns are not moved: the pivot of step j
// is applied in place and perm[l] records the physical (= original) column
// at logical position l, so R(i, l) = A(i, perm[l]) (interp uses perm as
// its column map).  Ties go to the smallest logical position, as Eigen's
// first-max over the current column order.  Four barriers per step.
// Scratch: upd, dir (n doubles), pos, lphys (n ints), red (32), ired (32),
// sc (8).  Returns the number of completed steps.
__device__ int cpqr_core(double* A, int M, int n, int lda, bool pivot, int steps_max,
                         double stop_eps, int* perm, double* diag, double* upd, double* dir,
                         int* pos, int* lphys, double* red, int* ired, double* sc) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int size = min(M, n);
  for (int c = tid; c < n; c += kT) {
    pos[c] = c;
    lphys[c] = c;
  }
  for (int c = tid; c < size; c += kT) diag[c] = 0.0;
  if (pivot) {
    for (int c = warp; c < n; c += kWarps) {
      double s = 0.0;
      for (int i = lane; i < M; i += 32) {
        const double v = A[i + size_t(c) * lda];
        s += v * v;
      }
      s = warp_sum(s);
      if (lane == 0) upd[c] = dir[c] = sqrt(s);
    }
  }
  __syncthreads();
  const double thr = sqrt(DBL_EPSILON);
  int done = 0;
  double r00 = 0.0;
  for (int j = 0; j < steps_max; ++j) {
    int p = lphys[j];
    if (pivot) {  // first max of the updated norms over logical positions >= j
      double bv = -1.0;
      int bp = 0x7fffffff, bq = -1;
      for (int c = tid; c < n; c += kT) {
        const int lc = pos[c];
        if (lc >= j && (upd[c] > bv || (upd[c] == bv && lc < bp))) {
          bv = upd[c];
          bp = lc;
          bq = c;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int op = __shfl_xor_sync(0xffffffffu, bp, o);
        const int oq = __shfl_xor_sync(0xffffffffu, bq, o);
        if (ov > bv || (ov == bv && op < bp)) {
          bv = ov;
          bp = op;
          bq = oq;
        }
      }
      if (lane == 0) {
        red[warp] = bv;
        ired[warp] = bp;
        ired[kWarps + warp] = bq;
      }
      __syncthreads();  // (1)
      bv = -1.0;
      bp = 0x7fffffff;
      for (int w = 0; w < kWarps; ++w)
        if (red[w] > bv || (red[w] == bv && ired[w] < bp)) {
          bv = red[w];
          bp = ired[w];
          bq = ired[kWarps + w];
        }
      p = bq;
    }
    // Householder vector of the pivot column (makeHouseholderInPlace): the
    // tail norm is a CTA-wide reduction, beta / tau are formed redundantly
    // by every thread, the scaling is spread over the CTA
    double* pc = A + size_t(p) * lda;
    {
      double part = 0.0;
      for (int i = j + 1 + tid; i < M; i += kT) part += pc[i] * pc[i];
      const double s = block_sum(part, red);
      const double c0 = pc[j];
      double tau = 0.0, beta = c0, denom = 0.0;
      if (s > DBL_MIN) {
        beta = sqrt(c0 * c0 + s);
        if (c0 >= 0.0) beta = -beta;
        denom = c0 - beta;
        tau = (beta - c0) / beta;
      }
      __syncthreads();  // every thread has read pc[j] and red
      for (int i = j + 1 + tid; i < M; i += kT) pc[i] = denom == 0.0 ? 0.0 : pc[i] / denom;
      if (tid == 0) {
        pc[j] = beta;
        diag[j] = fabs(beta);
        sc[0] = tau;
        sc[1] = beta;
        if (pivot) {  // logical swap: the column at position j moves to the pivot's slot
          const int lp = pos[p], q = lphys[j];
          lphys[lp] = q;
          pos[q] = lp;
          lphys[j] = p;
          pos[p] = j;
        }
      }
    }
    __syncthreads();  // (2)
    const double tau = sc[0], beta = sc[1];
    if (j == 0) r00 = fabs(beta);
    done = j + 1;
    if (pivot && stop_eps > 0.0 && !(fabs(beta) > stop_eps * r00)) break;
    // apply to the alive columns (4 per warp pass), then downdate their norms
    for (int c = 4 * warp; c < n; c += 4 * kWarps) {
      double* cols[4];
      int slot[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool live = c + u < n && pos[c + u] > j;
        cols[u] = live ? A + size_t(c + u) * lda : nullptr;
        slot[u] = c + u;
      }
      reflect_cols<4>(cols, slot, pc, j, M, tau, pivot, upd, dir, thr, lane);
    }
    __syncthreads();  // (3)
  }
  for (int l = tid; l < n; l += kT) perm[l] = lphys[l];
  __syncthreads();
  return done;
}

// Blocked column-pivoted QR (LAPACK dgeqp3/dlaqps organisation) with the
// pivot rule, Householder convention and norm downdating of cpqr_core.
// Within a block of kCpqrNb steps the trailing matrix is not touched: the
// pivot column gets the block's pending reflectors (A - V F^T), F gains one
// column per step (tau * (A^T v - F (V^T v))), and only the current row of
// the trailing matrix is updated (for the norm downdates).  One read of the
// trailing matrix per step instead of two reads and a write; the block ends
// early when a norm needs recomputation (LAPACK lsticc) and closes with one
// rank-jb update.  Same pivots as the unblocked loop in exact arithmetic.
constexpr int kCpqrNb = 8;

__host__ __device__ constexpr int cpqr_blocked_head(int n) { return 3 * n + 72 + kCpqrNb * n + 3 * kCpqrNb + (n + 1) / 2 + 2; }

__device__ int cpqr_core_blocked(double* A, int M, int n, int lda, int steps_max, double stop_eps, int* perm,
                                 double* diag, double* upd, double* dir, int* pos, int* lphys, double* red,
                                 int* ired, double* sc, double* F, double* aux, double* vrow, int* bp,
                                 int* rec) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int size = min(M, n);
  __shared__ int s_anyrec;
  for (int c = tid; c < n; c += kT) {
    pos[c] = c;
    lphys[c] = c;
    rec[c] = 0;
  }
  for (int c = tid; c < size; c += kT) diag[c] = 0.0;
  for (int c = warp; c < n; c += kWarps) {
    double s = 0.0;
    for (int i = lane; i < M; i += 32) {
      const double v = A[i + size_t(c) * lda];
      s += v * v;
    }
    s = warp_sum(s);
    if (lane == 0) upd[c] = dir[c] = sqrt(s);
  }
  if (tid == 0) s_anyrec = 0;
  __syncthreads();
  const double thr = sqrt(DBL_EPSILON);
  int done = 0, j = 0;
  double r00 = 0.0;
  bool stop = false;
  while (j < steps_max && !stop) {
    int nbk = 0;  // steps taken in this block
    for (; nbk < kCpqrNb && j < steps_max; ++nbk, ++j) {
      // (1) first max of the partial norms over logical positions >= j
      double bv = -1.0;
      int bpos = 0x7fffffff, bq = -1;
      for (int c = tid; c < n; c += kT) {
        const int lc = pos[c];
        if (lc >= j && (upd[c] > bv || (upd[c] == bv && lc < bpos))) {
          bv = upd[c];
          bpos = lc;
          bq = c;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int op = __shfl_xor_sync(0xffffffffu, bpos, o);
        const int oq = __shfl_xor_sync(0xffffffffu, bq, o);
        if (ov > bv || (ov == bv && op < bpos)) {
          bv = ov;
          bpos = op;
          bq = oq;
        }
      }
      if (lane == 0) {
        red[warp] = bv;
        ired[warp] = bpos;
        ired[kWarps + warp] = bq;
      }
      __syncthreads();
      bv = -1.0;
      bpos = 0x7fffffff;
      for (int w = 0; w < kWarps; ++w)
        if (red[w] > bv || (red[w] == bv && ired[w] < bpos)) {
          bv = red[w];
          bpos = ired[w];
          bq = ired[kWarps + w];
        }
      const int p = bq;
      double* pc = A + size_t(p) * lda;
      // (3) pending reflectors of the block on the pivot column, rows >= j
      for (int i = j + tid; i < M; i += kT) {
        double acc = pc[i];
        for (int b = 0; b < nbk; ++b) acc -= A[i + size_t(bp[b]) * lda] * F[size_t(p) * kCpqrNb + b];
        pc[i] = acc;
      }
      __syncthreads();
      if (tid == 0) {  // (2) logical swap: the column at position j moves to the pivot's slot
        const int lp = pos[p], q = lphys[j];
        lphys[lp] = q;
        pos[q] = lp;
        lphys[j] = p;
        pos[p] = j;
        bp[nbk] = p;
      }
      // (4) Householder vector (makeHouseholderInPlace)
      double part = 0.0;
      for (int i = j + 1 + tid; i < M; i += kT) part += pc[i] * pc[i];
      const double tail = block_sum(part, red);
      const double c0 = pc[j];
      double tau = 0.0, beta = c0, denom = 0.0;
      if (tail > DBL_MIN) {
        beta = sqrt(c0 * c0 + tail);
        if (c0 >= 0.0) beta = -beta;
        denom = c0 - beta;
        tau = (beta - c0) / beta;
      }
      for (int i = j + 1 + tid; i < M; i += kT) pc[i] = denom == 0.0 ? 0.0 : pc[i] / denom;
      if (j == 0) r00 = fabs(beta);
      if (tid == 0) {
        diag[j] = fabs(beta);
        pc[j] = beta;
      }
      done = j + 1;
      __syncthreads();
      if (!(fabs(beta) > stop_eps * r00) && stop_eps > 0.0) {
        stop = true;
        ++j;
        break;
      }
      // (5) aux_b = V_b^T v over rows >= j, then F(:, nbk) for the live columns
      if (warp < nbk) {
        const double* vb = A + size_t(bp[warp]) * lda;
        double a = lane == 0 ? vb[j] : 0.0;  // v_j = 1
        for (int i = j + 1 + lane; i < M; i += 32) a += vb[i] * pc[i];
        a = warp_sum(a);
        if (lane == 0) aux[warp] = a;
      }
      if (tid < nbk) vrow[tid] = A[j + size_t(bp[tid]) * lda];
      __syncthreads();
      for (int c = warp; c < n; c += kWarps) {
        if (pos[c] <= j) continue;
        const double* col = A + size_t(c) * lda;
        double a = lane == 0 ? col[j] : 0.0;
        for (int i = j + 1 + lane; i < M; i += 32) a += col[i] * pc[i];
        a = warp_sum(a);
        if (lane == 0) {
          double corr = 0.0;
          for (int b = 0; b < nbk; ++b) corr += F[size_t(c) * kCpqrNb + b] * aux[b];
          F[size_t(c) * kCpqrNb + nbk] = tau * (a - corr);
        }
      }
      __syncthreads();
      // (6) current row of the live columns, (7) norm downdating
      for (int c = tid; c < n; c += kT) {
        if (pos[c] <= j) continue;
        double a = A[j + size_t(c) * lda];
        for (int b = 0; b < nbk; ++b) a -= vrow[b] * F[size_t(c) * kCpqrNb + b];
        a -= F[size_t(c) * kCpqrNb + nbk];  // v_j = 1
        A[j + size_t(c) * lda] = a;
        const double uu = upd[c];
        if (uu == 0.0) continue;
        double t = fabs(a) / uu;
        t = (1.0 + t) * (1.0 - t);
        t = t < 0.0 ? 0.0 : t;
        const double rr = uu / dir[c];
        if (t * rr * rr <= thr) {
          rec[c] = 1;
          s_anyrec = 1;
        } else {
          upd[c] = uu * sqrt(t);
        }
      }
      __syncthreads();
      if (s_anyrec) {  // a norm must be recomputed from the updated column: close the block
        ++nbk;
        ++j;
        break;
      }
    }
    if (stop) break;
    // rank-nbk update of the live columns below the block's last row
    const int r0 = j;
    for (int c = warp; c < n; c += kWarps) {
      if (pos[c] < r0) continue;
      double* col = A + size_t(c) * lda;
      double f[kCpqrNb];
#pragma unroll
      for (int b = 0; b < kCpqrNb; ++b) f[b] = b < nbk ? F[size_t(c) * kCpqrNb + b] : 0.0;
      for (int i = r0 + lane; i < M; i += 32) {
        double acc = col[i];
#pragma unroll
        for (int b = 0; b < kCpqrNb; ++b)
          if (b < nbk) acc -= A[i + size_t(bp[b]) * lda] * f[b];
        col[i] = acc;
      }
    }
    __syncthreads();
    if (s_anyrec) {
      for (int c = warp; c < n; c += kWarps) {
        if (!rec[c]) continue;
        const double* col = A + size_t(c) * lda;
        double s2 = 0.0;
        for (int i = r0 + lane; i < M; i += 32) s2 += col[i] * col[i];
        s2 = warp_sum(s2);
        if (lane == 0) {
          upd[c] = dir[c] = sqrt(s2);
          rec[c] = 0;
        }
      }
      __syncthreads();
      if (tid == 0) s_anyrec = 0;
      __syncthreads();
    }
  }
  for (int l = tid; l < n; l += kT) perm[l] = lphys[l];
  __syncthreads();
  return done;
}

__global__ void __launch_bounds__(kT) qr_kernel(const QrJob* __restrict__ jobs, int smem_doubles, int blocked) {
  extern __shared__ double sm[];
  const QrJob jb = jobs[blockIdx.x];
  const int M = jb.M, n = jb.n;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* upd = sm;
  double* dir = upd + n;
  int* pos = reinterpret_cast<int*>(dir + n);
  int* lphys = pos + n;
  double* red = dir + 2 * n;                     // 32 (after the two int tables)
  int* ired = reinterpret_cast<int*>(red + 32);  // 32 (+32)
  double* sc = red + 64;                         // shared scalars (8)
  double* F = sc + 8;                            // blocked CPQR: n x kCpqrNb
  double* aux = F + size_t(kCpqrNb) * n;
  double* vrow = aux + kCpqrNb;
  int* bp = reinterpret_cast<int*>(vrow + kCpqrNb);
  int* rec = bp + kCpqrNb;
  const size_t head = blocked ? size_t(cpqr_blocked_head(n)) : size_t(3 * n + 72);
  double* mat = sm + head;
  const bool in_smem = head + size_t(M) * n <= size_t(smem_doubles);
  double* A = jb.a;
  int lda = jb.lda;
  if (in_smem) {
    for (int c = warp; c < n; c += kWarps)
      for (int i = lane; i < M; i += 32) mat[i + size_t(c) * M] = jb.a[i + size_t(c) * jb.lda];
    A = mat;
    lda = M;
  }
  const int size = min(M, n);
  const int steps_max = jb.max_steps > 0 ? min(size, jb.max_steps) : size;
  const int done =
      (blocked && jb.pivot)
          ? cpqr_core_blocked(A, M, n, lda, steps_max, jb.stop_eps, jb.perm, jb.diag, upd, dir, pos, lphys, red,
                              ired, sc, F, aux, vrow, bp, rec)
          : cpqr_core(A, M, n, lda, jb.pivot != 0, steps_max, jb.stop_eps, jb.perm, jb.diag, upd, dir, pos,
                      lphys, red, ired, sc);
  if (tid == 0 && jb.steps) *jb.steps = done;
  if (in_smem) {
    __syncthreads();
    for (int c = warp; c < n; c += kWarps)
      for (int i = lane; i < M; i += 32) jb.a[i + size_t(c) * jb.lda] = mat[i + size_t(c) * M];
  }
}

// Tall problems (M > n, n <= 144): a streaming TSQR first reduces W^T to its
// n x n triangular factor R0 in shared memory, then the Eigen CPQR runs on
// R0 in shared memory.  Column norms of R0 equal those of W^T, so the pivot
// order, |r_jj| and R11^{-1} R12 are those of CPQR(W^T) in exact arithmetic.
//
// TSQR: 128-row blocks of W^T live in registers (column c owned by warp
// c % 16, 4 rows per lane); each Householder step is one barrier — the warp
// owning column j+1 updates it first and publishes the next reflector
// (look-ahead) while the other warps finish step j.  R (pivoted) is written
// to the first n rows of the job matrix.
constexpr int kTsqrSlots = 9;  // columns per warp: n <= 16 * 9 = 144
constexpr int kTsqrRpl = 4;    // rows per lane: 128-row blocks
constexpr int kTsqrBm = 32 * kTsqrRpl;

__device__ __forceinline__ void tsqr_reflector(double (&b)[kTsqrRpl], double* R, int n, int jn,
                                               double* vbuf, double* tauv, int lane) {
  double sq = 0.0;
#pragma unroll
  for (int r = 0; r < kTsqrRpl; ++r) sq += b[r] * b[r];
  sq = warp_sum(sq);
  const double c0 = R[jn + jn * n];
  double tau = 0.0, beta = c0, denom = 0.0;
  if (sq > DBL_MIN) {
    beta = sqrt(c0 * c0 + sq);
    if (c0 >= 0.0) beta = -beta;
    denom = c0 - beta;
    tau = (beta - c0) / beta;
  }
#pragma unroll
  for (int r = 0; r < kTsqrRpl; ++r) {
    b[r] = denom == 0.0 ? 0.0 : b[r] / denom;
    vbuf[lane + 32 * r] = b[r];
  }
  if (lane == 0) {
    R[jn + jn * n] = beta;
    *tauv = tau;
  }
}

__global__ void __launch_bounds__(kT, 1) tsqr_cpqr_kernel(const QrJob* __restrict__ jobs, int blocked) {
  extern __shared__ double sm[];
  const QrJob jb = jobs[blockIdx.x];
  const int M = jb.M, n = jb.n;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* upd = sm;
  double* dir = upd + n;
  int* pos = reinterpret_cast<int*>(dir + n);
  int* lphys = pos + n;
  double* red = dir + 2 * n;
  int* ired = reinterpret_cast<int*>(red + 32);
  double* sc = red + 64;
  double* F = sc + 8;               // blocked CPQR: n x kCpqrNb
  double* aux = F + size_t(kCpqrNb) * n;
  double* vrow = aux + kCpqrNb;
  int* bp = reinterpret_cast<int*>(vrow + kCpqrNb);
  int* rec = bp + kCpqrNb;
  double* vb = sm + cpqr_blocked_head(n);  // 2 x 128 reflector buffers
  double* tauv = vb + 2 * kTsqrBm;  // 2 (+pad)
  double* R = tauv + 8;             // n x n, ld n
  for (int idx = tid; idx < n * n; idx += kT)
    R[idx] = (blocked & 4) ? jb.a[(idx % n) + size_t(idx / n) * jb.lda] : 0.0;
  double B[kTsqrSlots][kTsqrRpl];
  for (int r0 = 0; r0 < ((blocked & 4) ? 0 : M); r0 += kTsqrBm) {
    const int rb = min(kTsqrBm, M - r0);
#pragma unroll
    for (int u = 0; u < kTsqrSlots; ++u) {
      const int c = warp + 16 * u;
#pragma unroll
      for (int r = 0; r < kTsqrRpl; ++r) {
        const int row = lane + 32 * r;
        B[u][r] = (c < n && row < rb) ? jb.a[(r0 + row) + size_t(c) * jb.lda] : 0.0;
      }
    }
    __syncthreads();  // R from the previous block complete
    if (warp == 0) tsqr_reflector(B[0], R, n, 0, vb, tauv, lane);
    __syncthreads();
    for (int j = 0; j < n; ++j) {
      const int cur = j & 1;
      const double tau = tauv[cur];
      const double* v = vb + cur * kTsqrBm;
      double vr[kTsqrRpl];
#pragma unroll
      for (int r = 0; r < kTsqrRpl; ++r) vr[r] = v[lane + 32 * r];
      if (tau != 0.0) {
        // all owned trailing columns at once: the dot-product reductions of
        // the slots are interleaved so their shuffles pipeline
        double d[kTsqrSlots];
#pragma unroll
        for (int u = 0; u < kTsqrSlots; ++u) {
          d[u] = 0.0;
#pragma unroll
          for (int r = 0; r < kTsqrRpl; ++r) d[u] += vr[r] * B[u][r];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int u = 0; u < kTsqrSlots; ++u) d[u] += __shfl_xor_sync(0xffffffffu, d[u], o);
#pragma unroll
        for (int u = 0; u < kTsqrSlots; ++u) {
          const int c = warp + 16 * u;
          if (c <= j || c >= n) continue;
          const double tw = tau * (d[u] + R[j + c * n]);
#pragma unroll
          for (int r = 0; r < kTsqrRpl; ++r) B[u][r] -= vr[r] * tw;
          if (lane == 0) R[j + c * n] -= tw;
        }
      }
      if (j + 1 < n && ((j + 1) & 15) == warp) {  // look-ahead: next reflector
        const int un = (j + 1) >> 4;
#pragma unroll
        for (int u = 0; u < kTsqrSlots; ++u)
          if (u == un) tsqr_reflector(B[u], R, n, j + 1, vb + (cur ^ 1) * kTsqrBm, tauv + (cur ^ 1), lane);
      }
      __syncthreads();
    }
  }
  __syncthreads();
  const int steps_max = (blocked & 8) ? 0 : jb.max_steps > 0 ? min(n, jb.max_steps) : n;
  blocked &= 1;
  const int done = blocked ? cpqr_core_blocked(R, n, n, n, steps_max, jb.stop_eps, jb.perm, jb.diag, upd, dir,
                                               pos, lphys, red, ired, sc, F, aux, vrow, bp, rec)
                           : cpqr_core(R, n, n, n, true, steps_max, jb.stop_eps, jb.perm, jb.diag, upd, dir,
                                       pos, lphys, red, ired, sc);
  if (tid == 0 && jb.steps) *jb.steps = done;
  __syncthreads();
  for (int c = warp; c < n; c += kWarps)
    for (int i = lane; i < n; i += 32) jb.a[i + size_t(c) * jb.lda] = R[i + size_t(c) * n];
}

// Tall problems with n <= 128, quad layout: 256 threads; quad g (threads
// 4g..4g+3) owns columns g and g + 64 and, of each, the rows q + 4 i
// (q = thread & 3, i < 32) of the current 128-row block in registers.  A
// column's dot product with the Householder vector reduces over its quad
// (two shuffle levels instead of a warp's five), and the vector reaches the
// quads through shared memory in the owners' row order (row q + 4 i at
// v[q * kQPad + i]; one 16-byte broadcast load serves both columns).
//   TSQR: per 128-row block, n Householder steps on [R; B] with one barrier
//   each; the quad owning column j + 1 applies step j to it first and
//   publishes reflector j + 1 (look-ahead) while the others finish step j.
//   CPQR of R0 (n x n, loaded into the same registers): Eigen's
//   ColPivHouseholderQR pivot rule and xGEQPF norm downdating (as cpqr_core),
//   two barriers per step (pivot partials; reflector).
// Output contract as tsqr_cpqr_kernel: R0's CPQR factor in the first n rows
// of the job matrix, columns in place (perm[l] = physical column at l).
#ifndef SBX_QL
#define SBX_QL 8
#endif
constexpr int kQL = SBX_QL;            // lanes per column group ("quad"); 4 or 8
constexpr int kQT = 64 * kQL;          // threads: 64 groups, two columns each
constexpr int kQWarps = kQT / 32;
constexpr int kQRows = 128 / kQL;      // rows per thread and column
constexpr int kQBm = kQL * kQRows;     // rows per block; also the largest n
constexpr int kQHalf = kQT / kQL;      // column offset of a group's second column
constexpr int kQPad = kQRows + 2;      // padded per-lane stride of v

// quad-local shuffles: the callers branch per column pair (quad-uniformly)
__device__ __forceinline__ unsigned quad_mask() { return ((1u << kQL) - 1u) << (threadIdx.x & (32 - kQL)); }

__device__ __forceinline__ double quad_sum(double v) {
  const unsigned m = quad_mask();
#pragma unroll
  for (int o = 1; o < kQL; o <<= 1) v += __shfl_xor_sync(m, v, o);
  return v;
}

// register b[i] of the quad thread holding row `row` (quad-uniform result)
__device__ __forceinline__ double quad_row(const double (&b)[kQRows], int row) {
  double x = 0.0;
  const int ir = row / kQL;
#pragma unroll
  for (int i = 0; i < kQRows; ++i)
    if (i == ir) x = b[i];
  return __shfl_sync(quad_mask(), x, (threadIdx.x & (32 - kQL)) | (row & (kQL - 1)));
}

// shared-memory 16-byte load the compiler may not cache in registers across
// the two passes of a reflector application (it would hold v next to b)
__device__ __forceinline__ double2 lds_v2(const double* p) {
  double2 r;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
               : "=d"(r.x), "=d"(r.y)
               : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p))));
  return r;
}

// Applies the reflector (v, tau) to the live columns of a quad: A0 / A1 say
// which of its two columns take part; extra0 / extra1 are added to the dot
// products (the R-row entry in TSQR, 0 in the CPQR phase).  Returns tau * w.
template <bool A0, bool A1>
__device__ __forceinline__ void quad_apply(double (&b)[2][kQRows], const double* v, double tau, double extra0,
                                           double extra1, double& tw0, double& tw1) {
  double d0[4] = {0.0, 0.0, 0.0, 0.0}, d1[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int i = 0; i < kQRows; i += 2) {
    const double2 vv = lds_v2(v + i);
    if (A0) {
      d0[i & 3] = fma(vv.x, b[0][i], d0[i & 3]);
      d0[(i & 3) + 1] = fma(vv.y, b[0][i + 1], d0[(i & 3) + 1]);
    }
    if (A1) {
      d1[i & 3] = fma(vv.x, b[1][i], d1[i & 3]);
      d1[(i & 3) + 1] = fma(vv.y, b[1][i + 1], d1[(i & 3) + 1]);
    }
  }
  tw0 = A0 ? tau * (quad_sum((d0[0] + d0[1]) + (d0[2] + d0[3])) + extra0) : 0.0;
  tw1 = A1 ? tau * (quad_sum((d1[0] + d1[1]) + (d1[2] + d1[3])) + extra1) : 0.0;
#pragma unroll
  for (int i = 0; i < kQRows; i += 2) {
    const double2 vv = lds_v2(v + i);
    if (A0) {
      b[0][i] = fma(-vv.x, tw0, b[0][i]);
      b[0][i + 1] = fma(-vv.y, tw0, b[0][i + 1]);
    }
    if (A1) {
      b[1][i] = fma(-vv.x, tw1, b[1][i]);
      b[1][i + 1] = fma(-vv.y, tw1, b[1][i + 1]);
    }
  }
}

__device__ __forceinline__ void quad_apply_any(bool a0, bool a1, double (&b)[2][kQRows], const double* v, double tau,
                                               double e0, double e1, double& tw0, double& tw1) {
  tw0 = tw1 = 0.0;
  if (a0 && a1)
    quad_apply<true, true>(b, v, tau, e0, e1, tw0, tw1);
  else if (a1)
    quad_apply<false, true>(b, v, tau, e0, e1, tw0, tw1);
  else if (a0)
    quad_apply<true, false>(b, v, tau, e0, e1, tw0, tw1);
}

// TSQR reflector of one owned column (rows of the block) against R(jn, jn).
__device__ __forceinline__ void quad_tsqr_reflector(double (&b)[kQRows], double* R, int ldr, int jn, double* v,
                                                    double* tau_out, int q) {
  double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int i = 0; i < kQRows; ++i) s4[i & 3] = fma(b[i], b[i], s4[i & 3]);
  const double sq = quad_sum((s4[0] + s4[1]) + (s4[2] + s4[3]));
  const double c0 = R[jn * ldr + jn];
  double tau = 0.0, beta = c0, inv = 0.0;
  if (sq > DBL_MIN) {  // Q is discarded: reciprocals instead of divisions
    beta = sqrt(c0 * c0 + sq);
    if (c0 >= 0.0) beta = -beta;
    inv = 1.0 / (c0 - beta);
    tau = (beta - c0) * (1.0 / beta);
  }
  double* vw = v + q * kQPad;
#pragma unroll
  for (int i = 0; i < kQRows; i += 2) {
    b[i] *= inv;
    b[i + 1] *= inv;
    *reinterpret_cast<double2*>(vw + i) = make_double2(b[i], b[i + 1]);
  }
  if (q == 0) {
    R[jn * ldr + jn] = beta;
    *tau_out = tau;
  }
}

// CPQR reflector of the pivot column over rows >= j (Eigen
// makeHouseholderInPlace); v gets (0 above j, 1 at j, essential below).
__device__ __forceinline__ void quad_cpqr_reflector(double (&b)[kQRows], int j, double* v, double* sc, int q) {
  double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int i = 0; i < kQRows; ++i)
    if (q + kQL * i > j) s4[i & 3] = fma(b[i], b[i], s4[i & 3]);
  const double s = quad_sum((s4[0] + s4[1]) + (s4[2] + s4[3]));
  const double c0 = quad_row(b, j);
  double tau = 0.0, beta = c0, inv = 0.0;
  if (s > DBL_MIN) {
    beta = sqrt(c0 * c0 + s);
    if (c0 >= 0.0) beta = -beta;
    inv = 1.0 / (c0 - beta);
    tau = (beta - c0) / beta;
  }
  double* vw = v + q * kQPad;
#pragma unroll
  for (int i = 0; i < kQRows; i += 2) {
    double e[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int row = q + kQL * (i + h);
      if (row > j) {
        b[i + h] *= inv;
        e[h] = b[i + h];
      } else if (row == j) {
        b[i + h] = beta;
        e[h] = 1.0;
      } else {
        e[h] = 0.0;
      }
    }
    *reinterpret_cast<double2*>(vw + i) = make_double2(e[0], e[1]);
  }
  if (q == 0) {
    sc[0] = tau;
    sc[1] = beta;
  }
}

// xGEQPF downdate of one live column's norms after step j (quad-uniform).
__device__ __forceinline__ void quad_downdate(const double (&b)[kQRows], int j, int q, double& upd, double& dirn,
                                              double thr) {
  if (upd == 0.0) return;
  double t = fabs(quad_row(b, j)) / upd;
  t = (1.0 + t) * (1.0 - t);
  t = t < 0.0 ? 0.0 : t;
  const double rr = upd / dirn;
  if (t * rr * rr <= thr) {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < kQRows; ++i)
      if (q + kQL * i > j) s = fma(b[i], b[i], s);
    upd = dirn = sqrt(quad_sum(s));
  } else {
    upd *= sqrt(t);
  }
}

// CPQR of the n x n upper-triangular R0 (Eigen ColPivHouseholderQR
// semantics) held row-major in shared memory (ld ldr), quad layout (each
// quad of 4 threads owns two columns, 32 rows each in registers): the
// second phase of the TSQR and blocked-QR engines.  Writes the pivoted R
// into the top n rows of jb.a, perm, diag and steps.
__device__ __forceinline__ void quad_cpqr_r0(const QrJob& jb, const double* R, int ldr, double* vq, double* sc,
                                             double* red, int* ired, int phases) {
  const int n = jb.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = tid / kQL, q = tid % kQL;
  const int c0 = g, c1 = g + kQHalf;
  const bool h0 = c0 < n, h1 = c1 < n;
  double b[2][kQRows];
#pragma unroll
  for (int i = 0; i < kQRows; ++i) {
    const int row = q + kQL * i;
    b[0][i] = (h0 && row < n) ? R[row * ldr + c0] : 0.0;
    b[1][i] = (h1 && row < n) ? R[row * ldr + c1] : 0.0;
  }
  for (int l = tid; l < n; l += kQT) jb.diag[l] = 0.0;
  double upd0, dir0, upd1, dir1;
  {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int i = 0; i < kQRows; ++i) {
      s0 = fma(b[0][i], b[0][i], s0);
      s1 = fma(b[1][i], b[1][i], s1);
    }
    upd0 = dir0 = sqrt(quad_sum(s0));
    upd1 = dir1 = sqrt(quad_sum(s1));
  }
  const double thr = sqrt(DBL_EPSILON);
  int pos0 = c0, pos1 = c1;
  int done = 0;
  double r00 = 0.0;
  const int steps_max = (phases & 8) ? 0 : jb.max_steps > 0 ? min(n, jb.max_steps) : n;
  for (int j = 0; j < steps_max; ++j) {
    // (1) first max of the updated norms over logical positions >= j
    double bv = -1.0;
    int bp = 0x7fffffff, bq = -1;
    if (h0 && pos0 >= j) {
      bv = upd0;
      bp = pos0;
      bq = c0;
    }
    if (h1 && pos1 >= j && (upd1 > bv || (upd1 == bv && pos1 < bp))) {
      bv = upd1;
      bp = pos1;
      bq = c1;
    }
#pragma unroll
    for (int o = 16; o >= kQL; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      const int oq = __shfl_xor_sync(0xffffffffu, bq, o);
      if (ov > bv || (ov == bv && op < bp)) {
        bv = ov;
        bp = op;
        bq = oq;
      }
    }
    if (lane == 0) {
      red[warp] = bv;
      ired[warp] = bp;
      ired[kQWarps + warp] = bq;
    }
    __syncthreads();  // (A)
    bv = -1.0;
    bp = 0x7fffffff;
#pragma unroll
    for (int w = 0; w < kQWarps; ++w) {
      const double rv = red[w];
      const int rp = ired[w];
      if (rv > bv || (rv == bv && rp < bp)) {
        bv = rv;
        bp = rp;
        bq = ired[kQWarps + w];
      }
    }
    const int p = bq, lp = bp;
    double* v = vq + (j & 1) * (kQL * kQPad);
    // (2) Householder vector of the pivot column over rows >= j
    if (p == c0)
      quad_cpqr_reflector(b[0], j, v, sc, q);
    else if (p == c1)
      quad_cpqr_reflector(b[1], j, v, sc, q);
    // logical swap: the column at position j moves to the pivot's slot
    if (h0) pos0 = (c0 == p) ? j : (pos0 == j ? lp : pos0);
    if (h1) pos1 = (c1 == p) ? j : (pos1 == j ? lp : pos1);
    __syncthreads();  // (B)
    const double tau = sc[0], beta = sc[1];
    if (j == 0) r00 = fabs(beta);
    if (tid == 0) jb.diag[j] = fabs(beta);
    done = j + 1;
    if (jb.stop_eps > 0.0 && !(fabs(beta) > jb.stop_eps * r00)) break;
    // (3) the live columns: apply, then downdate their norms
    const bool a0 = h0 && pos0 > j, a1 = h1 && pos1 > j;
    if (a0 || a1) {
      if (tau != 0.0) {
        double tw0, tw1;
        quad_apply_any(a0, a1, b, v + q * kQPad, tau, 0.0, 0.0, tw0, tw1);
      }
      if (a0) quad_downdate(b[0], j, q, upd0, dir0, thr);
      if (a1) quad_downdate(b[1], j, q, upd1, dir1, thr);
    }
  }
  if (tid == 0 && jb.steps) *jb.steps = done;
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int cu = u ? c1 : c0;
    if (cu >= n) continue;
    if (q == 0) jb.perm[u ? pos1 : pos0] = cu;
#pragma unroll
    for (int i = 0; i < kQRows; ++i) {
      const int row = q + kQL * i;
      if (row < n) jb.a[row + size_t(cu) * jb.lda] = b[u][i];
    }
  }
}

size_t tsqr_quad_smem(int n) {
  return size_t(n) * size_t(n + 1) * sizeof(double) + size_t(2 * kQL * kQPad + 16 + 2 * kQWarps) * sizeof(double) +
         size_t(2 * kQWarps) * sizeof(int);
}

__global__ void __launch_bounds__(kQT, 1) tsqr_quad_kernel(const QrJob* __restrict__ jobs, int phases) {
  extern __shared__ double sm[];
  const QrJob jb = jobs[blockIdx.x];
  const int M = jb.M, n = jb.n, ldr = n + 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = tid / kQL, q = tid % kQL;
  const int c0 = g, c1 = g + kQHalf;         // owned columns
  const bool h0 = c0 < n, h1 = c1 < n;
  double* R = sm;                                  // n x n, row-major, ld n + 1
  double* vq = R + n * ldr;                        // 2 x (4 x kQPad) reflector buffers
  double* taus = vq + 2 * kQL * kQPad;               // 2 (+pad)
  double* sc = taus + 8;                           // tau, beta
  double* red = sc + 8;                            // kQWarps pivot partials
  int* ired = reinterpret_cast<int*>(red + 2 * kQWarps);
  for (int idx = tid; idx < n * ldr; idx += kQT) R[idx] = 0.0;
  double b[2][kQRows];
  // ---------------- TSQR: R0 of W^T
  for (int r0 = 0; r0 < ((phases & 4) ? 0 : M); r0 += kQBm) {
    const int rb = min(kQBm, M - r0);
    const double* s0 = jb.a + r0 + size_t(h0 ? c0 : 0) * jb.lda;
    const double* s1 = jb.a + r0 + size_t(h1 ? c1 : 0) * jb.lda;
#pragma unroll
    for (int i = 0; i < kQRows; ++i) {
      const int row = q + kQL * i;
      b[0][i] = (h0 && row < rb) ? __ldg(s0 + row) : 0.0;
      b[1][i] = (h1 && row < rb) ? __ldg(s1 + row) : 0.0;
    }
    __syncthreads();  // R of the previous block complete, buffers free
    if (g == 0) quad_tsqr_reflector(b[0], R, ldr, 0, vq, taus, q);
    __syncthreads();
    for (int j = 0; j < n; ++j) {
      const int cur = j & 1;
      const bool a0 = h0 && c0 > j, a1 = h1 && c1 > j;
      if (a0 || a1) {
        const double tau = taus[cur];
        if (tau != 0.0) {
          const double e0 = a0 ? R[j * ldr + c0] : 0.0, e1 = a1 ? R[j * ldr + c1] : 0.0;
          double tw0, tw1;
          quad_apply_any(a0, a1, b, vq + cur * (kQL * kQPad) + q * kQPad, tau, e0, e1, tw0, tw1);
          if (q == 0) {
            if (a0) R[j * ldr + c0] = e0 - tw0;
            if (a1) R[j * ldr + c1] = e1 - tw1;
          }
        }
        const int jn = j + 1;
        if (jn < n && (jn & (kQHalf - 1)) == g) {  // look-ahead: next reflector
          if (jn < kQHalf)
            quad_tsqr_reflector(b[0], R, ldr, jn, vq + (cur ^ 1) * (kQL * kQPad), taus + (cur ^ 1), q);
          else
            quad_tsqr_reflector(b[1], R, ldr, jn, vq + (cur ^ 1) * (kQL * kQPad), taus + (cur ^ 1), q);
        }
      }
      __syncthreads();
    }
  }
  if (phases & 4) {  // diagnostics: CPQR of the top n x n block alone
    __syncthreads();
    for (int idx = tid; idx < n * n; idx += kQT) R[(idx % n) * ldr + idx / n] = jb.a[(idx % n) + size_t(idx / n) * jb.lda];
    __syncthreads();
  }
  quad_cpqr_r0(jb, R, ldr, vq, sc, red, ired, phases);
}

// D = A B + C on the FP64 tensor cores (m8n8k4: lane l holds A[l/4][l%4],
// B[l%4][l/4], C[l/4][2(l%4) + {0,1}])
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------- blocked QR (engine 10)
// Tall W^T (M <= kBMaxM, n <= 128), one CTA per problem.  Phase 1 reduces
// W^T to R0 by a blocked Householder QR (LAPACK dgeqrf/dlarft/dlarfb,
// forward, columnwise): 16-column panels factored in shared memory (one
// CTA barrier per column), the trailing matrix updated in place in global
// memory (L2) by A <- A - V (T^T (V^T A)) on the FP64 tensor cores
// (mma.sync.m8n8k4.f64 -> DMMA).  Phase 2 is the CPQR of R0 of the TSQR
// engine (quad_cpqr_r0): same pivots as the CPQR of W^T in exact arithmetic
// (R0 has W^T's column space geometry).
constexpr int kBW = 16;           // panel width
constexpr int kBMaxM = 1280;      // rows (panel in shared memory)
constexpr int kBT = kQT;          // threads (the CPQR phase's quad layout)
constexpr int kBWarps = kBT / 32;
constexpr int kBLdW = 128 + 4;    // row stride of the W / W2 buffers
constexpr int kBRpl = (kBMaxM + 32 * (kQT / 32) - 1) / (32 * (kQT / 32));  // panel rows per lane

#ifdef SBX_CPQR_PROF
__device__ long long g_bqr_prof[16 * 8];
#define BQR_T(ph)                                                                               \
  do {                                                                                          \
    if (blockIdx.x == 0 && threadIdx.x == 0 && c0 / kBW < 16) g_bqr_prof[(c0 / kBW) * 8 + (ph)] = clock64(); \
  } while (0)
#else
#define BQR_T(ph) \
  do {            \
  } while (0)
#endif
size_t bqr_smem(int M, int n) {
  const size_t ldp = size_t((M + 3) / 4 * 4);
  const size_t p1 = ldp * kBW + 2 * size_t(kBW) * kBLdW + 2 * kBW * kBW + 2 * kBW;  // P, W, W2, G, T, tau
  const size_t p2 = size_t(n) * size_t(n + 1) + 2 * kQL * kQPad + 16 + 2 * kQWarps + kQWarps;  // R, vq, sc, red, ired
  return std::max(p1, p2) * sizeof(double);
}

// One column step of the panel QR (rows split over the warps): partial
// sums x^T a_k of the live panel columns k >= K0, reduce-scatter per warp,
// warp 0 forms the Householder scalars and R row j, every warp updates its
// rows.  Two CTA barriers.
template <int K0>
__device__ __forceinline__ void bqr_panel_column(double* P, int ldp, int j, int w, int ml, int rb0, int rb1, int lane,
                                                 int warp, double* part, double* scv, double* tau) {
  constexpr int NV = kBW - K0;  // values per lane (16 or 8)
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = 0.0;
#pragma unroll
  for (int t = 0; t < kBRpl; ++t) {
    const int i = rb0 + lane + 32 * t;
    if (i < rb1 && i > j && i < ml) {
      const double x = P[i + size_t(ldp) * j];
#pragma unroll
      for (int k = 0; k < NV; ++k) acc[k] = fma(x, P[i + size_t(ldp) * (K0 + k)], acc[k]);
    }
  }
  // reduce-scatter: after the halving steps lane l holds value (l >> 1) mod NV
  // summed over the lanes that differ in bits 1 .. log2(NV); the remaining
  // lane bits are summed by plain butterflies
#pragma unroll
  for (int h = NV / 2; h >= 1; h >>= 1) {
    const bool up = (lane & (2 * h)) != 0;
#pragma unroll
    for (int k = 0; k < h; ++k) {
      const double send = up ? acc[k] : acc[k + h];
      const double keep = up ? acc[k + h] : acc[k];
      acc[k] = keep + __shfl_xor_sync(0xffffffffu, send, 2 * h);
    }
  }
#pragma unroll
  for (int o = 2 * NV; o < 32; o <<= 1) acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], o);
  acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 1);
  if ((lane & ~(2 * NV - 2)) == 0) part[warp * kBW + K0 + (lane >> 1)] = acc[0];
  __syncthreads();
  if (warp == 0) {  // (the whole warp: the shuffle below)
    double tot = 0.0;
    if (lane >= K0 && lane < kBW) {
      double v[kBWarps];
#pragma unroll
      for (int q = 0; q < kBWarps; ++q) v[q] = part[q * kBW + lane];
#pragma unroll
      for (int q = 1; q < kBWarps; q <<= 1)  // fixed tree over the warps
#pragma unroll
        for (int r = 0; r + q < kBWarps; r += 2 * q) v[r] += v[r + q];
      tot = v[0];
    }
    const double s2 = __shfl_sync(0xffffffffu, tot, j);
    const double alpha = P[j + size_t(ldp) * j];
    double t = 0.0, beta = alpha, sc = 0.0;
    if (s2 > DBL_MIN) {
      beta = sqrt(fma(alpha, alpha, s2));
      if (alpha >= 0.0) beta = -beta;
      sc = 1.0 / (alpha - beta);
      t = (beta - alpha) / beta;
    }
    if (lane > j && lane < w) {
      const double tw = t * (P[j + size_t(ldp) * lane] + sc * tot);
      scv[lane] = tw * sc;
      P[j + size_t(ldp) * lane] -= tw;  // R(j, k)
    }
    if (lane == 0) {
      scv[kBW] = sc;
      tau[j] = t;
      P[j + size_t(ldp) * j] = beta;
    }
  }
  __syncthreads();
  const double sc = scv[kBW];
#pragma unroll
  for (int t = 0; t < kBRpl; ++t) {
    const int i = rb0 + lane + 32 * t;
    if (i < rb1 && i > j && i < ml) {
      double* xr = P + i;
      const double x = xr[size_t(ldp) * j];
#pragma unroll
      for (int k = K0; k < kBW; ++k)
        if (k > j && k < w) xr[size_t(ldp) * k] = fma(-x, scv[k], xr[size_t(ldp) * k]);
      xr[size_t(ldp) * j] = x * sc;
    }
  }
  // (each warp updates only its own rows, which its next partial sums read;
  // the scalars' buffers are rewritten after the next barrier)
}

__global__ void __launch_bounds__(kBT, 1) bqr_kernel(const QrJob* __restrict__ jobs, int phases) {
  extern __shared__ double sm[];
  const QrJob jb = jobs[blockIdx.x];
  const int M = jb.M, n = jb.n, lda = jb.lda;
  double* const A = jb.a;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int ldp = (M + 3) / 4 * 4;
  double* P = sm;                         // ldp x 16 (column-major): panel, then V
  double* W = P + size_t(ldp) * kBW;      // 16 x kBLdW: V^T A_trail
  double* W2 = W + kBW * kBLdW;           // 16 x kBLdW: T^T W
  double* Gm = W2 + kBW * kBLdW;          // 16 x 16: V^T V (column-major)
  double* T = Gm + kBW * kBW;             // 16 x 16 (column-major)
  double* tau = T + kBW * kBW;            // 16
  for (int c0 = 0; c0 < ((phases & 4) ? 0 : n); c0 += kBW) {
    const int w = min(kBW, n - c0), ml = M - c0, kp = (ml + 3) / 4 * 4, nt = n - c0 - w;
    BQR_T(0);
    // ---- (1) the panel: rows c0.., columns c0..c0+w (zero padded to kp x 16)
    for (int k = warp; k < kBW; k += kBWarps) {
      const double* src = A + c0 + size_t(c0 + (k < w ? k : 0)) * lda;
      for (int i0 = 0; i0 < kp; i0 += 128) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + lane + 32 * u;
          v[u] = (k < w && i < ml) ? src[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + lane + 32 * u;
          if (i < kp) P[i + size_t(ldp) * k] = v[u];
        }
      }
    }
    __syncthreads();
    BQR_T(1);
    // ---- (2) panel QR, rows split over the warps (warp w owns panel rows
    // [w rpw, (w + 1) rpw), lane rows w rpw + lane + 32 t): per column, the
    // partial sums x^T a_k of every warp (two CTA barriers per column)
    {
      const int rpw = (kp + kBWarps - 1) / kBWarps;
      const int rb0 = warp * rpw, rb1 = min(kp, rb0 + rpw);
      double* part = W;   // kBWarps x 16 partial sums (W is free until step 4)
      double* scv = W2;   // tw_k / (alpha - beta) per column, scale, beta
      for (int j = 0; j < w; ++j) {
        // columns below K0 are all pivoted once j >= 8: the second half of
        // the panel runs with the 8 live columns only
        if (j < kBW / 2)
          bqr_panel_column<0>(P, ldp, j, w, ml, rb0, rb1, lane, warp, part, scv, tau);
        else
          bqr_panel_column<kBW / 2>(P, ldp, j, w, ml, rb0, rb1, lane, warp, part, scv, tau);
      }
    }
    __syncthreads();
    BQR_T(2);
    // ---- (3) R rows of the panel to global memory; V gets its unit diagonal
    for (int k = warp; k < w; k += kBWarps)
      for (int i = lane; i <= k; i += 32) A[(c0 + i) + size_t(c0 + k) * lda] = P[i + size_t(ldp) * k];
    __syncthreads();
    for (int idx = tid; idx < kBW * kBW; idx += kBT) {
      const int i = idx % kBW, k = idx / kBW;
      if (i <= k) P[i + size_t(ldp) * k] = (i == k && k < w) ? 1.0 : 0.0;
    }
    if (nt <= 0) {
      __syncthreads();
      continue;
    }
    __syncthreads();
    BQR_T(3);
    // ---- (4) G = V^T V (warps 0-3: one 8 x 8 tile each) and W = V^T A_trail
    if (warp < 4) {
      const int ti = warp >> 1, tj2 = warp & 1;
      double g0 = 0.0, g1 = 0.0;
      for (int k0 = 0; k0 < kp; k0 += 4) {
        const double a = P[(k0 + tig) + size_t(ldp) * (ti * 8 + gid)];
        const double b = P[(k0 + tig) + size_t(ldp) * (tj2 * 8 + gid)];
        dmma(g0, g1, a, b);
      }
      Gm[(ti * 8 + gid) + kBW * (tj2 * 8 + 2 * tig)] = g0;
      Gm[(ti * 8 + gid) + kBW * (tj2 * 8 + 2 * tig + 1)] = g1;
    }
    {
      // W = V^T A_trail: a warp per 8-column tile of A_trail (both 8-row
      // tiles of W share its B fragments = A_trail(k0 + tig, cj * 8 + gid),
      // streamed from L2 with 8 loads in flight)
      const int ctiles = (nt + 7) / 8;
      for (int cj = warp; cj < ctiles; cj += kBWarps) {
        const bool cok = cj * 8 + gid < nt;
        const double* ac = A + c0 + size_t(cok ? c0 + w + cj * 8 + gid : c0 + w) * lda;
        double w00 = 0.0, w01 = 0.0, w10 = 0.0, w11 = 0.0;
        for (int k0 = 0; k0 < kp; k0 += 32) {
          double bb[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int r = k0 + 4 * u + tig;
            bb[u] = (cok && r < ml) ? ac[r] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int r = k0 + 4 * u + tig;
            if (k0 + 4 * u < kp) {
              dmma(w00, w01, P[r + size_t(ldp) * gid], bb[u]);
              dmma(w10, w11, P[r + size_t(ldp) * (8 + gid)], bb[u]);
            }
          }
        }
        W[gid * kBLdW + cj * 8 + 2 * tig] = w00;
        W[gid * kBLdW + cj * 8 + 2 * tig + 1] = w01;
        W[(8 + gid) * kBLdW + cj * 8 + 2 * tig] = w10;
        W[(8 + gid) * kBLdW + cj * 8 + 2 * tig + 1] = w11;
      }
    }
    __syncthreads();
    BQR_T(4);
    // ---- (5) T (dlarft, forward columnwise): T(0:j, j) = -tau_j T(0:j, 0:j) G(0:j, j)
    if (warp == 0) {
      for (int j = 0; j < kBW; ++j) {
        const double tj = j < w ? tau[j] : 0.0;
        double v = 0.0;
        if (lane < j) {
          double s2 = 0.0;
          for (int l = lane; l < j; ++l) s2 = fma(T[lane + kBW * l], Gm[l + kBW * j], s2);
          v = -tj * s2;
        }
        __syncwarp();
        if (lane < kBW) T[lane + kBW * j] = lane < j ? v : (lane == j ? tj : 0.0);
        __syncwarp();
      }
    }
    __syncthreads();
    BQR_T(5);
    // ---- (6) W2 = T^T W
    for (int idx = tid; idx < kBW * nt; idx += kBT) {
      const int a = idx / nt, c = idx % nt;
      double s2 = 0.0;
      for (int b = 0; b <= a; ++b) s2 = fma(T[b + kBW * a], W[b * kBLdW + c], s2);
      W2[a * kBLdW + c] = s2;
    }
    __syncthreads();
    BQR_T(6);
    // ---- (7) A_trail -= V W2 (8 x 8 tiles, K = 16: four DMMA each); a warp
    // takes four row tiles of one column tile at a time (8 loads in flight)
    {
      const int rtiles = (kp + 7) / 8, ctiles = (nt + 7) / 8, rgroups = (rtiles + 3) / 4;
      for (int t = warp; t < rgroups * ctiles; t += kBWarps) {
        const int rg = t % rgroups, cj = t / rgroups;
        const int cc = cj * 8 + 2 * tig;
        const bool c0ok = cc < nt, c1ok = cc + 1 < nt;
        double wb[4];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) wb[kk] = (cj * 8 + gid < nt) ? W2[(4 * kk + tig) * kBLdW + cj * 8 + gid] : 0.0;
        double d[4][2];
        double* ap[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int r = (rg * 4 + u) * 8 + gid;
          const bool rok = r < ml;
          ap[u] = A + (c0 + (rok ? r : 0)) + size_t(c0 + w + (c0ok ? cc : 0)) * lda;
          d[u][0] = (rok && c0ok) ? ap[u][0] : 0.0;
          d[u][1] = (rok && c1ok) ? ap[u][lda] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int rt = rg * 4 + u;
          if (rt >= rtiles) continue;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const double va = (rt * 8 + gid < kp) ? -P[(rt * 8 + gid) + size_t(ldp) * (4 * kk + tig)] : 0.0;
            dmma(d[u][0], d[u][1], va, wb[kk]);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int r = (rg * 4 + u) * 8 + gid;
          if (r < ml && c0ok) ap[u][0] = d[u][0];
          if (r < ml && c1ok) ap[u][lda] = d[u][1];
        }
      }
    }
    __syncthreads();
    BQR_T(7);
  }
  // ---- phase 2: CPQR of R0 (the top n rows' upper triangle)
  double* R = sm;
  const int ldr = n + 1;
  double* vq = R + n * ldr;
  double* sc = vq + 2 * kQL * kQPad;
  double* red = sc + 8;
  int* ired = reinterpret_cast<int*>(red + 2 * kQWarps);
  for (int idx = tid; idx < n * n; idx += kBT) {
    const int i = idx % n, k = idx / n;
    R[i * ldr + k] = i <= k ? A[i + size_t(k) * lda] : 0.0;
  }
  __syncthreads();
  quad_cpqr_r0(jb, R, ldr, vq, sc, red, ired, phases);
}

// ---------------------------------------------------------------- cooperative CPQR
struct CoopCtl {
  unsigned count, gen;
};
struct CoopPart {
  double val;
  int pos, phys;
};

constexpr int kCT = 256;
constexpr int kCWarps = kCT / 32;

__device__ void group_barrier(CoopCtl* ctl, unsigned nblocks) {
  // every thread publishes its own stores at gpu scope before arriving: a
  // fence by the arriving thread alone does not drain other warps' stores
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vg = &ctl->gen;
    const unsigned g = *vg;
    __threadfence();
    if (atomicAdd(&ctl->count, 1u) == nblocks - 1) {
      atomicExch(&ctl->count, 0u);
      __threadfence();
      atomicAdd(&ctl->gen, 1u);
    } else {
      while (*vg == g) __nanosleep(40);
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ bool better(double v, int p, double bv, int bp) {
  return v > bv || (v == bv && p < bp);
}

// First-max over the G published partials of a group, in parallel (one L2
// round trip instead of G serial loads).  Every thread gets the winner's
// physical column, logical position and owning CTA rank.
__device__ void coop_pick(const CoopPart* cur, int G, double* red, int* ired, int& out_phys,
                          int& out_pos, int& out_own) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nw = blockDim.x >> 5;
  double bv = -1.0;
  int bp = 0x7fffffff, bq = -1, bo = -1;
  for (int g = tid; g < G; g += blockDim.x) {
    const double pv = __ldcg(&cur[g].val);
    const int pp = __ldcg(&cur[g].pos), pq = __ldcg(&cur[g].phys);
    if (pq >= 0 && better(pv, pp, bv, bp)) {
      bv = pv;
      bp = pp;
      bq = pq;
      bo = g;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int op = __shfl_xor_sync(0xffffffffu, bp, o);
    const int oq = __shfl_xor_sync(0xffffffffu, bq, o);
    const int oo = __shfl_xor_sync(0xffffffffu, bo, o);
    if (better(ov, op, bv, bp)) {
      bv = ov;
      bp = op;
      bq = oq;
      bo = oo;
    }
  }
  __syncthreads();  // red / ired free
  if (lane == 0) {
    red[warp] = bv;
    ired[warp] = bp;
    ired[32 + warp] = bq;
    ired[64 + warp] = bo;
  }
  __syncthreads();
  if (warp == 0) {  // first max over the warps' winners (ascending warp order on ties)
    double v0 = -1.0;
    int p0 = 0x7fffffff, q0 = -1, o0 = -1;
    for (int w = 0; w < nw; ++w)
      if (better(red[w], ired[w], v0, p0)) {
        v0 = red[w];
        p0 = ired[w];
        q0 = ired[32 + w];
        o0 = ired[64 + w];
      }
    __syncwarp();
    if (lane == 0) {
      ired[0] = q0;
      ired[1] = p0;
      ired[2] = o0;
    }
  }
  __syncthreads();
  out_phys = ired[0];
  out_pos = ired[1];
  out_own = ired[2];
  __syncthreads();  // everyone has read ired
}

struct CoopArgs {
  const QrJob* jobs;
  const int* cta_job;
  const int* cta_rank;
  const int* job_ctas;
  CoopCtl* ctl;
  CoopPart* parts;
  const int* part_off;
  double* beta;        // signed R diagonal per job (offset beta_off)
  const i64* beta_off;
  double* vglob;       // per-CTA Householder vectors in global memory (null: in smem)
  i64 vstride;
};

__global__ void __launch_bounds__(kCT) cpqr_coop_kernel(CoopArgs args) {
  extern __shared__ double sm[];
  const int job = args.cta_job[blockIdx.x];
  const int rank = args.cta_rank[blockIdx.x];
  const int G = args.job_ctas[job];
  const QrJob jb = args.jobs[job];
  const int M = jb.M, n = jb.n, lda = jb.lda;
  double* A = jb.a;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c0 = int(i64(n) * rank / G), c1 = int(i64(n) * (rank + 1) / G);
  const int nown = c1 - c0;
  // Householder vector: shared memory, or this CTA's global (L2) slot for
  // functionals too many for it
  double* v = args.vglob ? args.vglob + size_t(blockIdx.x) * args.vstride : sm;  // M
  double* upd = args.vglob ? sm : v + M;  // nown
  double* dir = upd + nown;      // nown
  double* red = dir + nown;      // 32
  double* sc = red + 32;         // 8
  int* ired = reinterpret_cast<int*>(sc + 8);  // 96
  int* mypos = ired + 96;        // nown (logical position, -1 once pivoted)
  CoopCtl* ctl = args.ctl + job;
  CoopPart* parts = args.parts + args.part_off[job];
  double* sbeta = args.beta + args.beta_off[job];
  for (int c = tid; c < nown; c += kCT) mypos[c] = c0 + c;
  for (int c = warp; c < nown; c += kCWarps) {
    const double* col = A + size_t(c0 + c) * lda;
    double s = 0.0;
    for (int i = lane; i < M; i += 32) s += col[i] * col[i];
    s = warp_sum(s);
    if (lane == 0) upd[c] = dir[c] = sqrt(s);
  }
  __syncthreads();
  const int size = min(M, n);
  const int steps_max = jb.max_steps > 0 ? min(size, jb.max_steps) : size;
  const double thr = sqrt(DBL_EPSILON);
  int done = 0, prev_p = -1;
  double prev_beta = 0.0, r00 = 0.0;
  for (int j = 0; j < steps_max; ++j) {
    // local first-max over alive columns, ties by logical position
    double bv = -1.0;
    int bp = 0x7fffffff, bphys = -1;
    for (int c = tid; c < nown; c += kCT) {
      const int p = mypos[c];
      if (p >= 0 && better(upd[c], p, bv, bp)) {
        bv = upd[c];
        bp = p;
        bphys = c0 + c;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      const int oq = __shfl_xor_sync(0xffffffffu, bphys, o);
      if (better(ov, op, bv, bp)) {
        bv = ov;
        bp = op;
        bphys = oq;
      }
    }
    if (lane == 0) {
      red[warp] = bv;
      ired[warp] = bp;
    }
    __shared__ int wphys[kCWarps];
    if (lane == 0) wphys[warp] = bphys;
    __syncthreads();
    if (tid == 0) {
      double v0 = -1.0;
      int p0 = 0x7fffffff, q0 = -1;
      for (int w = 0; w < kCWarps; ++w)
        if (better(red[w], ired[w], v0, p0)) {
          v0 = red[w];
          p0 = ired[w];
          q0 = wphys[w];
        }
      // double-buffered by step parity: a CTA already in step j+1 must not
      // overwrite a partial another CTA is still reading for step j
      parts[(j & 1) * G + rank] = {v0, p0, q0};
    }
    group_barrier(ctl, unsigned(G));
    // previous pivot's diagonal, deferred so no CTA reads a half-written column
    if (prev_p >= 0 && prev_p >= c0 && prev_p < c1 && tid == 0)
      A[(j - 1) + size_t(prev_p) * lda] = prev_beta;
    // global pivot
    int p, lp, own_unused;
    coop_pick(parts + (j & 1) * G, G, red, ired, p, lp, own_unused);
    // logical swap: the column at position j moves to lp, p becomes position j
    for (int c = tid; c < nown; c += kCT) {
      if (c0 + c == p) mypos[c] = -1;
      else if (mypos[c] == j) mypos[c] = lp;
    }
    if (p >= c0 && p < c1 && tid == 0) jb.perm[j] = p;
    // Householder vector of the pivot column (redundant in every CTA)
    const double* pc = A + size_t(p) * lda;
    double part = 0.0;
    for (int i = j + 1 + tid; i < M; i += kCT) {
      const double x = __ldcg(pc + i);
      v[i] = x;
      part += x * x;
    }
    const double tail = [&] {
      double t = warp_sum(part);
      __syncthreads();
      if (lane == 0) red[warp] = t;
      __syncthreads();
      double u = lane < kCWarps ? red[lane] : 0.0;
      return warp_sum(u);
    }();
    const double cc = __ldcg(pc + j);
    double tau, beta, denom;
    if (tail <= DBL_MIN) {
      tau = 0.0;
      beta = cc;
      denom = 0.0;
    } else {
      beta = sqrt(cc * cc + tail);
      if (cc >= 0.0) beta = -beta;
      denom = cc - beta;
      tau = (beta - cc) / beta;
    }
    __syncthreads();
    for (int i = j + 1 + tid; i < M; i += kCT) v[i] = denom == 0.0 ? 0.0 : v[i] / denom;
    if (j == 0) r00 = fabs(beta);
    if (rank == 0 && tid == 0) sbeta[j] = beta;
    __syncthreads();
    prev_p = p;
    prev_beta = beta;
    done = j + 1;
    if (jb.stop_eps > 0.0 && !(fabs(beta) > jb.stop_eps * r00)) break;
    for (int c = 4 * warp; c < nown; c += 4 * kCWarps) {
      double* cols[4];
      int slot[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool live = c + u < nown && mypos[c + u] >= 0;
        cols[u] = live ? A + size_t(c0 + c + u) * lda : nullptr;
        slot[u] = c + u;
      }
      reflect_cols<4>(cols, slot, v, j, M, tau, true, upd, dir, thr, lane);
    }
    __syncthreads();
  }
  // finalisation: last diagonal, logical order of the untouched columns
  group_barrier(ctl, unsigned(G));
  if (prev_p >= c0 && prev_p < c1 && tid == 0) A[(done - 1) + size_t(prev_p) * lda] = prev_beta;
  for (int c = tid; c < nown; c += kCT)
    if (mypos[c] >= 0) jb.perm[mypos[c]] = c0 + c;
  for (int l = rank * kCT + tid; l < size; l += G * kCT)
    jb.diag[l] = l < done ? fabs(__ldcg(sbeta + l)) : 0.0;
  if (rank == 0 && tid == 0 && jb.steps) *jb.steps = done;
}

// ---------------------------------------------------------------- on-chip cooperative CPQR
// Same algorithm as cpqr_coop_kernel, but every CTA keeps its column slab in
// shared memory for the whole factorisation, so a step touches the matrix
// only on chip.  Each CTA publishes the current rows [j, M) of its local
// pivot candidate before the group barrier; after it, every CTA reads the
// winner's copy and forms the Householder vector redundantly.  One group
// barrier per step; the slab goes back to global memory at the end.
struct SmemCoopArgs {
  const QrJob* jobs;
  const int* cta_job;
  const int* cta_rank;
  const int* job_ctas;
  CoopCtl* ctl;
  CoopPart* parts;
  const int* part_off;  // 2 G entries per job (step parity)
  double* cand;         // 2 G M doubles per job
  const i64* cand_off;
  double* beta;
  const i64* beta_off;
};

constexpr int kSmemCoopU = 8;  // columns per block-wide reflector pass
constexpr int kOT = 512;        // threads of the on-chip / cluster CPQR CTA
constexpr int kOWarps = kOT / 32;

constexpr int kThreadColM = 96;  // slabs this short: one thread per column
// odd leading dimension for short slabs: thread-per-column access is then
// free of shared-memory bank conflicts
__host__ __device__ __forceinline__ int smem_coop_ld(int M) { return M <= kThreadColM ? (M | 1) : M; }
__host__ __device__ __forceinline__ size_t smem_coop_doubles(int M, int nown) {
  return size_t(smem_coop_ld(M)) * nown + M + 2 * nown + kOWarps * kSmemCoopU + 16 + (96 + 2 * nown + 1) / 2;
}

// kCl: one problem per thread-block cluster; partials and the pivot column
// are read from the peers' shared memory (DSMEM) and the group barrier is
// the hardware cluster barrier, so no grid-wide co-residency is needed.
#ifdef SBX_CPQR_PROF
__device__ long long g_cpqr_prof[64 * 8];
#define CPQR_T(ph)                                                              \
  do {                                                                          \
    if (blockIdx.x == 0 && threadIdx.x == 0 && j < 64) g_cpqr_prof[j * 8 + (ph)] = clock64(); \
  } while (0)
#else
#define CPQR_T(ph) \
  do {             \
  } while (0)
#endif
// The whole CTA applies step j's reflector to U slab columns cb.. (tall
// slabs with few columns per CTA): rows split over all threads, the column
// pointers and liveness hoisted out of the row loops; then the xGEQPF norm
// downdate of each live column (uniform decisions: every thread reads the
// same values).
template <int U>
__device__ __forceinline__ void tall_cols(double* S, int ldS, int cb, int nown, const int* mypos, const double* v,
                                          int j, int M, double tau, double* upd, double* dir, double thr,
                                          double* red) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* col[U];
  bool live[U];
  double d[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    live[u] = cb + u < nown && mypos[cb + u] >= 0;
    col[u] = S + size_t(cb + u) * ldS;
    d[u] = 0.0;
  }
  if (tau != 0.0 && M - j > 1) {
#pragma unroll 4
    for (int i = j + 1 + tid; i < M; i += kOT) {
      const double vi = v[i];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (live[u]) d[u] += vi * col[u][i];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) d[u] = warp_sum(d[u]);
    if (lane == 0)
#pragma unroll
      for (int u = 0; u < U; ++u) red[warp * U + u] = d[u];
    __syncthreads();
    double tw[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double t = 0.0;
      for (int w = 0; w < kOWarps; ++w) t += red[w * U + u];
      tw[u] = live[u] ? tau * (t + col[u][j]) : 0.0;
    }
    __syncthreads();  // everyone has read S[j, :] and red[]
#pragma unroll 4
    for (int i = j + 1 + tid; i < M; i += kOT) {
      const double vi = v[i];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (live[u]) col[u][i] -= vi * tw[u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (tid == u && live[u]) col[u][j] -= tw[u];
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (!live[u]) continue;
    const int c = cb + u;
    const double uu = upd[c];
    if (uu == 0.0) continue;
    double t = fabs(col[u][j]) / uu;
    t = (1.0 + t) * (1.0 - t);
    t = t < 0.0 ? 0.0 : t;
    const double rr = uu / dir[c];
    __syncthreads();  // all threads read upd[c] before it changes
    if (t * rr * rr <= thr) {
      double sacc = 0.0;
      for (int i = j + 1 + tid; i < M; i += kOT) sacc += col[u][i] * col[u][i];
      sacc = warp_sum(sacc);
      if (lane == 0) red[warp] = sacc;
      __syncthreads();
      if (tid == 0) {
        double s2 = 0.0;
        for (int w = 0; w < kOWarps; ++w) s2 += red[w];
        upd[c] = dir[c] = sqrt(s2);
      }
    } else if (tid == 0) {
      upd[c] = uu * sqrt(t);
    }
    __syncthreads();
  }
}

template <bool kCl>
__global__ void __launch_bounds__(kOT) cpqr_onchip_kernel(SmemCoopArgs args) {
  extern __shared__ double sm[];
  __shared__ CoopPart s_part[2];
  int job, rank, G;
  if constexpr (kCl) {
    cg::cluster_group cl = cg::this_cluster();
    G = int(cl.num_blocks());
    rank = int(cl.block_rank());
    job = int(blockIdx.x) / G;
  } else {
    job = args.cta_job[blockIdx.x];
    rank = args.cta_rank[blockIdx.x];
    G = args.job_ctas[job];
  }
  const QrJob jb = args.jobs[job];
  const int M = jb.M, n = jb.n, lda = jb.lda;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c0 = int(i64(n) * rank / G), c1 = int(i64(n) * (rank + 1) / G);
  const int nown = c1 - c0;
  const int ldS = smem_coop_ld(M);
  double* S = sm;                         // M x nown slab (ld ldS)
  double* v = S + size_t(ldS) * nown;     // M
  double* upd = v + M;                    // nown
  double* dir = upd + nown;               // nown
  double* red = dir + nown;               // kOWarps x kSmemCoopU
  double* sc = red + 8 * kSmemCoopU;      // 16
  int* ired = reinterpret_cast<int*>(sc + 16);  // 96
  int* mypos = ired + 96;                 // nown
  int* pivstep = mypos + nown;            // nown: step at which a column was pivoted
  CoopCtl* ctl = kCl ? nullptr : args.ctl + job;
  CoopPart* parts = kCl ? nullptr : args.parts + args.part_off[job];
  double* cand = kCl ? nullptr : args.cand + args.cand_off[job];
  double* sbeta = args.beta + args.beta_off[job];
  const double* Ag = jb.a;
  for (int c = warp; c < nown; c += kOWarps) {  // coalesced column loads, 4 in flight per lane
    const double* src = Ag + size_t(c0 + c) * lda;
    double* dst = S + size_t(c) * ldS;
    int i = lane;
    for (; i + 96 < M; i += 128) {
      const double x0 = __ldg(src + i), x1 = __ldg(src + i + 32), x2 = __ldg(src + i + 64),
                   x3 = __ldg(src + i + 96);
      dst[i] = x0;
      dst[i + 32] = x1;
      dst[i + 64] = x2;
      dst[i + 96] = x3;
    }
    for (; i < M; i += 32) dst[i] = __ldg(src + i);
  }
  for (int c = tid; c < nown; c += kOT) {
    mypos[c] = c0 + c;
    pivstep[c] = -1;
  }
  __syncthreads();
  if (nown >= kOWarps) {
    for (int c = warp; c < nown; c += kOWarps) {
      const double* col = S + size_t(c) * ldS;
      double s = 0.0;
      for (int i = lane; i < M; i += 32) s += col[i] * col[i];
      s = warp_sum(s);
      if (lane == 0) upd[c] = dir[c] = sqrt(s);
    }
  } else {  // few, tall columns: the whole CTA per column
    for (int c = 0; c < nown; ++c) {
      const double* col = S + size_t(c) * ldS;
      double s = 0.0;
      for (int i = tid; i < M; i += kOT) s += col[i] * col[i];
      s = warp_sum(s);
      if (lane == 0) red[warp] = s;
      __syncthreads();
      if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < kOWarps; ++w) t += red[w];
        upd[c] = dir[c] = sqrt(t);
      }
      __syncthreads();
    }
  }
  __syncthreads();
  const int size = min(M, n);
  const int steps_max = jb.max_steps > 0 ? min(size, jb.max_steps) : size;
  const double thr = sqrt(DBL_EPSILON);
  // wide slabs: a warp per 4 columns; tall, narrow slabs: the whole CTA per
  // column (rows split over all threads)
  const bool thread_mode = M <= kThreadColM;  // one thread per column
  const bool warp_mode = !thread_mode && (nown >= 8 || M <= 256);
  int done = 0;
  double r00 = 0.0;
  __shared__ int s_p;
  for (int j = 0; j < steps_max; ++j) {
    CPQR_T(0);
    double bv = -1.0;
    int bp = 0x7fffffff, bphys = -1;
    for (int c = tid; c < nown; c += kOT) {
      const int p = mypos[c];
      if (p >= 0 && better(upd[c], p, bv, bp)) {
        bv = upd[c];
        bp = p;
        bphys = c0 + c;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      const int oq = __shfl_xor_sync(0xffffffffu, bphys, o);
      if (better(ov, op, bv, bp)) {
        bv = ov;
        bp = op;
        bphys = oq;
      }
    }
    __shared__ int wphys[kOWarps];
    if (lane == 0) {
      red[warp] = bv;
      ired[warp] = bp;
      wphys[warp] = bphys;
    }
    __syncthreads();
    if (tid == 0) {
      double v0 = -1.0;
      int p0 = 0x7fffffff, q0 = -1;
      for (int w = 0; w < kOWarps; ++w)
        if (better(red[w], ired[w], v0, p0)) {
          v0 = red[w];
          p0 = ired[w];
          q0 = wphys[w];
        }
      if constexpr (kCl) {
        s_part[j & 1] = {v0, p0, q0};
      } else {
        parts[(j & 1) * G + rank] = {v0, p0, q0};
        s_p = q0;
      }
    }
    int p, lp, own;
    if constexpr (kCl) {
      cg::cluster_group cl = cg::this_cluster();
      CPQR_T(1);
      cl.sync();  // every CTA's partial visible (release / acquire at cluster scope)
      __shared__ int s_pick[3];
      if (warp == 0) {
        double bv = -1.0;
        int bp = 0x7fffffff, bq = -1, bo = -1;
        if (lane < G) {
          const CoopPart pt = *cl.map_shared_rank(&s_part[j & 1], lane);
          if (pt.phys >= 0) {
            bv = pt.val;
            bp = pt.pos;
            bq = pt.phys;
            bo = lane;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
          const int op = __shfl_xor_sync(0xffffffffu, bp, o);
          const int oq = __shfl_xor_sync(0xffffffffu, bq, o);
          const int oo = __shfl_xor_sync(0xffffffffu, bo, o);
          if (better(ov, op, bv, bp)) {
            bv = ov;
            bp = op;
            bq = oq;
            bo = oo;
          }
        }
        if (lane == 0) {
          s_pick[0] = bq;
          s_pick[1] = bp;
          s_pick[2] = bo;
        }
      }
      CPQR_T(2);
      __syncthreads();
      p = s_pick[0];
      lp = s_pick[1];
      own = s_pick[2];
    } else {
      __syncthreads();
      {  // publish the candidate's current rows [j, M)
        const int q = s_p;
        if (q >= 0) {
          const double* src = S + size_t(q - c0) * ldS;
          double* dst = cand + (size_t(j & 1) * G + rank) * M;
          for (int i = j + tid; i < M; i += kOT) __stcg(dst + i, src[i]);
        }
      }
      CPQR_T(6);
      group_barrier(ctl, unsigned(G));
      CPQR_T(1);
      coop_pick(parts + (j & 1) * G, G, red, ired, p, lp, own);
      CPQR_T(2);
    }
    for (int c = tid; c < nown; c += kOT) {
      if (c0 + c == p) {
        mypos[c] = -1;
        pivstep[c] = j;
      } else if (mypos[c] == j) {
        mypos[c] = lp;
      }
    }
    if (p >= c0 && p < c1 && tid == 0) jb.perm[j] = p;
    // the pivot column as its owner left it: a peer's slab (cluster) or the
    // owner's published copy; the owner never touches it again this launch
    const double* pc;
    if constexpr (kCl) {
      const int oc0 = int(i64(n) * own / G);
      pc = cg::this_cluster().map_shared_rank(S, own) + size_t(p - oc0) * ldS;
    } else {
      pc = cand + (size_t(j & 1) * G + own) * M;
    }
    auto ldp = [&](int i) { return kCl ? pc[i] : __ldcg(pc + i); };
    double part = 0.0;
    {
      // the pivot column comes from L2 (or a peer's shared memory): keep 8
      // loads in flight per thread; the sum keeps its ascending row order
      int i = j + 1 + tid;
      for (; i + 7 * kOT < M; i += 8 * kOT) {
        double x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = ldp(i + u * kOT);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          v[i + u * kOT] = x[u];
          part += x[u] * x[u];
        }
      }
      for (; i < M; i += kOT) {
        const double x = ldp(i);
        v[i] = x;
        part += x * x;
      }
    }
    part = warp_sum(part);
    if (lane == 0) red[warp] = part;
    __syncthreads();
    CPQR_T(3);
    const double tail = warp_sum(lane < kOWarps ? red[lane] : 0.0);
    const double cc = ldp(j);
    double tau, beta, denom;
    if (tail <= DBL_MIN) {
      tau = 0.0;
      beta = cc;
      denom = 0.0;
    } else {
      beta = sqrt(cc * cc + tail);
      if (cc >= 0.0) beta = -beta;
      denom = cc - beta;
      tau = (beta - cc) / beta;
    }
    __syncthreads();  // red[] reads done
    {
      const double rd = denom == 0.0 ? 0.0 : 1.0 / denom;
      for (int i = j + 1 + tid; i < M; i += kOT) v[i] *= rd;
    }
    if (j == 0) r00 = fabs(beta);
    if (rank == 0 && tid == 0) sbeta[j] = beta;
    __syncthreads();
    done = j + 1;
    CPQR_T(4);
    if (jb.stop_eps > 0.0 && !(fabs(beta) > jb.stop_eps * r00)) break;
    if (thread_mode) {
      for (int c = tid; c < nown; c += kOT) {
        if (mypos[c] < 0) continue;
        double* col = S + size_t(c) * ldS;
        if (tau != 0.0 && M - j > 1) {
          double d = col[j];
          for (int i = j + 1; i < M; ++i) d += v[i] * col[i];
          const double tw = tau * d;
          col[j] -= tw;
          for (int i = j + 1; i < M; ++i) col[i] -= v[i] * tw;
        }
        const double uu = upd[c];
        if (uu == 0.0) continue;
        double t = fabs(col[j]) / uu;
        t = (1.0 + t) * (1.0 - t);
        t = t < 0.0 ? 0.0 : t;
        const double rr = uu / dir[c];
        if (t * rr * rr <= thr) {
          double sacc = 0.0;
          for (int i = j + 1; i < M; ++i) sacc += col[i] * col[i];
          upd[c] = dir[c] = sqrt(sacc);
        } else {
          upd[c] = uu * sqrt(t);
        }
      }
    } else if (warp_mode) {
      for (int c = 4 * warp; c < nown; c += 4 * kOWarps) {
        double* cols[4];
        int slot[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const bool live = c + u < nown && mypos[c + u] >= 0;
          cols[u] = live ? S + size_t(c + u) * ldS : nullptr;
          slot[u] = c + u;
        }
        reflect_cols<4>(cols, slot, v, j, M, tau, true, upd, dir, thr, lane);
      }
    } else {
      for (int cb = 0; cb < nown;) {
        const int rem = nown - cb;
        const int U = rem <= 1 ? 1 : rem <= 2 ? 2 : rem <= 4 ? 4 : 8;
        if (U == 1) tall_cols<1>(S, ldS, cb, nown, mypos, v, j, M, tau, upd, dir, thr, red);
        else if (U == 2) tall_cols<2>(S, ldS, cb, nown, mypos, v, j, M, tau, upd, dir, thr, red);
        else if (U == 4) tall_cols<4>(S, ldS, cb, nown, mypos, v, j, M, tau, upd, dir, thr, red);
        else tall_cols<8>(S, ldS, cb, nown, mypos, v, j, M, tau, upd, dir, thr, red);
        cb += U;
      }
    }
    __syncthreads();
    CPQR_T(5);
  }
  if constexpr (kCl)
    cg::this_cluster().sync();  // peers are done reading this slab; sbeta complete
  else
    group_barrier(ctl, unsigned(G));
  for (int c = tid; c < nown; c += kOT)  // R diagonal of the pivoted columns
    if (pivstep[c] >= 0) S[pivstep[c] + size_t(c) * ldS] = __ldcg(sbeta + pivstep[c]);
  __syncthreads();
  double* Aw = jb.a;
  for (int c = warp; c < nown; c += kOWarps)
    for (int i = lane; i < M; i += 32) Aw[i + size_t(c0 + c) * lda] = S[i + size_t(c) * ldS];
  for (int c = tid; c < nown; c += kOT)
    if (mypos[c] >= 0) jb.perm[mypos[c]] = c0 + c;
  for (int l = rank * kOT + tid; l < size; l += G * kOT)
    jb.diag[l] = l < done ? fabs(__ldcg(sbeta + l)) : 0.0;
  if (rank == 0 && tid == 0 && jb.steps) *jb.steps = done;
}

// ---------------------------------------------------------------- register-resident cluster CPQR
// One problem per thread-block cluster of G CTAs (columns split across CTAs
// like cpqr_onchip_kernel<true>), but the slab lives in REGISTERS: warp w of
// a CTA owns CPW whole columns, lane l rows l + 32 r (r < RPL).  Per step:
//  (1) every warp picks its best live column (first max of the downdated
//      norms) and builds that column's Householder vector speculatively
//      (warp reductions only);
//  (2) one CTA barrier; every warp reduces the 16 warp candidates, the
//      winning warp publishes its vector in shared memory and pushes the
//      CTA candidate (norm, position, beta, tau) into every peer's smem;
//  (3) one cluster barrier; every warp reduces the G candidates locally,
//      copies the winner's vector from the owner CTA (DSMEM) and applies the
//      reflector + the xGEQPF norm downdate to its columns in registers.
// Two barriers and one DSMEM round trip per step.  Same pivot rule, stop
// rule and R layout (columns never move, perm names them) as the other
// engines; results agree to rounding (the Householder norms are summed per
// warp instead of across the CTA).
struct RegPart {
  double val, beta, tau;
  int pos, phys;
};

// First max of (val, pos) over the first W lanes (W a power of two <= 32);
// returns the winning lane, every lane gets it.
template <int W>
__device__ __forceinline__ int lane_argmax(double val, int pos) {
  int id = threadIdx.x & 31;
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, val, o);
    const int op = __shfl_xor_sync(0xffffffffu, pos, o);
    const int oi = __shfl_xor_sync(0xffffffffu, id, o);
    if (better(ov, op, val, pos)) {
      val = ov;
      pos = op;
      id = oi;
    }
  }
  return __shfl_sync(0xffffffffu, id, 0);
}

template <int RPL, int CPW>
__global__ void __launch_bounds__(kOT, 1) cpqr_reg_kernel(const QrJob* __restrict__ jobs) {
  cg::cluster_group cl = cg::this_cluster();
  const int G = int(cl.num_blocks()), rank = int(cl.block_rank());
  const QrJob jb = jobs[int(blockIdx.x) / G];
  const int M = jb.M, n = jb.n, lda = jb.lda;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c0 = int(i64(n) * rank / G), c1 = int(i64(n) * (rank + 1) / G);
  constexpr int MR = 32 * RPL;
  extern __shared__ double rsm[];
  double* pubv = rsm;            // 2 x MR: this CTA's candidate vector (step parity), v_j = 1
  double* vloc = rsm + 2 * MR;   // MR: the winning vector, local copy
  double* betas = vloc + MR;     // min(M, n)
  __shared__ RegPart wpart[kOWarps];
  __shared__ RegPart cpart[2][16];
  double a[CPW][RPL];
  double upd[CPW], dir[CPW];
  int pos[CPW], pst[CPW];
#pragma unroll
  for (int u = 0; u < CPW; ++u) {
    const int c = c0 + warp * CPW + u;
    const bool live = c < c1;
    const double* src = jb.a + size_t(live ? c : 0) * lda;
    double sq = 0.0;
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = lane + 32 * r;
      a[u][r] = (live && i < M) ? src[i] : 0.0;
      sq += a[u][r] * a[u][r];
    }
    sq = warp_sum(sq);
    upd[u] = dir[u] = sqrt(sq);
    pos[u] = live ? c : -1;
    pst[u] = -1;
  }
  const int size = min(M, n);
  const int steps_max = jb.max_steps > 0 ? min(size, jb.max_steps) : size;
  const double thr = sqrt(DBL_EPSILON);
  int done = 0;
  double r00 = 0.0;
  for (int j = 0; j < steps_max; ++j) {
    const int par = j & 1, rj = j >> 5, lj = j & 31;
    CPQR_T(0);
    // (1) warp candidate + its Householder vector
    int wu = -1;
    double wv = -1.0;
    int wp = 0x7fffffff;
#pragma unroll
    for (int u = 0; u < CPW; ++u)
      if (pos[u] >= 0 && better(upd[u], pos[u], wv, wp)) {
        wv = upd[u];
        wp = pos[u];
        wu = u;
      }
    double beta = 0.0, tau = 0.0, rd = 0.0;
    if (wu >= 0) {
      double part = 0.0, ccl = 0.0;
#pragma unroll
      for (int u = 0; u < CPW; ++u)
        if (u == wu) {  // warp-uniform
#pragma unroll
          for (int r = 0; r < RPL; ++r) {
            const int i = lane + 32 * r;
            if (i > j) part += a[u][r] * a[u][r];
            if (r == rj) ccl = a[u][r];
          }
        }
      const double tail = warp_sum(part);
      const double cc = __shfl_sync(0xffffffffu, ccl, lj);
      double denom;
      if (tail <= DBL_MIN) {
        tau = 0.0;
        beta = cc;
        denom = 0.0;
      } else {
        beta = sqrt(cc * cc + tail);
        if (cc >= 0.0) beta = -beta;
        denom = cc - beta;
        tau = (beta - cc) / beta;
      }
      rd = denom == 0.0 ? 0.0 : 1.0 / denom;
    }
    CPQR_T(1);
    if (lane == 0)
      wpart[warp] = {wu >= 0 ? wv : -1.0, beta, tau, wu >= 0 ? wp : 0x7fffffff, wu >= 0 ? c0 + warp * CPW + wu : -1};
    __syncthreads();
    // (2) CTA candidate; its warp publishes the vector and the candidate
    {
      const bool in = lane < kOWarps;
      const int bid = lane_argmax<kOWarps>(in ? wpart[lane].val : -1.0, in ? wpart[lane].pos : 0x7fffffff);
      if (warp == bid) {
#pragma unroll
        for (int u = 0; u < CPW; ++u)
          if (u == wu) {
#pragma unroll
            for (int r = 0; r < RPL; ++r) {
              const int i = lane + 32 * r;
              pubv[par * MR + i] = i > j ? a[u][r] * rd : (i == j ? 1.0 : 0.0);
            }
          }
        if (lane < G) *cl.map_shared_rank(&cpart[par][rank], lane) = wpart[bid];
      }
    }
    CPQR_T(2);
    cl.sync();
    CPQR_T(3);
    // (3) cluster winner
    const int own = lane_argmax<16>(lane < G ? cpart[par][lane].val : -1.0,
                                    lane < G ? cpart[par][lane].pos : 0x7fffffff);
    const RegPart w = cpart[par][own];
    const int p = w.phys, lp = w.pos;
    beta = w.beta;
    tau = w.tau;
    if (tid == 0) {
      betas[j] = beta;
      if (p >= c0 && p < c1) jb.perm[j] = p;
    }
#pragma unroll
    for (int u = 0; u < CPW; ++u) {
      if (c0 + warp * CPW + u == p) {
        pos[u] = -1;
        pst[u] = j;
      } else if (pos[u] == j) {
        pos[u] = lp;
      }
    }
    if (j == 0) r00 = fabs(beta);
    done = j + 1;
    if (jb.stop_eps > 0.0 && !(fabs(beta) > jb.stop_eps * r00)) break;
    CPQR_T(4);
    {
      const double* rv = cl.map_shared_rank(pubv + par * MR, own);
      for (int i = tid; i < MR; i += kOT) vloc[i] = rv[i];
    }
    __syncthreads();
    CPQR_T(5);
    double d[CPW];
#pragma unroll
    for (int u = 0; u < CPW; ++u) d[u] = 0.0;
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const double vi = vloc[lane + 32 * r];
#pragma unroll
      for (int u = 0; u < CPW; ++u) d[u] += vi * a[u][r];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int u = 0; u < CPW; ++u) d[u] += __shfl_xor_sync(0xffffffffu, d[u], o);
    double rowj[CPW];
#pragma unroll
    for (int u = 0; u < CPW; ++u) {
      rowj[u] = 0.0;
      if (pos[u] < 0) continue;  // warp-uniform
      const double tw = tau * d[u];
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        a[u][r] -= vloc[lane + 32 * r] * tw;
        if (r == rj) rowj[u] = a[u][r];
      }
    }
    // xGEQPF downdate, all columns at once (no branches between the
    // divisions); the rare recomputations afterwards
    bool rec[CPW];
#pragma unroll
    for (int u = 0; u < CPW; ++u) {
      const double colj = __shfl_sync(0xffffffffu, rowj[u], lj);
      const double uu = upd[u];
      double t = fabs(colj) / uu;
      t = (1.0 + t) * (1.0 - t);
      t = t < 0.0 ? 0.0 : t;
      const double rr = uu / dir[u];
      const bool live = pos[u] >= 0 && uu != 0.0;
      rec[u] = live && t * rr * rr <= thr;
      if (live && !rec[u]) upd[u] = uu * sqrt(t);
    }
#pragma unroll
    for (int u = 0; u < CPW; ++u) {
      if (!rec[u]) continue;  // warp-uniform
      double sq = 0.0;
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const int i = lane + 32 * r;
        if (i > j) sq += a[u][r] * a[u][r];
      }
      upd[u] = dir[u] = sqrt(warp_sum(sq));
    }
    CPQR_T(6);
  }
  cl.sync();  // peers are done reading this CTA's shared memory
#pragma unroll
  for (int u = 0; u < CPW; ++u) {
    const int c = c0 + warp * CPW + u;
    if (c >= c1) continue;
    double* dst = jb.a + size_t(c) * lda;
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = lane + 32 * r;
      if (i < M) dst[i] = i == pst[u] ? betas[i] : a[u][r];
    }
    if (pos[u] >= 0 && lane == 0) jb.perm[pos[u]] = c;
  }
  if (rank == 0) {
    for (int l = tid; l < size; l += kOT) jb.diag[l] = l < done ? fabs(betas[l]) : 0.0;
    if (tid == 0 && jb.steps) *jb.steps = done;
  }
}

// ---------------------------------------------------------------- streaming one-CTA CPQR
// One CTA (16 warps) per problem; the first ns columns of W^T live in shared
// memory, the rest are updated in place in global memory (L2 resident for
// these sizes), so any M <= 32 RPL fits one SM and a crowded batch needs one
// SM per problem instead of a cluster.  Warp w owns columns w, w + 16, ...;
// a column is processed in registers (lane l: rows l + 32 r, only rows >= j
// touched at step j).  Per step: warp-local candidate (after its downdate),
// one CTA barrier, the owner warp of the winner builds the Householder
// vector (v_j = 1 stored explicitly), a second barrier, then every warp
// reflects its live columns (read, dot, update, write back, downdate).
// Pivot rule, stop rule and R layout as the other engines; results agree to
// rounding.
struct StreamCand {
  double val;
  int pos, col;
};

template <int RPL>
__device__ __forceinline__ double reg_row(const double (&x)[RPL], int r) {
  double v = 0.0;
#pragma unroll
  for (int q = 0; q < RPL; ++q)
    if (q == r) v = x[q];
  return v;
}

template <int RPL>
__global__ void __launch_bounds__(kOT, 1) cpqr_stream_kernel(const QrJob* __restrict__ jobs, int ns_cap) {
  extern __shared__ double ssm[];
  const QrJob jb = jobs[blockIdx.x];
  const int M = jb.M, n = jb.n, lda = jb.lda;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int MR = 32 * RPL;
  const int size = min(M, n);
  double* v = ssm;                        // MR: Householder vector of the step (v_j = 1)
  double* upd = v + MR;                   // n
  double* dir = upd + n;                  // n
  double* betas = dir + n;                // size
  int* pos = reinterpret_cast<int*>(betas + size);  // n
  int* pst = pos + n;                               // n
  double* S = betas + size + (n + 1);     // ns x M resident slab (ld M)
  const int ns = min(n, ns_cap);
  __shared__ StreamCand wbest[kOWarps];
  __shared__ double s_beta, s_tau;
  auto colp = [&](int c) -> double* { return c < ns ? S + size_t(c) * M : jb.a + size_t(c) * lda; };
  // load the resident slab, column norms, positions
  for (int c = warp; c < n; c += kOWarps) {
    double* dst = colp(c);
    const double* src = jb.a + size_t(c) * lda;
    double sq = 0.0;
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = lane + 32 * r;
      if (i < M) {
        const double x = src[i];
        if (c < ns) dst[i] = x;
        sq += x * x;
      }
    }
    sq = warp_sum(sq);
    if (lane == 0) {
      upd[c] = dir[c] = sqrt(sq);
      pos[c] = c;
      pst[c] = -1;
    }
  }
  for (int i = tid; i < MR; i += kOT) v[i] = 0.0;
  __syncthreads();
  // warp candidates of step 0
  auto warp_candidate = [&]() {
    double bv = -1.0;
    int bp = 0x7fffffff, bc = -1;
    for (int c = warp + kOWarps * lane; c < n; c += kOWarps * 32) {
      const int pc = pos[c];
      if (pc >= 0 && better(upd[c], pc, bv, bp)) {
        bv = upd[c];
        bp = pc;
        bc = c;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
      if (better(ov, op, bv, bp)) {
        bv = ov;
        bp = op;
        bc = oc;
      }
    }
    if (lane == 0) wbest[warp] = {bc >= 0 ? bv : -1.0, bc >= 0 ? bp : 0x7fffffff, bc};
  };
  warp_candidate();
  const int steps_max = jb.max_steps > 0 ? min(size, jb.max_steps) : size;
  const double thr = sqrt(DBL_EPSILON);
  int done = 0;
  double r00 = 0.0;
  for (int j = 0; j < steps_max; ++j) {
    const int rj = j >> 5, lj = j & 31;
    __syncthreads();  // candidates published; previous reflections written
    // CTA winner (every warp computes it)
    StreamCand w = lane < kOWarps ? wbest[lane] : StreamCand{-1.0, 0x7fffffff, -1};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, w.val, o);
      const int op = __shfl_xor_sync(0xffffffffu, w.pos, o);
      const int oc = __shfl_xor_sync(0xffffffffu, w.col, o);
      if (better(ov, op, w.val, w.pos)) w = {ov, op, oc};
    }
    const int p = w.col, lp = w.pos;
    if (warp == (p & (kOWarps - 1))) {  // owner builds the Householder vector
      const double* pc = colp(p);
      double a[RPL];
      double part = 0.0, ccl = 0.0;
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const int i = lane + 32 * r;
        a[r] = (i >= j && i < M) ? pc[i] : 0.0;
        if (i > j) part += a[r] * a[r];
        if (r == rj) ccl = a[r];
      }
      const double tail = warp_sum(part);
      const double cc = __shfl_sync(0xffffffffu, ccl, lj);
      double beta, tau, denom;
      if (tail <= DBL_MIN) {
        tau = 0.0;
        beta = cc;
        denom = 0.0;
      } else {
        beta = sqrt(cc * cc + tail);
        if (cc >= 0.0) beta = -beta;
        denom = cc - beta;
        tau = (beta - cc) / beta;
      }
      const double rd = denom == 0.0 ? 0.0 : 1.0 / denom;
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const int i = lane + 32 * r;
        if (i >= j - 1 && i < MR) v[i] = i > j ? a[r] * rd : (i == j ? 1.0 : 0.0);
      }
      if (lane == 0) {
        s_beta = beta;
        s_tau = tau;
        betas[j] = beta;
        jb.perm[j] = p;
      }
    }
    // positions (each warp its own columns; the winner's owner marks it)
    for (int c = warp + kOWarps * lane; c < n; c += kOWarps * 32) {
      if (c == p) {
        pos[c] = -1;
        pst[c] = j;
      } else if (pos[c] == j) {
        pos[c] = lp;
      }
    }
    __syncthreads();  // v, beta, tau, positions visible
    const double beta = s_beta, tau = s_tau;
    if (j == 0) r00 = fabs(beta);
    done = j + 1;
    if (jb.stop_eps > 0.0 && !(fabs(beta) > jb.stop_eps * r00)) break;
    const bool refl = tau != 0.0 && M - j > 1;
    // CPI columns per pass share the loads of v and the row masks; row
    // blocks below j are skipped (warp-uniform), v is zero there anyway
    constexpr int CPI = RPL <= 20 ? 2 : 1;
    for (int cb = warp; cb < n; cb += CPI * kOWarps) {
      int cc[CPI];
      bool live[CPI], any = false;
      double* colv[CPI];
#pragma unroll
      for (int u = 0; u < CPI; ++u) {
        cc[u] = cb + u * kOWarps;
        live[u] = cc[u] < n && pos[cc[u]] >= 0;
        any |= live[u];
        colv[u] = live[u] ? colp(cc[u]) : nullptr;
      }
      if (!any) continue;  // warp-uniform
      double a[CPI][RPL];
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const int i = lane + 32 * r;
        const bool ok = r >= rj && i >= j && i < M;
#pragma unroll
        for (int u = 0; u < CPI; ++u) a[u][r] = (ok && live[u]) ? colv[u][i] : 0.0;
      }
      double rowj[CPI];
#pragma unroll
      for (int u = 0; u < CPI; ++u) rowj[u] = 0.0;
      if (refl) {
        double d[CPI];
#pragma unroll
        for (int u = 0; u < CPI; ++u) d[u] = 0.0;
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          if (r < rj) continue;
          const double vi = v[lane + 32 * r];
#pragma unroll
          for (int u = 0; u < CPI; ++u) d[u] += vi * a[u][r];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int u = 0; u < CPI; ++u) d[u] += __shfl_xor_sync(0xffffffffu, d[u], o);
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          if (r < rj) continue;
          const int i = lane + 32 * r;
          const double vi = v[i];
          const bool st = i >= j && i < M;
#pragma unroll
          for (int u = 0; u < CPI; ++u) {
            a[u][r] -= vi * (tau * d[u]);
            if (st && live[u]) colv[u][i] = a[u][r];
            if (r == rj) rowj[u] = a[u][r];
          }
        }
      } else {
#pragma unroll
        for (int u = 0; u < CPI; ++u) rowj[u] = reg_row(a[u], rj);
      }
#pragma unroll
      for (int u = 0; u < CPI; ++u) {
        if (!live[u]) continue;
        const int c = cc[u];
        const double colj = __shfl_sync(0xffffffffu, rowj[u], lj);
        const double uu = upd[c];
        if (uu == 0.0) continue;
        double t = fabs(colj) / uu;
        t = (1.0 + t) * (1.0 - t);
        t = t < 0.0 ? 0.0 : t;
        const double rr = uu / dir[c];
        if (t * rr * rr <= thr) {
          double sq = 0.0;
#pragma unroll
          for (int r = 0; r < RPL; ++r) {
            const int i = lane + 32 * r;
            if (i > j) sq += a[u][r] * a[u][r];
          }
          sq = sqrt(warp_sum(sq));
          if (lane == 0) upd[c] = dir[c] = sq;
        } else if (lane == 0) {
          upd[c] = uu * sqrt(t);
        }
      }
    }
    __syncwarp();
    warp_candidate();
  }
  __syncthreads();
  // write back: resident columns, and the R diagonal of the pivoted ones
  for (int c = warp; c < n; c += kOWarps) {
    double* dst = jb.a + size_t(c) * lda;
    const int ps = pst[c];
    if (c < ns) {
      const double* src = S + size_t(c) * M;
      for (int i = lane; i < M; i += 32) dst[i] = i == ps ? betas[i] : src[i];
    } else if (ps >= 0 && lane == 0) {
      dst[ps] = betas[ps];
    }
    if (lane == 0 && pos[c] >= 0) jb.perm[pos[c]] = c;
  }
  for (int l = tid; l < size; l += kOT) jb.diag[l] = l < done ? fabs(betas[l]) : 0.0;
  if (tid == 0 && jb.steps) *jb.steps = done;
}

// ---------------------------------------------------------------- interpolation
// One work item = (job, first column of a 128-column chunk of R12), or
// (job, -1) for the k identity rows.  Every row of P is written exactly once,
// so P needs no zero fill.
constexpr int kIT = 128;

__global__ void __launch_bounds__(kIT) interp_kernel(const InterpJob* __restrict__ jobs,
                                                    const int2* __restrict__ items) {
  const int2 it = items[blockIdx.x];
  const InterpJob jb = jobs[it.x];
  const int n = jb.n, k = jb.k, nk = n - k;
  if (it.y < 0) {  // P(J_i, :) = e_i
    for (i64 idx = threadIdx.x; idx < i64(k) * k; idx += kIT) {
      const int i = int(idx % k), c = int(idx / k);
      jb.P[jb.perm[i] + size_t(c) * jb.ldp] = i == c ? 1.0 : 0.0;
    }
    return;
  }
  const int* cm = jb.colmap;
  const int j = it.y + threadIdx.x;
  if (j >= nk) return;
  const double* R = jb.a;
  const size_t cj = size_t(cm ? cm[k + j] : k + j);
  for (int i = k - 1; i >= 0; --i) {  // back substitution R11 t = r12 (T row-major [i][j])
    double s = R[i + cj * jb.lda];
    for (int l = i + 1; l < k; ++l) s -= R[i + size_t(cm ? cm[l] : l) * jb.lda] * jb.T[size_t(l) * nk + j];
    jb.T[size_t(i) * nk + j] = s / R[i + size_t(cm ? cm[i] : i) * jb.lda];
  }
  double* prow = jb.P + jb.perm[k + j];
  for (int i = 0; i < k; ++i) prow[size_t(i) * jb.ldp] = jb.T[size_t(i) * nk + j];
}

// Warp per column of R12 (k <= 32 * RPL): lane l holds rows l, l + 32, ...
// of the right-hand side in registers; column-oriented back substitution
// (x_i broadcast by shuffle, then an axpy with column i of R11), so the
// dependent chain per step is one shuffle + one division instead of a
// k-long dot product per row.  Eight columns per CTA.
constexpr int kIWarps = 8;

template <int RPL>
__global__ void __launch_bounds__(kIWarps * 32) interp_warp_kernel(const InterpJob* __restrict__ jobs,
                                                                   const int2* __restrict__ items) {
  const int2 it = items[blockIdx.x];
  const InterpJob jb = jobs[it.x];
  const int n = jb.n, k = jb.k, nk = n - k;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (it.y < 0) {  // P(J_i, :) = e_i
    for (i64 idx = threadIdx.x; idx < i64(k) * k; idx += kIWarps * 32) {
      const int i = int(idx % k), c = int(idx / k);
      jb.P[jb.perm[i] + size_t(c) * jb.ldp] = i == c ? 1.0 : 0.0;
    }
    return;
  }
  const int j = it.y + warp;
  if (j >= nk) return;
  const int* cm = jb.colmap;
  const double* R = jb.a;
  const size_t lda = size_t(jb.lda);
  const double* rj = R + size_t(cm ? cm[k + j] : k + j) * lda;
  double b[RPL];
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    const int l = lane + 32 * r;
    b[r] = l < k ? rj[l] : 0.0;
  }
  double* prow = jb.P + jb.perm[k + j];
  auto col_of = [&](int i) { return R + size_t(cm ? cm[i] : i) * lda; };
#pragma unroll
  for (int rb = RPL - 1; rb >= 0; --rb) {
    if (32 * rb >= k) continue;
    const int top = min(31, k - 1 - 32 * rb);
    // column i of R11 is fetched one step ahead of its use
    const double* ri = col_of(32 * rb + top);
    double d = ri[32 * rb + top], rv[RPL];
#pragma unroll
    for (int r = 0; r <= rb; ++r) rv[r] = lane + 32 * r < k ? ri[lane + 32 * r] : 0.0;
    for (int ii = top; ii >= 0; --ii) {
      const int i = 32 * rb + ii;
      double dn = 1.0, vn[RPL];
      if (ii > 0) {
        const double* rn = col_of(i - 1);
        dn = rn[i - 1];
#pragma unroll
        for (int r = 0; r <= rb; ++r) vn[r] = lane + 32 * r < k ? rn[lane + 32 * r] : 0.0;
      }
      const double x = __shfl_sync(0xffffffffu, b[rb], ii) / d;
      if (lane == 0) prow[size_t(i) * jb.ldp] = x;
#pragma unroll
      for (int r = 0; r <= rb; ++r)
        if (r < rb || lane < ii) b[r] -= rv[r] * x;
      d = dn;
#pragma unroll
      for (int r = 0; r <= rb; ++r) rv[r] = vn[r];
    }
  }
}

// ---------------------------------------------------------------- GEMM (DMMA)
constexpr int gTM = 64, gTN = 64, gKC = 16, gPad = 8;


// 8-byte asynchronous global -> shared copy; src_bytes 0 zero-fills
__device__ __forceinline__ void gcp_async8(double* dst, const double* src, bool pred) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(pred ? 8 : 0));
}
__device__ __forceinline__ void gcp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void gcp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

constexpr int gStages = 4;
struct GemmSmem {
  double As[gStages][gKC][gTM + gPad];
  double Bs[gStages][gKC][gTN + gPad];
};

// 64 x 64 output tile per CTA on FP64 tensor cores (mma.sync.m8n8k4 ->
// DMMA), 8 warps of 16 x 32; K moves through a gStages-deep cp.async
// pipeline (8-byte copies: operands may be transposed and unaligned), so
// the global loads of chunk ch + 3 are in flight while chunk ch computes.
__global__ void __launch_bounds__(256) gemm_kernel(const GemmJob* __restrict__ jobs,
                                                   const int4* __restrict__ tiles) {
  extern __shared__ __align__(16) double gsm[];
  GemmSmem& S = *reinterpret_cast<GemmSmem*>(gsm);
  const int4 tl = tiles[blockIdx.x];
  const GemmJob jb = jobs[tl.x];
  const int row0 = tl.y, col0 = tl.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int wm = (warp & 3) * 16, wn = (warp >> 2) * 32;
  double c[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) c[a][b][0] = c[a][b][1] = 0.0;
  const int kbeg = jb.splitk > 1 ? tl.w * jb.kchunk : 0;
  const int K = jb.splitk > 1 ? min(jb.k, kbeg + jb.kchunk) : jb.k;
  const int nch = (K - kbeg + gKC - 1) / gKC;
  auto issue = [&](int st, int k0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = threadIdx.x + q * 256;
      int kk, rr;
      if (!jb.ta) {
        kk = idx >> 6;
        rr = idx & 63;
      } else {
        rr = idx >> 4;
        kk = idx & 15;
      }
      const int gr = row0 + rr, gk = k0 + kk;
      const bool pa = gr < jb.m && gk < K;
      gcp_async8(&S.As[st][kk][rr], pa ? (jb.ta ? jb.A + gk + size_t(gr) * jb.lda : jb.A + gr + size_t(gk) * jb.lda)
                                       : jb.A,
                 pa);
      int kb, cc;
      if (!jb.tb) {
        cc = idx >> 4;
        kb = idx & 15;
      } else {
        kb = idx >> 6;
        cc = idx & 63;
      }
      const int gc = col0 + cc, gkb = k0 + kb;
      const bool pb = gc < jb.n && gkb < K;
      gcp_async8(&S.Bs[st][kb][cc],
                 pb ? (jb.tb ? jb.B + gc + size_t(gkb) * jb.ldb : jb.B + gkb + size_t(gc) * jb.ldb) : jb.B, pb);
    }
  };
#pragma unroll
  for (int st = 0; st < gStages - 1; ++st) {
    if (st < nch) issue(st, kbeg + st * gKC);
    gcp_commit();
  }
  for (int ch = 0; ch < nch; ++ch) {
    const int st = ch % gStages;
    gcp_wait<gStages - 2>();
    __syncthreads();  // chunk ch visible to all; stage (ch - 1) % gStages free
    const int nx = ch + gStages - 1;
    if (nx < nch) issue(nx % gStages, kbeg + nx * gKC);
    gcp_commit();
#pragma unroll
    for (int k4 = 0; k4 < gKC; k4 += 4) {
      double af[2], bf[4];
#pragma unroll
      for (int a = 0; a < 2; ++a) af[a] = S.As[st][k4 + tig][wm + a * 8 + gid];
#pragma unroll
      for (int b = 0; b < 4; ++b) bf[b] = S.Bs[st][k4 + tig][wn + b * 8 + gid];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma(c[a][b][0], c[a][b][1], af[a], bf[b]);
    }
  }
  gcp_wait<0>();
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int row = row0 + wm + a * 8 + gid;
    if (row >= jb.m) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = col0 + wn + b * 8 + 2 * tig + h;
        if (col >= jb.n) continue;
        if (jb.splitk > 1) {
          jb.part[size_t(tl.w) * jb.m * jb.n + row + size_t(col) * jb.m] = c[a][b][h];
        } else {
          double* dst = jb.C + row + size_t(col) * jb.ldc;
          const double v = jb.alpha * c[a][b][h];
          *dst = jb.beta == 0.0 ? v : v + jb.beta * *dst;
        }
      }
  }
}

// ---------------------------------------------------------------- thin product (m, n <= 160, long K)
// C = A B with a small output and a long inner dimension (the Woodbury
// operator's R X, els.cpp:124: 146 x 40960 x 146): one CTA per K range
// computes the WHOLE output block as DMMA accumulator tiles in registers
// (8 warps, 4 x 2, each 5 x 10 tiles of 8 x 8), so no output-tile padding to
// 64 and every operand element is read once; A (column-major, rows
// contiguous) and B (column-major, k contiguous) move through a 4-stage
// 16-byte cp.async pipeline into layouts whose fragment loads are
// bank-conflict free.  After a grid barrier (cooperative launch, one CTA per
// SM) every CTA sums its slice of the output over all partials in a fixed
// order (deterministic).
constexpr int kThinKC = 16, kThinStages = 4, kThinTA = 5;
constexpr int kThinMP = 160;            // 4 warp rows x 5 tiles x 8 = 2 warp columns x 10 tiles x 8
constexpr int kThinLdA = kThinMP + 4;   // As[k][row]: (tig * ld + gid) distinct mod 16
constexpr int kThinLdB = kThinKC + 4;   // Bs[col][k]: (gid * ld + tig) distinct mod 16
struct ThinSmem {
  double As[kThinStages][kThinKC][kThinLdA];
  double Bs[kThinStages][kThinMP][kThinLdB];
};

__device__ __forceinline__ void gcp_async16(double* dst, const double* src, int bytes) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(bytes));
}

// WC warp columns x TB tile columns per warp: <2, 10> (8 warps) or <4, 5> (16 warps) cover 160 output
// columns, <4, 2> covers 64 (R y of a 64-RHS Woodbury solve)
template <int WC, int TB>
__global__ void __launch_bounds__(128 * WC, 1) thin_gemm_kernel(const GemmJob* __restrict__ jobs) {
  constexpr int NT = 128 * WC, kThinTB = TB;
  extern __shared__ __align__(16) double gsm[];
  ThinSmem& S = *reinterpret_cast<ThinSmem*>(gsm);
  const GemmJob jb = jobs[0];
  const int m = jb.m, n = jb.n;
  const int kb = int(blockIdx.x) * jb.kchunk, ke = min(jb.k, kb + jb.kchunk);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int wr = warp & 3, wc = warp >> 2;
  const int mp = (m + 1) / 2;  // 16-byte pairs per A column
  auto issue = [&](int st, int k0) {
    for (int e = tid; e < kThinKC * mp; e += NT) {  // A: rows contiguous
      const int kk = e / mp, r = (e - kk * mp) * 2;
      const int gk = k0 + kk;
      const int bytes = gk < ke ? (r + 1 < m ? 16 : 8) : 0;
      gcp_async16(&S.As[st][kk][r], bytes ? jb.A + r + size_t(gk) * jb.lda : jb.A, bytes);
    }
    for (int e = tid; e < n * (kThinKC / 2); e += NT) {  // B: k contiguous
      const int c = e / (kThinKC / 2), kk = (e - c * (kThinKC / 2)) * 2;
      const int gk = k0 + kk;
      const int bytes = gk + 1 < ke ? 16 : (gk < ke ? 8 : 0);
      gcp_async16(&S.Bs[st][c][kk], bytes ? jb.B + gk + size_t(c) * jb.ldb : jb.B, bytes);
    }
  };
  double acc[kThinTA][kThinTB][2];
#pragma unroll
  for (int a = 0; a < kThinTA; ++a)
#pragma unroll
    for (int b = 0; b < kThinTB; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int nch = (ke - kb + kThinKC - 1) / kThinKC;
#pragma unroll
  for (int c = 0; c < kThinStages - 1; ++c) {
    if (c < nch) issue(c, kb + c * kThinKC);
    gcp_commit();
  }
  for (int ch = 0; ch < nch; ++ch) {
    const int st = ch % kThinStages;
    gcp_wait<kThinStages - 2>();
    __syncthreads();  // chunk ch visible; the stage of chunk ch - 1 is free
    const int nx = ch + kThinStages - 1;
    if (nx < nch) issue(nx % kThinStages, kb + nx * kThinKC);
    gcp_commit();
#pragma unroll
    for (int k4 = 0; k4 < kThinKC; k4 += 4) {
      double af[kThinTA];
#pragma unroll
      for (int a = 0; a < kThinTA; ++a) af[a] = S.As[st][k4 + tig][8 * (kThinTA * wr + a) + gid];
#pragma unroll
      for (int b = 0; b < kThinTB; ++b) {
        const double bf = S.Bs[st][8 * (kThinTB * wc + b) + gid][k4 + tig];
#pragma unroll
        for (int a = 0; a < kThinTA; ++a) dmma(acc[a][b][0], acc[a][b][1], af[a], bf);
      }
    }
  }
  gcp_wait<0>();
  double* part = jb.part + size_t(blockIdx.x) * m * n;
#pragma unroll
  for (int a = 0; a < kThinTA; ++a)
#pragma unroll
    for (int b = 0; b < kThinTB; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int row = 8 * (kThinTA * wr + a) + gid, col = 8 * (kThinTB * wc + b) + 2 * tig + e;
        if (row < m && col < n) part[row + size_t(col) * m] = acc[a][b][e];
      }
  // every CTA then reduces its own slice of the output over all partials, in a
  // fixed order (cooperative launch: the grid is co-resident)
  cooperative_groups::this_grid().sync();
  const int total = m * n, G = int(gridDim.x);
  const int per = (total + G - 1) / G, o0 = int(blockIdx.x) * per;
  const int cnt = min(per, total - o0);
  auto store = [&](int o, double v) {
    const int idx = o0 + o, row = idx % m, col = idx / m;
    double* dst = jb.C + row + size_t(col) * jb.ldc;
    v *= jb.alpha;
    *dst = jb.beta == 0.0 ? v : v + jb.beta * *dst;
  };
  if (per <= NT) {  // NT / per groups of threads take interleaved partials; combined in group order
    const int groups = min(NT / per, 8);
    const int g = tid / per, o = tid - g * per;
    double* sred = gsm;
    if (g < groups && o < cnt) {
      double v = 0.0;
      const double* src = jb.part + o0 + o;
      int q = g;
      for (; q + 15 * groups < G; q += 16 * groups) {  // 16 loads in flight, summed in split order
        double t[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) t[i] = __ldcg(src + size_t(q + i * groups) * total);
#pragma unroll
        for (int i = 0; i < 16; ++i) v += t[i];
      }
      for (; q < G; q += groups) v += __ldcg(src + size_t(q) * total);
      sred[g * per + o] = v;
    }
    __syncthreads();
    if (tid < cnt) {
      double v = sred[tid];
      for (int q = 1; q < groups; ++q) v += sred[q * per + tid];
      store(tid, v);
    }
  } else {
    for (int o = tid; o < cnt; o += NT) {
      double v = 0.0;
      for (int q = 0; q < G; ++q) v += __ldcg(jb.part + size_t(q) * total + o0 + o);
      store(o, v);
    }
  }
}

// fixed-order reduction of split-K partials: C = alpha * sum_s part_s + beta * C
__global__ void splitk_reduce_kernel(const GemmJob* __restrict__ jobs) {
  const GemmJob jb = jobs[blockIdx.y];
  if (jb.splitk <= 1) return;
  const i64 total = i64(jb.m) * jb.n;
  for (i64 idx = blockIdx.x * i64(blockDim.x) + threadIdx.x; idx < total;
       idx += i64(gridDim.x) * blockDim.x) {
    double acc = 0.0;
    int s = 0;
    for (; s + 16 <= jb.splitk; s += 16) {  // 16 loads in flight, summed in split order
      double v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = __ldcg(jb.part + size_t(s + q) * total + idx);
#pragma unroll
      for (int q = 0; q < 16; ++q) acc += v[q];
    }
    for (; s < jb.splitk; ++s) acc += __ldcg(jb.part + size_t(s) * total + idx);
    const i64 row = idx % jb.m, col = idx / jb.m;
    double* dst = jb.C + row + col * jb.ldc;
    const double v = jb.alpha * acc;
    *dst = jb.beta == 0.0 ? v : v + jb.beta * *dst;
  }
}

// ---------------------------------------------------------------- LU
// Warp-level forward/back substitution on one column held in registers
// (lanes own rows lane, lane+32, ...).  Up to 16 values per lane (n <= 512).
constexpr int kMaxRowsPerLane = 16;

// Register-resident slot access (a dynamic index would spill the array).
__device__ __forceinline__ double rget(const double (&x)[kMaxRowsPerLane], int s) {
  double v = 0.0;
#pragma unroll
  for (int q = 0; q < kMaxRowsPerLane; ++q)
    if (q == s) v = x[q];
  return v;
}
__device__ __forceinline__ void rset(double (&x)[kMaxRowsPerLane], int s, double val) {
#pragma unroll
  for (int q = 0; q < kMaxRowsPerLane; ++q)
    if (q == s) x[q] = val;
}

__device__ void warp_lu_solve(const double* lu, int n, int lda, double (&x)[kMaxRowsPerLane],
                              int lane) {
  // L z = x (unit lower)
  for (int j = 0; j < n; ++j) {
    const double zj = __shfl_sync(0xffffffffu, rget(x, j >> 5), j & 31);
#pragma unroll
    for (int q = 0; q < kMaxRowsPerLane; ++q) {
      const int i = lane + 32 * q;
      if (i > j && i < n) x[q] -= lu[i + size_t(j) * lda] * zj;
    }
  }
  // U x = z
  for (int j = n - 1; j >= 0; --j) {
    const int owner = j & 31, slot = j >> 5;
    double xj = __shfl_sync(0xffffffffu, rget(x, slot), owner);
    xj /= lu[j + size_t(j) * lda];
    if (lane == owner) rset(x, slot, xj);
#pragma unroll
    for (int q = 0; q < kMaxRowsPerLane; ++q) {
      const int i = lane + 32 * q;
      if (i < j) x[q] -= lu[i + size_t(j) * lda] * xj;
    }
  }
}

// (A^T) x = b with PA = LU:  U^T y = b, L^T z = y, x = P^T z
__device__ void warp_lu_solve_t(const double* lu, int n, int lda, double (&x)[kMaxRowsPerLane],
                                int lane) {
  for (int j = 0; j < n; ++j) {  // U^T y = b : y_j = (b_j - sum_{p<j} U(p,j) y_p)/U(j,j)
    const int owner = j & 31, slot = j >> 5;
    double part = 0.0;
#pragma unroll
    for (int q = 0; q < kMaxRowsPerLane; ++q) {
      const int p = lane + 32 * q;
      if (p < j) part += lu[p + size_t(j) * lda] * x[q];
    }
    part = warp_sum(part);
    if (lane == owner) rset(x, slot, (rget(x, slot) - part) / lu[j + size_t(j) * lda]);
    __syncwarp();
  }
  for (int j = n - 1; j >= 0; --j) {  // L^T z = y : z_j = y_j - sum_{p>j} L(p,j) z_p
    const int owner = j & 31, slot = j >> 5;
    double part = 0.0;
#pragma unroll
    for (int q = 0; q < kMaxRowsPerLane; ++q) {
      const int p = lane + 32 * q;
      if (p > j && p < n) part += lu[p + size_t(j) * lda] * x[q];
    }
    part = warp_sum(part);
    if (lane == owner) rset(x, slot, rget(x, slot) - part);
    __syncwarp();
  }
}

// Reciprocal 1-norm condition estimate (Eigen ConditionEstimator.h,
// Hager/Higham) of a matrix with 1-norm l1 from its explicit inverse X
// (n x n, ld n), CTA-wide (NT threads; with NT < kT the caller presets
// red[NT/32..] = 0 and ired likewise beyond the live warps' slots: the block
// reductions read kWarps slots).  work: 4n doubles; red/ired: block scratch.
template <int NT = kT>
__device__ double rcond_from_inverse(const double* X, int n, double l1, double* work, double* red, int* ired) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  {
    __shared__ int s_flag;
    double* v = work;          // n
    double* sg = work + n;     // n
    double* osg = work + 2 * n;  // n
    double* tmp = work + 3 * n;  // n
    auto gemv = [&](const double* x, double* y, bool trans) {  // y = X x or X^T x
      if (!trans) {
        for (int i = tid; i < n; i += NT) {
          double a = 0.0;
          for (int c = 0; c < n; ++c) a += X[i + size_t(c) * n] * x[c];
          y[i] = a;
        }
      } else {
        for (int c = warp; c < n; c += NT / 32) {
          double a = 0.0;
          for (int i = lane; i < n; i += 32) a += X[i + size_t(c) * n] * x[i];
          a = warp_sum(a);
          if (lane == 0) y[c] = a;
        }
      }
      __syncthreads();
    };
    auto l1sum = [&](const double* x) {
      double a = 0.0;
      for (int i = tid; i < n; i += NT) a += fabs(x[i]);
      return block_sum(a, red);
    };
    double result;
    if (l1 == 0.0) {
      result = 0.0;
    } else if (n == 1) {
      result = 1.0;
    } else {
      for (int i = tid; i < n; i += NT) tmp[i] = 1.0 / double(n);
      __syncthreads();
      gemv(tmp, v, false);
      double lower = l1sum(v), old_lower = lower;
      int old_vmax = -1;
      for (int it = 0; it < 4; ++it) {
        int differs = 0;
        for (int i = tid; i < n; i += NT) {
          sg[i] = v[i] < 0.0 ? -1.0 : 1.0;
          if (it > 0 && sg[i] != osg[i]) differs = 1;
        }
        if (tid == 0) s_flag = 0;
        __syncthreads();
        if (differs) s_flag = 1;
        __syncthreads();
        if (it > 0 && s_flag == 0) break;
        gemv(sg, tmp, true);
        double bv = -1.0;
        int bi = 0x7fffffff;
        for (int i = tid; i < n; i += NT)
          if (fabs(tmp[i]) > bv) {
            bv = fabs(tmp[i]);
            bi = i;
          }
        double mv;
        int vmax;
        block_argmax(bv, bi, red, ired, mv, vmax);
        if (vmax == old_vmax) break;
        for (int i = tid; i < n; i += NT) v[i] = X[i + size_t(vmax) * n];
        __syncthreads();
        lower = l1sum(v);
        if (lower <= old_lower) break;
        for (int i = tid; i < n; i += NT) osg[i] = sg[i];
        __syncthreads();
        old_vmax = vmax;
        old_lower = lower;
      }
      for (int i = tid; i < n; i += NT)
        tmp[i] = (i % 2 == 0 ? 1.0 : -1.0) * (1.0 + double(i) / double(n - 1));
      __syncthreads();
      gemv(tmp, v, false);
      const double alt = 2.0 * l1sum(v) / (3.0 * double(n));
      const double inv_norm = fmax(lower, alt);
      result = inv_norm == 0.0 ? 0.0 : (1.0 / inv_norm) / l1;
    }
    return result;
  }
}

__global__ void __launch_bounds__(kT) lu_kernel(const LuJob* __restrict__ jobs, int smem_doubles) {
  extern __shared__ double sm[];
  const LuJob jb = jobs[blockIdx.x];
  const int n = jb.n;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* red = sm;
  int* ired = reinterpret_cast<int*>(sm + 32);
  double* mat = sm + 64;
  const bool in_smem = 64 + size_t(n) * n <= size_t(smem_doubles);
  double* A = jb.a;
  int lda = jb.lda;
  // 1-norm of the original matrix (Eigen m_l1_norm)
  __shared__ double l1;
  if (tid == 0) l1 = 0.0;
  __syncthreads();
  for (int c = warp; c < n; c += kWarps) {
    double s = 0.0;
    for (int i = lane; i < n; i += 32) s += fabs(jb.a[i + size_t(c) * jb.lda]);
    s = warp_sum(s);
    if (lane == 0) atomicMax(reinterpret_cast<unsigned long long*>(&l1), __double_as_longlong(s));
  }
  if (in_smem) {
    for (int c = warp; c < n; c += kWarps)
      for (int i = lane; i < n; i += 32) mat[i + size_t(c) * n] = jb.a[i + size_t(c) * jb.lda];
    A = mat;
    lda = n;
  }
  for (int i = tid; i < n; i += kT) jb.piv[i] = i;
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int i = k + tid; i < n; i += kT) {
      const double v = fabs(A[i + size_t(k) * lda]);
      if (v > bv) {
        bv = v;
        bi = i;
      }
    }
    double mv;
    int p;
    block_argmax(bv, bi, red, ired, mv, p);
    if (mv != 0.0) {
      if (p != k) {
        for (int j = tid; j < n; j += kT) {
          const double t = A[k + size_t(j) * lda];
          A[k + size_t(j) * lda] = A[p + size_t(j) * lda];
          A[p + size_t(j) * lda] = t;
        }
        if (tid == 0) {
          const int t = jb.piv[k];
          jb.piv[k] = jb.piv[p];
          jb.piv[p] = t;
        }
      }
      __syncthreads();
      const double d = A[k + size_t(k) * lda];
      for (int i = k + 1 + tid; i < n; i += kT) A[i + size_t(k) * lda] /= d;
    }
    __syncthreads();
    const int rr = n - k - 1;
    for (int idx = tid; idx < rr * rr; idx += kT) {
      const int i = k + 1 + idx % rr, j = k + 1 + idx / rr;
      A[i + size_t(j) * lda] -= A[i + size_t(k) * lda] * A[k + size_t(j) * lda];
    }
    __syncthreads();
  }
  // explicit inverse X = U^{-1} L^{-1} P by blocked triangular solves
  // (16-row diagonal blocks, rank-16 trailing updates), CTA-wide
  double* X = jb.inv;
  const int n2 = n;
  for (i64 idx = tid; idx < i64(n2) * n2; idx += kT) {
    const int i = int(idx % n2), c = int(idx / n2);
    X[idx] = jb.piv[i] == c ? 1.0 : 0.0;
  }
  __syncthreads();
  constexpr int BS = 16;
  for (int kb = 0; kb < n; kb += BS) {  // L (unit lower)
    const int be = min(kb + BS, n);
    for (int c = tid; c < n; c += kT) {
      double* xc = X + size_t(c) * n;
      for (int i = kb + 1; i < be; ++i) {
        double sacc = xc[i];
        for (int l = kb; l < i; ++l) sacc -= A[i + size_t(l) * lda] * xc[l];
        xc[i] = sacc;
      }
    }
    __syncthreads();
    const int rows = n - be;
    for (i64 idx = tid; idx < i64(rows) * n; idx += kT) {
      const int i = be + int(idx % rows), c = int(idx / rows);
      double* xc = X + size_t(c) * n;
      double sacc = xc[i];
      for (int l = kb; l < be; ++l) sacc -= A[i + size_t(l) * lda] * xc[l];
      xc[i] = sacc;
    }
    __syncthreads();
  }
  for (int kb = ((n - 1) / BS) * BS; kb >= 0; kb -= BS) {  // U
    const int be = min(kb + BS, n);
    for (int c = tid; c < n; c += kT) {
      double* xc = X + size_t(c) * n;
      for (int i = be - 1; i >= kb; --i) {
        double sacc = xc[i];
        for (int l = i + 1; l < be; ++l) sacc -= A[i + size_t(l) * lda] * xc[l];
        xc[i] = sacc / A[i + size_t(i) * lda];
      }
    }
    __syncthreads();
    for (i64 idx = tid; idx < i64(kb) * n; idx += kT) {
      const int i = int(idx % kb), c = int(idx / kb);
      double* xc = X + size_t(c) * n;
      double sacc = xc[i];
      for (int l = kb; l < be; ++l) sacc -= A[i + size_t(l) * lda] * xc[l];
      xc[i] = sacc;
    }
    __syncthreads();
  }
  // reciprocal condition estimate (Eigen ConditionEstimator.h) with the
  // explicit inverse standing in for the LU solves
  if (jb.rcond) {
    const double r = rcond_from_inverse(X, n, l1, jb.work, red, ired);
    if (tid == 0) *jb.rcond = r;
  }
  __syncthreads();
  if (in_smem) {
    for (int c = warp; c < n; c += kWarps)
      for (int i = lane; i < n; i += 32) jb.a[i + size_t(c) * jb.lda] = mat[i + size_t(c) * n];
  }
}


// ---------------------------------------------------------------- Gauss-Jordan inverse (n <= 128)
// Explicit inverse by in-place Gauss-Jordan with partial (row) pivoting and
// the matrix held in REGISTERS: lane l of warp w owns rows l + 32a (a < RA)
// and columns w + 16b (b < CB).  Rows are never moved: row i used as the
// pivot of step k gives inv[k, piv[m]] = M[i, m] at the end.  The pivot of
// step k is the first largest |M[i, k]| over the rows not yet used, which in
// exact arithmetic is the pivot PartialPivLU takes (the unused rows carry
// LU's Schur complement); results agree with lu_kernel to rounding.
// Per step: the owner warp of column k picks the pivot and publishes the
// column; the owners of the pivot row publish it scaled; everyone updates its
// register tile (two CTA barriers per step).
template <int RA, int CB>
__global__ void __launch_bounds__(kT) gj_inverse_kernel(const LuJob* __restrict__ jobs) {
  static_assert(kT == 512, "16 warps x 32 lanes");
  extern __shared__ double sm[];
  const LuJob jb = jobs[blockIdx.x];
  const int n = jb.n;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* X = sm;                            // n x n (final inverse, for rcond)
  double* colb = X + size_t(n) * n;          // 2 x 128: pivot column, double buffered
  double* rowb = colb + 256;                 // 2 x 128: scaled pivot row
  double* red = rowb + 256;                  // 64
  int* ired = reinterpret_cast<int*>(red + 64);  // 64
  int* pivrow = ired + 64;                   // 128: row used at step k
  int* rowstep = pivrow + 128;               // 128: step at which row i pivoted
  __shared__ int sp[2];
  __shared__ double s_l1;
  __shared__ int s_sing;
  if (tid == 0) {
    s_l1 = 0.0;
    s_sing = 0;
  }
  double M[RA][CB];
#pragma unroll
  for (int a = 0; a < RA; ++a)
#pragma unroll
    for (int b = 0; b < CB; ++b) {
      const int i = lane + 32 * a, j = warp + 16 * b;
      M[a][b] = (i < n && j < n) ? jb.a[i + size_t(j) * jb.lda] : 0.0;
    }
  __syncthreads();
  // 1-norm of A (max column sum)
#pragma unroll
  for (int b = 0; b < CB; ++b) {
    double cs = 0.0;
#pragma unroll
    for (int a = 0; a < RA; ++a) cs += fabs(M[a][b]);
    cs = warp_sum(cs);
    if (lane == 0 && warp + 16 * b < n)
      atomicMax(reinterpret_cast<unsigned long long*>(&s_l1), __double_as_longlong(cs));
  }
  unsigned used = 0;  // bit a: row lane + 32 a already pivoted
  // Pivot search of column k by its owner warp (values in registers), which
  // publishes the column for the other warps: the step's only barrier.
  auto search = [&](int k) {
    double* col = colb + 128 * (k & 1);
    const int bk = k >> 4;
    double bv = -1.0;
    int bi = 0x7fffffff;
#pragma unroll
    for (int b = 0; b < CB; ++b)
      if (b == bk) {
#pragma unroll
        for (int a = 0; a < RA; ++a) {
          const int i = lane + 32 * a;
          if (i < n) {
            col[i] = M[a][b];
            const double v = fabs(M[a][b]);
            if (!((used >> a) & 1u) && v > bv) {
              bv = v;
              bi = i;
            }
          }
        }
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      sp[k & 1] = bi;
      pivrow[k] = bi;
      rowstep[bi] = k;
      if (!(bv > 0.0)) s_sing = 1;
    }
  };
  if (warp == 0) search(0);
  for (int k = 0; k < n; ++k) {
    __syncthreads();  // column k and its pivot published
    const double* col = colb + 128 * (k & 1);
    const int p = sp[k & 1];
    const int ap = p >> 5, lp = p & 31;
    const double piv = col[p];
    const double rinv = piv != 0.0 ? 1.0 / piv : 0.0;
    // the pivot row of this warp's columns lives in lane lp: broadcast it
    double pr[CB];
#pragma unroll
    for (int b = 0; b < CB; ++b) {
      double x = 0.0;
#pragma unroll
      for (int a = 0; a < RA; ++a)
        if (a == ap) x = M[a][b];
      pr[b] = __shfl_sync(0xffffffffu, x, lp) * rinv;
    }
    const bool own_k = warp == (k & 15);
    const int bk = k >> 4;
#pragma unroll
    for (int a = 0; a < RA; ++a) {
      const int i = lane + 32 * a;
      if (i >= n) continue;
      if (i == p) {  // the pivot row becomes the scaled row (column k: 1/piv)
        used |= 1u << a;
#pragma unroll
        for (int b = 0; b < CB; ++b) M[a][b] = (own_k && b == bk) ? rinv : pr[b];
        continue;
      }
      const double f = col[i];
#pragma unroll
      for (int b = 0; b < CB; ++b) M[a][b] = (own_k && b == bk) ? -f * rinv : M[a][b] - f * pr[b];
    }
    if (k + 1 < n && warp == ((k + 1) & 15)) search(k + 1);
  }
  // unscramble: inv[k, pivrow[m]] = M[pivrow[k], m]
#pragma unroll
  for (int a = 0; a < RA; ++a)
#pragma unroll
    for (int b = 0; b < CB; ++b) {
      const int i = lane + 32 * a, m = warp + 16 * b;
      if (i < n && m < n) {
        const size_t o = size_t(rowstep[i]) + size_t(pivrow[m]) * n;
        X[o] = M[a][b];
        jb.inv[o] = M[a][b];
      }
    }
  for (int q = tid; q < n; q += kT) jb.piv[q] = pivrow[q];
  __syncthreads();
  if (jb.rcond) {
    const double r = s_sing ? 0.0 : rcond_from_inverse(X, n, s_l1, jb.work, red, ired);
    if (tid == 0) *jb.rcond = r;
  }
}

// Gauss-Jordan for 128 < n <= 160 with the matrix in shared memory (the
// register tile would not fit): same pivoting and unscrambling as above; per
// step one warp picks the pivot, the pivot row and column are staged, every
// thread updates its elements.
__global__ void __launch_bounds__(kT) gj_inverse_smem_kernel(const LuJob* __restrict__ jobs) {
  extern __shared__ double sm[];
  const LuJob jb = jobs[blockIdx.x];
  const int n = jb.n;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* A = sm;                     // n x n, ld n
  double* col = A + size_t(n) * n;    // n
  double* row = col + n;              // n
  double* red = row + n;              // 64
  int* ired = reinterpret_cast<int*>(red + 64);  // 64
  int* pivrow = ired + 64;            // n
  int* rowstep = pivrow + n;          // n
  int* used = rowstep + n;            // n
  __shared__ int s_p, s_sing;
  __shared__ double s_l1;
  // element ownership: row ti of columns tj, tj + cpp, ...
  const int R = (n + 31) / 32 * 32, cpp = kT / R;
  const int ti = tid % R, tj = tid / R;
  if (tid == 0) {
    s_sing = 0;
    s_l1 = 0.0;
  }
  for (int c = warp; c < n; c += kWarps) {
    double cs = 0.0;
    for (int i = lane; i < n; i += 32) {
      const double x = jb.a[i + size_t(c) * jb.lda];
      A[i + size_t(c) * n] = x;
      cs += fabs(x);
    }
    cs = warp_sum(cs);
    if (lane == 0) atomicMax(reinterpret_cast<unsigned long long*>(&s_l1), __double_as_longlong(cs));
  }
  for (int i = tid; i < n; i += kT) used[i] = 0;
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    if (warp == 0) {
      double bv = -1.0;
      int bi = 0x7fffffff;
      for (int i = lane; i < n; i += 32) {
        const double v = fabs(A[i + size_t(k) * n]);
        if (!used[i] && v > bv) {
          bv = v;
          bi = i;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (lane == 0) {
        s_p = bi;
        pivrow[k] = bi;
        rowstep[bi] = k;
        used[bi] = 1;
        if (!(bv > 0.0)) s_sing = 1;
      }
    }
    __syncthreads();
    const int p = s_p;
    const double piv = A[p + size_t(k) * n];
    const double rinv = piv != 0.0 ? 1.0 / piv : 0.0;
    for (int j = tid; j < n; j += kT) {
      const double u = j == k ? rinv : A[p + size_t(j) * n] * rinv;
      row[j] = u;
      A[p + size_t(j) * n] = u;
      col[j] = A[j + size_t(k) * n];
    }
    __syncthreads();
    if (ti < n && tj < cpp && ti != p) {
      const double f = col[ti];
      for (int j = tj; j < n; j += cpp) {
        double* a = A + ti + size_t(j) * n;
        *a = j == k ? -f * rinv : *a - f * row[j];
      }
    }
    __syncthreads();
  }
  if (ti < n && tj < cpp) {
    const size_t o = size_t(rowstep[ti]);
    for (int m = tj; m < n; m += cpp) jb.inv[o + size_t(pivrow[m]) * n] = A[ti + size_t(m) * n];
  }
  for (int q = tid; q < n; q += kT) jb.piv[q] = pivrow[q];
  __syncthreads();
  if (jb.rcond) {
    const double r = s_sing ? 0.0 : rcond_from_inverse(jb.inv, n, s_l1, jb.work, red, ired);
    if (tid == 0) *jb.rcond = r;
  }
}

// ---------------------------------------------------------------- Gauss-Jordan inverse on DMMA accumulators
// Explicit inverse (n <= 32 TA) by BLOCKED in-place Gauss-Jordan with the
// matrix held in registers as m8n8k4 accumulator tiles: 4 x 4 warps, each
// owning TA x TA tiles of 8 x 8 (the matrix is padded with the identity to
// NP = 32 TA).  Steps go in blocks of 4 pivot columns:
//   1. the block's 4 columns are copied out of the tiles (shared memory);
//   2. ONE warp factors that n x 4 panel in its registers, four pivoted
//      Gauss-Jordan steps with no CTA barrier (pivot = first largest
//      |M[i, k]| over the unused rows, found by a warp reduction);
//   3. the 4 pivot rows are copied out of the tiles and brought up to date
//      by one thread per column (a 4-term recurrence in registers);
//   4. everything else is updated by ONE DMMA per tile,  M <- M - U R  with
//      U = the four pivot columns (zero at their own pivot rows) and R = the
//      four scaled pivot rows; pivot rows and the block's columns are then
//      rewritten from their step-by-step values.
// Four CTA barriers per block of four steps.  Same pivot rule, no row
// movement and the same unscrambling as gj_inverse_kernel; results agree
// with it up to the summation order of the four products of a block.
// els.cpp:124-127 (PartialPivLU of W and rcond()).
constexpr int kGjNb = 4;
template <int TA>
constexpr int gj_dmma_ld() { return 32 * TA + 4; }
template <int TA>
size_t gj_dmma_smem(int n) {
  const size_t head = (64 + 32 + 2 * 16 * TA) * sizeof(double);  // red, ired, pivrow/rowstep
  const size_t panels = (7 * kGjNb * size_t(gj_dmma_ld<TA>()) + 32) * sizeof(double);
  return head + std::max(panels, size_t(n) * n * sizeof(double));
}

#ifdef SBX_GJ_PROFILE  // diagnostics: cycles per phase (thread 0), printed at the end
#define GJP_DECL long long gjp_t[8] = {0, 0, 0, 0, 0, 0, 0, 0}, gjp_last = clock64()
#define GJP(i)                          \
  do {                                  \
    const long long now_ = clock64();   \
    gjp_t[i] += now_ - gjp_last;        \
    gjp_last = now_;                    \
  } while (0)
#define GJP_PRINT                                                                                   \
  if (tid == 0)                                                                                     \
  printf("[gj n=%d] load %lld extract %lld panel %lld rows %lld fix %lld dmma %lld out %lld rcond %lld\n", n, \
         gjp_t[0], gjp_t[1], gjp_t[2], gjp_t[3], gjp_t[4], gjp_t[5], gjp_t[6], gjp_t[7])
#else
#define GJP_DECL
#define GJP(i)
#define GJP_PRINT
#endif

constexpr int kGjT = 256;  // 8 warps: 4 row groups x 2 column groups, up to 255 registers per thread
template <int TA>
__global__ void __launch_bounds__(kGjT, 1) gj_inverse_dmma_kernel(const LuJob* __restrict__ jobs) {
  constexpr int NP = 32 * TA, LD = gj_dmma_ld<TA>(), NB = kGjNb, TB = 2 * TA;
  static_assert(NB == 4, "one m8n8k4 per tile and block");
  static_assert(NP <= kGjT, "one thread per column in the row phase");
  extern __shared__ double sm[];
  const LuJob jb = jobs[blockIdx.x];
  const int n = jb.n;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int wr = warp & 3, wc = warp >> 2;
  double* red = sm;                                  // 64
  int* ired = reinterpret_cast<int*>(red + 64);      // 64
  int* pivrow = ired + 64;                           // NP
  int* rowstep = pivrow + NP;                        // NP
  double* body = sm + 64 + 32 + 2 * 16 * TA;
  double* Cm = body;                // 2 x 2 x NB x LD: the block's columns (double buffered across blocks,
                                    // and ping-pong between the steps of a panel)
  double* U = Cm + 4 * NB * LD;     // NB x LD: pivot columns (0 at the step's pivot row)
  double* Rm = U + NB * LD;         // NB x LD: scaled pivot rows; before that the raw rows
  double* Fm = Rm + NB * LD;        // NB x LD: pivot rows as they stand at the end of the block
  double* rblk = Fm + NB * LD;      // NB x NB: the pivot rows inside the block's columns
  double* rinvs = rblk + NB * NB;   // NB
  double* X = body;                 // n x n: the inverse, for rcond (after the last block)
  __shared__ int s_sing;
  __shared__ double s_l1;
  if (tid == 0) {
    s_sing = 0;
    s_l1 = 0.0;
  }
  if (tid < 64) {  // the block reductions of rcond read kWarps slots; the dead warps' stay neutral
    red[tid] = 0.0;
    ired[tid] = 0x7fffffff;
  }
  __syncthreads();
  for (int c = warp; c < n; c += kGjT / 32) {
    double cs = 0.0;
    for (int i = lane; i < n; i += 32) cs += fabs(jb.a[i + size_t(c) * jb.lda]);
    cs = warp_sum(cs);
    if (lane == 0) atomicMax(reinterpret_cast<unsigned long long*>(&s_l1), __double_as_longlong(cs));
  }
  GJP_DECL;
  double acc[TA][TB][2];
#pragma unroll
  for (int a = 0; a < TA; ++a)
#pragma unroll
    for (int b = 0; b < TB; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int row = 8 * (TA * wr + a) + gid, col = 8 * (TB * wc + b) + 2 * tig + e;
        acc[a][b][e] = (row < n && col < n) ? jb.a[row + size_t(col) * jb.lda] : (row == col ? 1.0 : 0.0);
      }
  unsigned usedmask = 0;  // warp 0: bit q set when row lane + 32 q has been a pivot
  GJP(0);
  for (int k0 = 0, blk = 0; k0 < n; k0 += NB, ++blk) {
    const int nb = min(NB, n - k0);
    const int tc0 = k0 >> 3, half = (k0 >> 2) & 1;
    const bool own_cols = wc == tc0 / TB && (tig >> 1) == half;
    const int bsel = tc0 % TB, cloc = (2 * tig) & 3;
    double* Cb = Cm + (blk & 1) * 2 * NB * LD;         // panel input (step 0 reads it)
    double* Cfin = Cb + (nb & 1) * NB * LD;            // where the panel's last step leaves the columns
    if (own_cols) {
#pragma unroll
      for (int a = 0; a < TA; ++a)
#pragma unroll
        for (int b = 0; b < TB; ++b)
          if (b == bsel) {
            const int row = 8 * (TA * wr + a) + gid;
            Cb[cloc * LD + row] = acc[a][b][0];
            Cb[(cloc + 1) * LD + row] = acc[a][b][1];
          }
    }
    __syncthreads();
    GJP(1);
    if (warp == 0) {  // the n x 4 panel in shared memory: lane owns rows lane + 32 q
#pragma unroll
      for (int s = 0; s < NB; ++s) {
        // step s reads one buffer and writes the other (no load waits on a store)
        const double* __restrict__ pin = Cb + (s & 1) * NB * LD;
        double* __restrict__ pout = Cb + ((s + 1) & 1) * NB * LD;
        if (s < nb) {
          double cs[TA];
#pragma unroll
          for (int q = 0; q < TA; ++q) cs[q] = pin[s * LD + lane + 32 * q];
          // pivot: first largest |x| over the unused rows, compared as integers
          // (the bit pattern of |x| is monotone; NaN counts as the largest)
          long long bk = -1;
          int bi = 0x7fffffff;
#pragma unroll
          for (int q = 0; q < TA; ++q) {
            const int i = lane + 32 * q;
            long long key = __double_as_longlong(fabs(cs[q]));
            if (key > 0x7ff0000000000000ll) key = 0x7ff0000000000000ll;
            if (i < n && !((usedmask >> q) & 1u) && key > bk) {
              bk = key;
              bi = i;
            }
          }
          const int hi = int(bk >> 32);
          const unsigned lo = unsigned(bk);
          const int mh = __reduce_max_sync(0xffffffffu, hi);
          const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
          const int p = int(__reduce_min_sync(0xffffffffu, (hi == mh && lo == ml) ? unsigned(bi) : 0x7fffffffu));
          const bool nonzero = mh > 0 || (mh == 0 && ml > 0);
          double r[NB];  // the scaled pivot row inside the block's columns
#pragma unroll
          for (int c = 0; c < NB; ++c) r[c] = pin[c * LD + p];
          const double piv = r[s];
          const double rinv = piv != 0.0 ? 1.0 / piv : 0.0;
#pragma unroll
          for (int c = 0; c < NB; ++c) r[c] = c == s ? rinv : r[c] * rinv;
#pragma unroll
          for (int q = 0; q < TA; ++q) {
            const int i = lane + 32 * q;
            if (i == p) cs[q] = 0.0;  // u: the pivot column, zero at the pivot row
            U[s * LD + i] = cs[q];
          }
#pragma unroll
          for (int c = 0; c < NB; ++c) {
            double x[TA];
#pragma unroll
            for (int q = 0; q < TA; ++q) x[q] = c == s ? 0.0 : pin[c * LD + lane + 32 * q];
#pragma unroll
            for (int q = 0; q < TA; ++q) {
              const int i = lane + 32 * q;
              pout[c * LD + i] = i == p ? r[c] : x[q] - cs[q] * r[c];
            }
          }
          if (lane == (p & 31)) usedmask |= 1u << (p >> 5);
          if (lane == 0) {
            pivrow[k0 + s] = p;
            rowstep[p] = k0 + s;
            rinvs[s] = rinv;
            if (!nonzero) s_sing = 1;
          }
          if (lane < NB) {
            double t = r[0];
#pragma unroll
            for (int c = 1; c < NB; ++c)
              if (lane == c) t = r[c];
            rblk[s * NB + lane] = t;
          }
          __syncwarp();
        } else {
#pragma unroll
          for (int q = 0; q < TA; ++q) U[s * LD + lane + 32 * q] = 0.0;
        }
      }
    }
    __syncthreads();
    GJP(2);
    for (int s = 0; s < nb; ++s) {  // the pivot rows as they stood at the start of the block
      const int ps = pivrow[k0 + s], tr = ps >> 3;
      if (wr == tr / TA && gid == (ps & 7)) {
        const int asel = tr % TA;
#pragma unroll
        for (int a = 0; a < TA; ++a)
          if (a == asel) {
#pragma unroll
            for (int b = 0; b < TB; ++b) {
              const int col = 8 * (TB * wc + b) + 2 * tig;
              Rm[s * LD + col] = acc[a][b][0];
              Rm[s * LD + col + 1] = acc[a][b][1];
            }
          }
      }
    }
    __syncthreads();
    GJP(3);
    if (tid < NP) {  // one thread per column: rows up to date and scaled, then as at the end of the block
      const int j = tid;
      const bool inblk = j >= k0 && j < k0 + NB;
      double r[NB], upp[NB][NB];
      int ps[NB];
#pragma unroll
      for (int s = 0; s < NB; ++s) ps[s] = s < nb ? pivrow[k0 + s] : 0;
#pragma unroll
      for (int s = 0; s < NB; ++s)
#pragma unroll
        for (int t = 0; t < NB; ++t) upp[t][s] = t != s ? U[t * LD + ps[s]] : 0.0;  // U[t][p_s] (0 for t >= nb)
#pragma unroll
      for (int s = 0; s < NB; ++s) {
        r[s] = 0.0;
        if (s < nb) {
          if (inblk) {
            r[s] = rblk[s * NB + (j - k0)];
          } else {
            double v = Rm[s * LD + j];
#pragma unroll
            for (int t = 0; t < s; ++t) v -= upp[t][s] * r[t];
            r[s] = v * rinvs[s];
          }
        }
      }
#pragma unroll
      for (int s = 0; s < NB; ++s) {
        double f = r[s];
#pragma unroll
        for (int t = s + 1; t < NB; ++t) f -= upp[t][s] * r[t];
        Rm[s * LD + j] = r[s];
        Fm[s * LD + j] = f;
      }
    }
    __syncthreads();
    GJP(4);
    {
      double af[TA];
#pragma unroll
      for (int a = 0; a < TA; ++a) af[a] = -U[tig * LD + 8 * (TA * wr + a) + gid];
#pragma unroll
      for (int b = 0; b < TB; ++b) {
        const double bf = Rm[tig * LD + 8 * (TB * wc + b) + gid];
#pragma unroll
        for (int a = 0; a < TA; ++a) dmma(acc[a][b][0], acc[a][b][1], af[a], bf);
      }
    }
    for (int s = 0; s < nb; ++s) {
      const int ps = pivrow[k0 + s], tr = ps >> 3;
      if (wr == tr / TA && gid == (ps & 7)) {
        const int asel = tr % TA;
#pragma unroll
        for (int a = 0; a < TA; ++a)
          if (a == asel) {
#pragma unroll
            for (int b = 0; b < TB; ++b) {
              const int col = 8 * (TB * wc + b) + 2 * tig;
              acc[a][b][0] = Fm[s * LD + col];
              acc[a][b][1] = Fm[s * LD + col + 1];
            }
          }
      }
    }
    if (own_cols) {
#pragma unroll
      for (int a = 0; a < TA; ++a)
#pragma unroll
        for (int b = 0; b < TB; ++b)
          if (b == bsel) {
            const int row = 8 * (TA * wr + a) + gid;
            acc[a][b][0] = Cfin[cloc * LD + row];
            acc[a][b][1] = Cfin[(cloc + 1) * LD + row];
          }
    }
    GJP(5);
    // no barrier: the next block writes the other Cm buffer, and U / Rm / Fm
    // only after its first barrier
  }
  __syncthreads();
  // unscramble into X (shared, over the dead panels), then out
#pragma unroll
  for (int a = 0; a < TA; ++a)
#pragma unroll
    for (int b = 0; b < TB; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int row = 8 * (TA * wr + a) + gid, col = 8 * (TB * wc + b) + 2 * tig + e;
        if (row < n && col < n) X[rowstep[row] + size_t(pivrow[col]) * n] = acc[a][b][e];
      }
  for (int q = tid; q < n; q += kGjT) jb.piv[q] = pivrow[q];
  __syncthreads();
  for (int e = tid; e < n * n; e += kGjT) jb.inv[e] = X[e];
  GJP(6);
  if (jb.rcond) {
    const double r = s_sing ? 0.0 : rcond_from_inverse<kGjT>(X, n, s_l1, jb.work, red, ired);
    if (tid == 0) *jb.rcond = r;
  }
  GJP(7);
  GJP_PRINT;
}

constexpr int kGjSmemMax = 160;
size_t gj_smem_bytes(int n) { return (size_t(n) * n + 2 * size_t(n) + 64 + 32 + 2 * size_t(n)) * sizeof(double); }

constexpr int kGjMax = 128;
size_t gj_smem(int n) { return (size_t(n) * n + 256 + 256 + 64 + 32 + 128) * sizeof(double); }

// ---------------------------------------------------------------- blocked LU (large n)
// Right-looking partial-pivot LU in panels of kLuNb columns: panel
// factorisation by one CTA (smem when it fits, else L2), row swaps, unit
// lower TRSM for the U12 block row and the A22 update as a DMMA GEMM; the
// explicit inverse by blocked forward/backward substitution (diagonal-block
// kernels + DMMA GEMM updates).  Same pivots (first max) and rounding model
// as lu_kernel up to summation order; used for the large dense blocks
// (A_pp up to 2048, Woodbury W, upper HBS levels).
constexpr int kLuNb = 32;
constexpr int kLuBlockedMin = 384;

__global__ void l1norm_kernel(const double* __restrict__ A, int n, int lda, double* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * (blockDim.x >> 5) + warp;
  if (c >= n) return;
  double s = 0.0;
  for (int i = lane; i < n; i += 32) s += fabs(A[i + size_t(c) * lda]);
  s = warp_sum(s);
  if (lane == 0) atomicMax(reinterpret_cast<unsigned long long*>(out), __double_as_longlong(s));
}

__global__ void __launch_bounds__(kT) panel_lu_kernel(double* A, int n, int lda, int j0, int nb, int* ipiv,
                                                      int smem_doubles) {
  extern __shared__ double sm[];
  const int tid = threadIdx.x;
  double* red = sm;
  int* ired = reinterpret_cast<int*>(sm + 32);
  double* P = sm + 64;
  const int m = n - j0;
  const bool in_smem = 64 + size_t(m) * nb <= size_t(smem_doubles);
  double* Pn = in_smem ? P : A + j0 + size_t(j0) * lda;
  const int ld = in_smem ? m : lda;
  if (in_smem) {
    for (int e = tid; e < m * nb; e += kT) {
      const int i = e % m, c = e / m;
      P[e] = A[j0 + i + size_t(j0 + c) * lda];
    }
    __syncthreads();
  }
  for (int c = 0; c < nb; ++c) {
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int i = c + tid; i < m; i += kT) {
      const double v = fabs(Pn[i + size_t(c) * ld]);
      if (v > bv) {
        bv = v;
        bi = i;
      }
    }
    double mv;
    int p;
    block_argmax(bv, bi, red, ired, mv, p);
    if (mv == 0.0) p = c;  // exactly singular column: no swap, no scaling
    if (tid == 0) ipiv[j0 + c] = j0 + p;
    if (p != c)
      for (int q = tid; q < nb; q += kT) {
        const double t = Pn[c + size_t(q) * ld];
        Pn[c + size_t(q) * ld] = Pn[p + size_t(q) * ld];
        Pn[p + size_t(q) * ld] = t;
      }
    __syncthreads();
    if (mv != 0.0) {
      const double d = Pn[c + size_t(c) * ld];
      for (int i = c + 1 + tid; i < m; i += kT) Pn[i + size_t(c) * ld] /= d;
    }
    __syncthreads();
    const int rr = m - c - 1, cc = nb - c - 1;
    for (int e = tid; e < rr * cc; e += kT) {
      const int i = c + 1 + e % rr, q = c + 1 + e / rr;
      Pn[i + size_t(q) * ld] -= Pn[i + size_t(c) * ld] * Pn[c + size_t(q) * ld];
    }
    __syncthreads();
  }
  if (in_smem)
    for (int e = tid; e < m * nb; e += kT) {
      const int i = e % m, c = e / m;
      A[j0 + i + size_t(j0 + c) * lda] = P[e];
    }
}

// The panel's row interchanges applied to the columns outside it.
__global__ void lu_swap_kernel(double* A, int n, int lda, int j0, int nb, const int* __restrict__ ipiv) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= n || (col >= j0 && col < j0 + nb)) return;
  double* a = A + size_t(col) * lda;
  for (int c = 0; c < nb; ++c) {
    const int p = ipiv[j0 + c], r = j0 + c;
    if (p != r) {
      const double t = a[r];
      a[r] = a[p];
      a[p] = t;
    }
  }
}

// B(r0:r0+nb, cols) <- T^{-1} B(r0:r0+nb, cols), T = the nb x nb diagonal
// block of L (unit lower, lower=1) or U (upper, lower=0) at (r0, r0) of A.
__global__ void lu_diag_trsm_kernel(const double* __restrict__ A, int lda, int r0, int nb, double* B, int ldb,
                                    int c0, int ncols, int lower) {
  __shared__ double T[kLuNb * kLuNb];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int i = e % nb, j = e / nb;
    T[e] = A[r0 + i + size_t(r0 + j) * lda];
  }
  __syncthreads();
  const int col = c0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= c0 + ncols) return;
  double* b = B + size_t(col) * ldb + r0;
  double x[kLuNb];
#pragma unroll
  for (int i = 0; i < kLuNb; ++i) x[i] = i < nb ? b[i] : 0.0;
  if (lower) {
#pragma unroll
    for (int i = 0; i < kLuNb; ++i) {
      if (i >= nb) break;
      double acc = x[i];
#pragma unroll
      for (int l = 0; l < kLuNb; ++l)
        if (l < i) acc -= T[i + l * nb] * x[l];
      x[i] = acc;
    }
  } else {
#pragma unroll
    for (int i = kLuNb - 1; i >= 0; --i) {
      if (i >= nb) continue;
      double acc = x[i];
#pragma unroll
      for (int l = 0; l < kLuNb; ++l)
        if (l > i && l < nb) acc -= T[i + l * nb] * x[l];
      x[i] = acc / T[i + i * nb];
    }
  }
#pragma unroll
  for (int i = 0; i < kLuNb; ++i)
    if (i < nb) b[i] = x[i];
}

__global__ void perm_identity_kernel(double* X, int n, const int* __restrict__ perm) {
  const i64 total = i64(n) * n;
  for (i64 e = blockIdx.x * i64(blockDim.x) + threadIdx.x; e < total; e += i64(gridDim.x) * blockDim.x) {
    const int i = int(e % n), c = int(e / n);
    X[e] = perm[i] == c ? 1.0 : 0.0;
  }
}

__global__ void __launch_bounds__(kT) rcond_kernel(const double* __restrict__ X, int n, const double* l1,
                                                   double* work, double* out) {
  __shared__ double red[32];
  __shared__ int ired[64];
  const double r = rcond_from_inverse(X, n, *l1, work, red, ired);
  if (threadIdx.x == 0) *out = r;
}

__global__ void ipiv_to_perm_kernel(const int* __restrict__ ipiv, int n, int* perm) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  for (int i = 0; i < n; ++i) perm[i] = i;
  for (int i = 0; i < n; ++i) {
    const int p = ipiv[i];
    const int t = perm[i];
    perm[i] = perm[p];
    perm[p] = t;
  }
}

__global__ void lu_solve_kernel(const double* __restrict__ lu, int n, int lda,
                                const int* __restrict__ piv, double* B, int ldb, int nrhs,
                                double* scratch) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= nrhs) return;
  double* b = B + size_t(warp) * ldb;
  double x[kMaxRowsPerLane];
#pragma unroll
  for (int q = 0; q < kMaxRowsPerLane; ++q) {
    const int i = lane + 32 * q;
    x[q] = i < n ? b[piv[i]] : 0.0;
  }
  __syncwarp();
  warp_lu_solve(lu, n, lda, x, lane);
#pragma unroll
  for (int q = 0; q < kMaxRowsPerLane; ++q) {
    const int i = lane + 32 * q;
    if (i < n) b[i] = x[q];
  }
}

__global__ void copy2d_kernel(const double* __restrict__ src, i64 lds, double* __restrict__ dst,
                              i64 ldd, i64 rows, i64 cols) {
  const i64 total = rows * cols;
  for (i64 idx = blockIdx.x * i64(blockDim.x) + threadIdx.x; idx < total;
       idx += i64(gridDim.x) * blockDim.x) {
    const i64 r = idx % rows, c = idx / rows;
    dst[r + c * ldd] = src[r + c * lds];
  }
}

__global__ void copy_jobs_kernel(const CopyJob* __restrict__ jobs) {
  const CopyJob jb = jobs[blockIdx.y];
  const i64 total = i64(jb.rows) * jb.cols;
  for (i64 idx = blockIdx.x * i64(blockDim.x) + threadIdx.x; idx < total;
       idx += i64(gridDim.x) * blockDim.x) {
    const int r = int(idx % jb.rows), c = int(idx / jb.rows);
    jb.dst[r + size_t(c) * jb.ldd] = jb.trans ? jb.src[c + size_t(r) * jb.lds] : jb.src[r + size_t(c) * jb.lds];
  }
}

__global__ void scatter_jobs_kernel(const ScatterJob* __restrict__ jobs) {
  const ScatterJob jb = jobs[blockIdx.y];
  const i64 total = i64(jb.rows) * jb.cols;
  for (i64 idx = blockIdx.x * i64(blockDim.x) + threadIdx.x; idx < total;
       idx += i64(gridDim.x) * blockDim.x) {
    const int r = int(idx % jb.rows), c = int(idx / jb.rows);
    const i64 mr = jb.map ? jb.map[r] : r;
    if (jb.gather)
      jb.dst[r + size_t(jb.col_off + c) * jb.ldd] = jb.alpha * jb.src[mr + size_t(c) * jb.lds];
    else
      jb.dst[mr + size_t(jb.col_off + c) * jb.ldd] = jb.alpha * jb.src[r + size_t(c) * jb.lds];
  }
}

__global__ void add_identity_kernel(double* a, i64 lda, i64 n) {
  for (i64 i = blockIdx.x * i64(blockDim.x) + threadIdx.x; i < n; i += i64(gridDim.x) * blockDim.x)
    a[i + i * lda] += 1.0;
}

}  // namespace

namespace {
// Largest TSQR row block that fits next to the n x n factor.
size_t tsqr_smem(int n) { return size_t(cpqr_blocked_head(n) + 2 * kTsqrBm + 8 + n * n) * sizeof(double); }
}  // namespace

size_t qr_smem_need(int M, int n, bool blocked) {
  return (size_t(blocked ? cpqr_blocked_head(n) : 3 * n + 72) + size_t(M) * n) * sizeof(double);
}

int cpqr_blocked_enabled() {
  // the blocked loop reads the trailing matrix once per step instead of
  // three times, but one-CTA CPQR is bound by per-step latency, not shared
  // memory traffic: measured no faster, so it is opt-in (SBX_CPQR_BLOCKED=1)
  static const int on = std::getenv("SBX_CPQR_BLOCKED") ? 1 : 0;
  return on;
}

void qr_batched(const std::vector<QrJob>& jobs, cudaStream_t s) {
  if (jobs.empty()) return;
  static thread_local JobTable<QrJob> tab, ttab, qtab;
  static std::once_flag attr;
  std::call_once(attr, [] {
    SBX_CUDA(cudaFuncSetAttribute(qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(kSmemCap)));
    SBX_CUDA(cudaFuncSetAttribute(tsqr_cpqr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(kSmemCap)));
    SBX_CUDA(cudaFuncSetAttribute(tsqr_quad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(tsqr_quad_smem(kQBm))));
  });
  std::vector<QrJob> plain, tall;
  static const bool no_tsqr = std::getenv("SBX_NO_TSQR") != nullptr;  // diagnostics
  for (const auto& j : jobs) {
    const bool tsqr = !no_tsqr && j.pivot && j.n <= 16 * kTsqrSlots && j.M > j.n && tsqr_smem(j.n) <= kSmemCap &&
                      qr_smem_need(j.M, j.n, true) > kSmemCap;
    (tsqr ? tall : plain).push_back(j);
  }
  static const int phases = [] {  // diagnostics: bit 2 skips the TSQR, bit 3 the CPQR of R0
    const char* e = std::getenv("SBX_TSQR_PHASES");
    return e ? std::atoi(e) : 0;
  }();
  static const bool old_tsqr = std::getenv("SBX_TSQR_WARP") != nullptr;  // diagnostics: warp-layout kernel
  std::vector<QrJob> quad, wide;
  for (const auto& j : tall) (!old_tsqr && j.n <= kQBm ? quad : wide).push_back(j);
  // the three launches (quad TSQR, warp TSQR, one-CTA CPQR) run side by side:
  // all but the first on streams forked from s
  const cudaStream_t s0 = s;
  std::vector<std::unique_ptr<SideStream>> sides;
  int used = 0;
  static const bool no_fork = std::getenv("SBX_QR_NOFORK") != nullptr;  // diagnostics
  // side streams fork from s before the first launch (no launch waits for another)
  const int nlaunch = int(!quad.empty()) + int(!wide.empty()) + int(!plain.empty());
  if (!no_fork)
    for (int q = 1; q < nlaunch; ++q) sides.emplace_back(new SideStream(s0));
  auto next_stream = [&]() -> cudaStream_t {
    const int u = used++;
    return (u == 0 || no_fork) ? s0 : sides[size_t(u - 1)]->get();
  };
  struct Join {
    std::vector<std::unique_ptr<SideStream>>& v;
    cudaStream_t p;
    ~Join() {
      for (auto& x : v) x->join(p);
    }
  } join{sides, s0};
  if (!quad.empty()) {
    s = next_stream();
    int nmax = 0;
    for (const auto& j : quad) nmax = std::max(nmax, j.n);
    const QrJob* d = qtab.upload(quad, s);
    tsqr_quad_kernel<<<unsigned(quad.size()), kQT, tsqr_quad_smem(nmax), s>>>(d, phases);
    SBX_LAUNCHED();
  }
  if (!wide.empty()) {
    s = next_stream();
    int nmax = 0;
    for (const auto& j : wide) nmax = std::max(nmax, j.n);
    const size_t smem = tsqr_smem(nmax);
    const QrJob* d = ttab.upload(wide, s);
    tsqr_cpqr_kernel<<<unsigned(wide.size()), kT, smem, s>>>(d, cpqr_blocked_enabled() | phases);
    SBX_LAUNCHED();
  }
  if (plain.empty()) return;
  // the blocked loop's F table (kCpqrNb doubles per column) must fit next
  // to the norm tables; very wide problems keep the unblocked loop
  int blk = cpqr_blocked_enabled();
  for (const auto& j : plain)
    if (size_t(cpqr_blocked_head(j.n)) * sizeof(double) > kSmemCap) blk = 0;
  size_t need = 0;
  for (const auto& j : plain) {
    const size_t sz = qr_smem_need(j.M, j.n, blk != 0);
    if (sz <= kSmemCap) need = std::max(need, sz);
  }
  size_t base = 0;
  for (const auto& j : plain)
    base = std::max(base, size_t(blk ? cpqr_blocked_head(j.n) : 3 * j.n + 72) * sizeof(double));
  need = std::max(need, base);
  require(base <= kSmemCap, "qr_batched: too many columns for the norm tables");
  s = next_stream();
  const QrJob* d = tab.upload(plain, s);
  qr_kernel<<<unsigned(plain.size()), kT, need, s>>>(d, int(need / sizeof(double)), blk);
  SBX_LAUNCHED();
}

constexpr size_t kBSmemCap = 225 * 1024;
bool bqr_ok(int M, int n) {
  return n >= 1 && n <= kQBm && M > n && M <= kBMaxM && bqr_smem(M, n) <= kBSmemCap;
}

#ifdef SBX_CPQR_PROF
void bqr_prof_dump() {
  long long h[16 * 8];
  SBX_CUDA(cudaMemcpyFromSymbol(h, g_bqr_prof, sizeof(h)));
  for (int p = 0; p < 16; ++p) {
    if (h[p * 8 + 7] == 0) break;
    std::fprintf(stderr, "bqr panel %2d:", p);
    for (int q = 1; q < 8; ++q) std::fprintf(stderr, " %7lld", h[p * 8 + q] - h[p * 8 + q - 1]);
    std::fprintf(stderr, "\n");
  }
}
#endif

void bqr_batched(const std::vector<QrJob>& jobs, cudaStream_t s) {
  if (jobs.empty()) return;
  static std::once_flag attr;
  std::call_once(attr, [] {
    SBX_CUDA(cudaFuncSetAttribute(bqr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kBSmemCap)));
  });
  size_t smem = 0;
  for (const auto& j : jobs) {
    require(bqr_ok(j.M, j.n), "bqr: problem outside the blocked-QR engine's range");
    smem = std::max(smem, bqr_smem(j.M, j.n));
  }
  static thread_local JobTable<QrJob> tab;
  const QrJob* d = tab.upload(jobs, s);
  static const int phases = [] {  // diagnostics: bit 2 skips phase 1, bit 3 the CPQR of R0
    const char* e = std::getenv("SBX_BQR_PHASES");
    return e ? std::atoi(e) : 0;
  }();
  bqr_kernel<<<unsigned(jobs.size()), kBT, smem, s>>>(d, phases);
  SBX_LAUNCHED();
}

void cpqr_coop_batched(const std::vector<QrJob>& jobs, cudaStream_t s) {
  if (jobs.empty()) return;
  int dev = 0, sms = 148;
  SBX_CUDA(cudaGetDevice(&dev));
  SBX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // first pass: CTAs in proportion to work (columns bound the split)
  double W = 0.0;
  for (const auto& j : jobs) W += double(j.M) * double(j.n);
  int maxM = 0;
  for (const auto& j : jobs) maxM = std::max(maxM, j.M);
  const bool vglob = size_t(maxM) * 8 > kSmemCap / 2;  // tall: Householder vector in L2
  auto smem_for = [&](const std::vector<int>& G) {
    size_t mx = 0;
    for (size_t q = 0; q < jobs.size(); ++q) {
      const int nown = (jobs[q].n + G[q] - 1) / G[q];
      mx = std::max(mx, size_t((vglob ? 0 : jobs[q].M) + 2 * nown + 40) * 8 + size_t(96 + nown) * 4 + 64);
    }
    return mx;
  };
  static std::once_flag attr;
  std::call_once(attr, [] {
    SBX_CUDA(cudaFuncSetAttribute(cpqr_coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(kSmemCap)));
  });
  std::vector<int> G(jobs.size(), 1);
  auto split = [&](int T) {
    int used = 0;
    for (size_t q = 0; q < jobs.size(); ++q) {
      const double w = double(jobs[q].M) * double(jobs[q].n) / W;
      G[q] = std::max(1, std::min(jobs[q].n, int(std::floor(w * (T - int(jobs.size())))) + 1));
      used += G[q];
    }
    return used;
  };
  int per_sm = 1;
  require(int(jobs.size()) <= sms, "cpqr_coop: too many concurrent problems for one cooperative launch");
  split(sms);
  for (int iter = 0; iter < 2; ++iter) {
    const size_t smem = smem_for(G);
    require(smem <= kSmemCap, "cpqr_coop: problem too tall for the shared-memory Householder vector");
    SBX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cpqr_coop_kernel, kCT, smem));
    per_sm = std::max(1, std::min(per_sm, 4));
    const int used = split(sms * per_sm);
    if (used > sms * per_sm || smem_for(G) > smem) split(sms);  // stay co-resident
  }
  if (const char* cap = std::getenv("SBX_COOP_MAXG")) {  // debugging aid
    for (auto& g : G) g = std::max(1, std::min(g, std::atoi(cap)));
  }
  const size_t smem = smem_for(G);
  require(smem <= kSmemCap, "cpqr_coop: problem too tall for the shared-memory Householder vector");
  std::vector<int> cta_job, cta_rank, part_off(jobs.size());
  std::vector<i64> beta_off(jobs.size());
  i64 boff = 0;
  int poff = 0;
  for (size_t q = 0; q < jobs.size(); ++q) {
    part_off[q] = poff;
    poff += 2 * G[q];
    beta_off[q] = boff;
    boff += std::min(jobs[q].M, jobs[q].n);
    for (int r = 0; r < G[q]; ++r) {
      cta_job.push_back(int(q));
      cta_rank.push_back(r);
    }
  }
  static thread_local JobTable<QrJob> tjobs;
  static thread_local DevBuf<int> d_ints;
  static thread_local DevBuf<CoopCtl> d_ctl;
  static thread_local DevBuf<CoopPart> d_parts;
  static thread_local DevBuf<double> d_beta;
  static thread_local DevBuf<i64> d_boff;
  std::vector<int> ints;
  ints.insert(ints.end(), cta_job.begin(), cta_job.end());
  ints.insert(ints.end(), cta_rank.begin(), cta_rank.end());
  ints.insert(ints.end(), G.begin(), G.end());
  ints.insert(ints.end(), part_off.begin(), part_off.end());
  d_ints.upload(ints, s);
  d_ctl.reserve(jobs.size());
  SBX_CUDA(cudaMemsetAsync(d_ctl.get(), 0, jobs.size() * sizeof(CoopCtl), s));
  d_parts.reserve(size_t(poff));
  d_beta.reserve(size_t(std::max<i64>(boff, 1)));
  d_boff.upload(beta_off, s);
  CoopArgs a;
  a.jobs = tjobs.upload(jobs, s);
  a.cta_job = d_ints.get();
  a.cta_rank = d_ints.get() + cta_job.size();
  a.job_ctas = d_ints.get() + 2 * cta_job.size();
  a.part_off = d_ints.get() + 2 * cta_job.size() + G.size();
  a.ctl = d_ctl.get();
  a.parts = d_parts.get();
  a.beta = d_beta.get();
  a.beta_off = d_boff.get();
  static thread_local DevBuf<double> d_v;
  a.vglob = nullptr;
  a.vstride = 0;
  if (vglob) {
    a.vstride = (i64(maxM) + 31) / 32 * 32;
    d_v.reserve(size_t(a.vstride) * cta_job.size());
    a.vglob = d_v.get();
  }
  void* params[] = {&a};
  SBX_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(cpqr_coop_kernel),
                                       dim3(unsigned(cta_job.size())), dim3(kCT), params, smem, s));
  SBX_LAUNCHED();
}

int cpqr_smem_ctas(int M, int n) {
  if (M <= 0 || n <= 0) return 0;
  const size_t cap = kSmemCap / sizeof(double);
  if (smem_coop_doubles(M, 1) > cap) return 0;
  int lo = 1, hi = n;  // smallest G whose widest slab fits
  while (lo < hi) {
    const int g = (lo + hi) / 2;
    if (smem_coop_doubles(M, (n + g - 1) / g) <= cap) hi = g;
    else lo = g + 1;
  }
  return lo;
}

void cpqr_smem_batched(const std::vector<QrJob>& jobs, cudaStream_t s) {
  if (jobs.empty()) return;
  int dev = 0, sms = 148;
  SBX_CUDA(cudaGetDevice(&dev));
  SBX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  static std::once_flag attr;
  std::call_once(attr, [] {
    SBX_CUDA(cudaFuncSetAttribute(cpqr_onchip_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(kSmemCap)));
  });
  static thread_local JobTable<QrJob> tjobs;
  static thread_local DevBuf<int> d_ints;
  static thread_local DevBuf<CoopCtl> d_ctl;
  static thread_local DevBuf<CoopPart> d_parts;
  static thread_local DevBuf<double> d_beta, d_cand;
  static thread_local DevBuf<i64> d_offs;
  // waves: every CTA of a cooperative launch must be co-resident
  size_t first = 0;
  while (first < jobs.size()) {
    std::vector<QrJob> wave;
    std::vector<int> G;
    size_t smem = 0;
    int ctas = 0, per_sm = 1;
    size_t q = first;
    for (; q < jobs.size(); ++q) {
      const int g = cpqr_smem_ctas(jobs[q].M, jobs[q].n);
      require(g > 0 && g <= sms, "cpqr_smem: problem does not fit on chip");
      const size_t sm2 = std::max(smem, smem_coop_doubles(jobs[q].M, (jobs[q].n + g - 1) / g) * sizeof(double));
      int ps = 1;
      SBX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, cpqr_onchip_kernel<false>, kOT, sm2));
      ps = std::max(1, ps);
      if (!wave.empty() && ctas + g > sms * ps) break;
      wave.push_back(jobs[q]);
      G.push_back(g);
      ctas += g;
      smem = sm2;
      per_sm = ps;
    }
    (void)per_sm;
    first = q;
    std::vector<int> cta_job, cta_rank, part_off(wave.size());
    std::vector<i64> offs(2 * wave.size());
    i64 boff = 0, coff = 0;
    int poff = 0;
    for (size_t w = 0; w < wave.size(); ++w) {
      part_off[w] = poff;
      poff += 2 * G[w];
      offs[w] = boff;
      boff += std::min(wave[w].M, wave[w].n);
      offs[wave.size() + w] = coff;
      coff += 2 * i64(G[w]) * wave[w].M;
      for (int r = 0; r < G[w]; ++r) {
        cta_job.push_back(int(w));
        cta_rank.push_back(r);
      }
    }
    std::vector<int> ints;
    ints.insert(ints.end(), cta_job.begin(), cta_job.end());
    ints.insert(ints.end(), cta_rank.begin(), cta_rank.end());
    ints.insert(ints.end(), G.begin(), G.end());
    ints.insert(ints.end(), part_off.begin(), part_off.end());
    d_ints.upload(ints, s);
    d_ctl.reserve(wave.size());
    SBX_CUDA(cudaMemsetAsync(d_ctl.get(), 0, wave.size() * sizeof(CoopCtl), s));
    d_parts.reserve(size_t(poff));
    d_beta.reserve(size_t(std::max<i64>(boff, 1)));
    d_cand.reserve(size_t(std::max<i64>(coff, 1)));
    d_offs.upload(offs, s);
    SmemCoopArgs a;
    a.jobs = tjobs.upload(wave, s);
    a.cta_job = d_ints.get();
    a.cta_rank = d_ints.get() + cta_job.size();
    a.job_ctas = d_ints.get() + 2 * cta_job.size();
    a.part_off = d_ints.get() + 2 * cta_job.size() + G.size();
    a.ctl = d_ctl.get();
    a.parts = d_parts.get();
    a.cand = d_cand.get();
    a.cand_off = d_offs.get() + wave.size();
    a.beta = d_beta.get();
    a.beta_off = d_offs.get();
    void* params[] = {&a};
    static const bool plain = std::getenv("SBX_COOP_PLAIN") != nullptr;  // diagnostics
    if (plain)
      SBX_CUDA(cudaLaunchKernel(reinterpret_cast<void*>(cpqr_onchip_kernel<false>), dim3(unsigned(cta_job.size())),
                                dim3(kOT), params, smem, s));
    else
      SBX_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(cpqr_onchip_kernel<false>),
                                           dim3(unsigned(cta_job.size())), dim3(kOT), params, smem, s));
    SBX_LAUNCHED();
  }
}

int cpqr_cluster_size(int M, int n) {
  const int g = cpqr_smem_ctas(M, n);
  if (g <= 0 || g > 16) return 0;
  int c = 1;
  while (c < g) c <<= 1;
  return c;
}

#ifdef SBX_CPQR_PROF
void cpqr_prof_dump() {
  long long h[64 * 8];
  SBX_CUDA(cudaMemcpyFromSymbol(h, g_cpqr_prof, sizeof(h)));
  for (int j = 0; j < 64; ++j) {
    if (h[j * 8 + 5] == 0) break;
    std::fprintf(stderr, "step %2d: (rel. to slot 0)", j);
    for (int q = 1; q < 8; ++q) std::fprintf(stderr, " %8lld", h[j * 8 + q] ? h[j * 8 + q] - h[j * 8] : 0LL);
    std::fprintf(stderr, "  | next %lld\n", j < 63 && h[j * 8 + 8] ? h[j * 8 + 8] - h[j * 8] : 0LL);
  }
}
#endif

void cpqr_cluster_batched(const std::vector<QrJob>& all, cudaStream_t s) {
  if (all.empty()) return;
  // one launch per cluster size: a batch mixing sizes would otherwise give
  // every problem the largest cluster (and the fewest co-resident clusters)
  std::vector<QrJob> jobs;
  std::vector<int> csz;
  {
    std::vector<std::pair<int, size_t>> order;
    for (size_t q = 0; q < all.size(); ++q) {
      const int c = cpqr_cluster_size(all[q].M, all[q].n);
      require(c > 0, "cpqr_cluster: problem does not fit one cluster");
      order.push_back({c, q});
    }
    std::stable_sort(order.begin(), order.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
    for (const auto& o : order) {
      jobs.push_back(all[o.second]);
      csz.push_back(o.first);
    }
  }
  i64 boff = 0;
  std::vector<i64> offs;
  for (const auto& j : jobs) {
    offs.push_back(boff);
    boff += std::min(j.M, j.n);
  }
  static std::once_flag attr;
  std::call_once(attr, [] {
    SBX_CUDA(cudaFuncSetAttribute(cpqr_onchip_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(kSmemCap)));
    SBX_CUDA(cudaFuncSetAttribute(cpqr_onchip_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  });
  static thread_local JobTable<QrJob> tjobs;
  static thread_local DevBuf<double> d_beta;
  static thread_local DevBuf<i64> d_offs;
  d_beta.reserve(size_t(std::max<i64>(boff, 1)));
  d_offs.upload(offs, s);
  const QrJob* dj = tjobs.upload(jobs, s);
  for (size_t g0 = 0; g0 < jobs.size();) {
    const int C = csz[g0];
    size_t g1 = g0;
    size_t smem = 0;
    while (g1 < jobs.size() && csz[g1] == C) {
      smem = std::max(smem, smem_coop_doubles(jobs[g1].M, (jobs[g1].n + C - 1) / C) * sizeof(double));
      ++g1;
    }
    SmemCoopArgs a{};
    a.jobs = dj + g0;
    a.beta = d_beta.get();
    a.beta_off = d_offs.get() + g0;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned((g1 - g0) * size_t(C)));
    cfg.blockDim = dim3(kOT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = unsigned(C);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    SBX_CUDA(cudaLaunchKernelEx(&cfg, cpqr_onchip_kernel<true>, a));
    SBX_LAUNCHED();
    g0 = g1;
  }
}

namespace {
struct RegCfg {
  int rpl, cpw;
};
constexpr RegCfg kRegCfgs[] = {{9, 4}, {17, 2}, {20, 2}, {27, 1}, {34, 1}};
constexpr int kRegCfgN = int(sizeof(kRegCfgs) / sizeof(kRegCfgs[0]));

template <int RPL, int CPW>
void launch_reg(const QrJob* d, int np, int G, int size_max, cudaStream_t s) {
  static std::once_flag attr;
  std::call_once(attr, [] {
    SBX_CUDA(cudaFuncSetAttribute(cpqr_reg_kernel<RPL, CPW>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    SBX_CUDA(cudaFuncSetAttribute(cpqr_reg_kernel<RPL, CPW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int((3 * 32 * 34 + 2048) * sizeof(double))));
  });
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(np * G));
  cfg.blockDim = dim3(kOT);
  cfg.dynamicSmemBytes = (size_t(3 * 32 * RPL) + size_t(size_max)) * sizeof(double);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = unsigned(G);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  SBX_CUDA(cudaLaunchKernelEx(&cfg, cpqr_reg_kernel<RPL, CPW>, d));
  SBX_LAUNCHED();
}
}  // namespace

namespace {
constexpr int kStreamRpl[] = {9, 17, 20, 27, 34};
size_t stream_fixed_doubles(int M, int n, int rpl) {
  return size_t(32 * rpl) + 3 * size_t(n) + size_t(std::min(M, n)) + size_t(n) + 1;
}
template <int RPL>
void launch_stream(const QrJob* d, int np, int ns_cap, size_t smem, cudaStream_t s) {
  static std::once_flag attr;
  std::call_once(attr, [] {
    SBX_CUDA(cudaFuncSetAttribute(cpqr_stream_kernel<RPL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(kSmemCap)));
  });
  cpqr_stream_kernel<RPL><<<unsigned(np), kOT, smem, s>>>(d, ns_cap);
  SBX_LAUNCHED();
}
}  // namespace

bool cpqr_stream_ok(int M, int n) {
  if (M <= 0 || n <= 0 || M > 32 * 34) return false;
  int rpl = 0;
  for (int r : kStreamRpl)
    if (32 * r >= M) {
      rpl = r;
      break;
    }
  return stream_fixed_doubles(M, n, rpl) * sizeof(double) + size_t(M) * sizeof(double) <= kSmemCap;
}

void cpqr_stream_batched(const std::vector<QrJob>& all, cudaStream_t s) {
  if (all.empty()) return;
  // one launch per register layout; the resident slab takes what the
  // fixed tables leave of the shared memory
  std::vector<QrJob> cls[5];
  for (const auto& j : all) {
    require(cpqr_stream_ok(j.M, j.n), "cpqr_stream: problem does not fit the streaming engine");
    int c = 0;
    while (32 * kStreamRpl[c] < j.M) ++c;
    cls[c].push_back(j);
  }
  static thread_local JobTable<QrJob> tj[5];
  for (int c = 0; c < 5; ++c) {
    if (cls[c].empty()) continue;
    size_t fixed = 0;
    int Mmax = 1;
    for (const auto& j : cls[c]) {
      fixed = std::max(fixed, stream_fixed_doubles(j.M, j.n, kStreamRpl[c]));
      Mmax = std::max(Mmax, j.M);
    }
    const size_t cap = kSmemCap / sizeof(double);
    const int ns_cap = int((cap - fixed) / size_t(Mmax));
    const size_t smem = kSmemCap;
    const QrJob* d = tj[c].upload(cls[c], s);
    const int np = int(cls[c].size());
    switch (c) {
      case 0: launch_stream<9>(d, np, ns_cap, smem, s); break;
      case 1: launch_stream<17>(d, np, ns_cap, smem, s); break;
      case 2: launch_stream<20>(d, np, ns_cap, smem, s); break;
      case 3: launch_stream<27>(d, np, ns_cap, smem, s); break;
      default: launch_stream<34>(d, np, ns_cap, smem, s); break;
    }
  }
}

int cpqr_reg_config(int M, int n, int* G) {
  if (M <= 0 || n <= 0) return -1;
  for (int c = 0; c < kRegCfgN; ++c) {
    if (32 * kRegCfgs[c].rpl < M) continue;
    const int g = (n + 16 * kRegCfgs[c].cpw - 1) / (16 * kRegCfgs[c].cpw);
    if (g > 16 || std::min(M, n) > 2048) return -1;
    if (G) *G = g;
    return c;
  }
  return -1;
}

void cpqr_reg_batched(const std::vector<QrJob>& all, cudaStream_t s) {
  if (all.empty()) return;
  // one launch per (register layout, cluster size)
  std::vector<std::pair<int, size_t>> order;
  for (size_t q = 0; q < all.size(); ++q) {
    int G = 0;
    const int c = cpqr_reg_config(all[q].M, all[q].n, &G);
    require(c >= 0, "cpqr_reg: problem does not fit the register engine");
    order.push_back({c * 64 + G, q});
  }
  std::stable_sort(order.begin(), order.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
  std::vector<QrJob> jobs;
  for (const auto& o : order) jobs.push_back(all[o.second]);
  static thread_local JobTable<QrJob> tjobs;
  const QrJob* dj = tjobs.upload(jobs, s);
  // the launches (one per layout / cluster size) run side by side: all but
  // the first on streams forked from s
  static const bool no_fork = std::getenv("SBX_REG_NOFORK") != nullptr;  // diagnostics
  std::vector<std::unique_ptr<SideStream>> sides;
  {  // side streams fork from s before the first launch
    int nl = 0;
    for (size_t q = 0; q < order.size(); ++q) nl += (q == 0 || order[q].first != order[q - 1].first) ? 1 : 0;
    if (!no_fork)
      for (int q = 1; q < nl; ++q) sides.emplace_back(new SideStream(s));
  }
  size_t used = 0;
  for (size_t g0 = 0; g0 < jobs.size();) {
    const int key = order[g0].first;
    size_t g1 = g0;
    int size_max = 1;
    while (g1 < jobs.size() && order[g1].first == key) {
      size_max = std::max(size_max, std::min(jobs[g1].M, jobs[g1].n));
      ++g1;
    }
    const int c = key / 64, G = key % 64, np = int(g1 - g0);
    cudaStream_t st = (g0 > 0 && !no_fork) ? sides[used++]->get() : s;
    switch (c) {
      case 0: launch_reg<9, 4>(dj + g0, np, G, size_max, st); break;
      case 1: launch_reg<17, 2>(dj + g0, np, G, size_max, st); break;
      case 2: launch_reg<20, 2>(dj + g0, np, G, size_max, st); break;
      case 3: launch_reg<27, 1>(dj + g0, np, G, size_max, st); break;
      default: launch_reg<34, 1>(dj + g0, np, G, size_max, st); break;
    }
    g0 = g1;
  }
  for (auto& sd : sides) sd->join(s);
}

void interp_batched(const std::vector<InterpJob>& all, cudaStream_t s) {
  if (all.empty()) return;
  static thread_local JobTable<InterpJob> tab, wtab[3];
  static thread_local JobTable<int2> itab, witab[3];
  // register-resident warp kernel by rank class; very high ranks keep the
  // thread-per-column kernel
  std::vector<InterpJob> cls[3], rest;
  for (const auto& j : all) {
    if (j.k <= 64)
      cls[0].push_back(j);
    else if (j.k <= 128)
      cls[1].push_back(j);
    else if (j.k <= 256)
      cls[2].push_back(j);
    else
      rest.push_back(j);
  }
  for (int c = 0; c < 3; ++c) {
    if (cls[c].empty()) continue;
    std::vector<int2> items;
    for (size_t q = 0; q < cls[c].size(); ++q) {
      items.push_back(make_int2(int(q), -1));
      for (int col = 0; col < cls[c][q].n - cls[c][q].k; col += kIWarps) items.push_back(make_int2(int(q), col));
    }
    const InterpJob* d = wtab[c].upload(cls[c], s);
    const int2* di = witab[c].upload(items, s);
    const unsigned g = unsigned(items.size());
    if (c == 0)
      interp_warp_kernel<2><<<g, kIWarps * 32, 0, s>>>(d, di);
    else if (c == 1)
      interp_warp_kernel<4><<<g, kIWarps * 32, 0, s>>>(d, di);
    else
      interp_warp_kernel<8><<<g, kIWarps * 32, 0, s>>>(d, di);
    SBX_LAUNCHED();
  }
  if (rest.empty()) return;
  std::vector<int2> items;
  for (size_t q = 0; q < rest.size(); ++q) {
    items.push_back(make_int2(int(q), -1));
    for (int c = 0; c < rest[q].n - rest[q].k; c += kIT) items.push_back(make_int2(int(q), c));
  }
  const InterpJob* d = tab.upload(rest, s);
  const int2* di = itab.upload(items, s);
  interp_kernel<<<unsigned(items.size()), kIT, 0, s>>>(d, di);
  SBX_LAUNCHED();
}

void gemm_batched(const std::vector<GemmJob>& jobs, cudaStream_t s) {
  if (jobs.empty()) return;
  static thread_local JobTable<GemmJob> tab;
  static thread_local JobTable<int4> ttab;
  static thread_local DevBuf<double> parts;
  std::vector<GemmJob> js = jobs;
  // one small output block over a long inner dimension: the thin-product kernel
  static const bool no_thin = std::getenv("SBX_NO_THIN_GEMM") != nullptr;  // diagnostics
  if (!no_thin && js.size() == 1) {
    GemmJob& j = js[0];
    const bool aligned = (reinterpret_cast<uintptr_t>(j.A) % 16 == 0) && j.lda % 2 == 0 &&
                         (reinterpret_cast<uintptr_t>(j.B) % 16 == 0) && j.ldb % 2 == 0;
    if (!j.ta && !j.tb && j.m > 64 && j.n >= 32 && j.m <= kThinMP && j.n <= kThinMP && j.k >= 8192 && aligned) {
      int sms = 148;
      {
        int dev = 0;
        SBX_CUDA(cudaGetDevice(&dev));
        SBX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      }
      j.kchunk = ((j.k + sms - 1) / sms + kThinKC - 1) / kThinKC * kThinKC;
      j.splitk = std::max(2, (j.k + j.kchunk - 1) / j.kchunk);  // k >= 8192: always several ranges
      parts.reserve(size_t(j.splitk) * j.m * j.n);
      j.part = parts.get();
      const GemmJob* d = tab.upload(js, s);
      static std::once_flag tattr;
      std::call_once(tattr, [] {
        SBX_CUDA(cudaFuncSetAttribute(thin_gemm_kernel<2, 10>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(sizeof(ThinSmem))));
        SBX_CUDA(cudaFuncSetAttribute(thin_gemm_kernel<4, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(sizeof(ThinSmem))));
        SBX_CUDA(cudaFuncSetAttribute(thin_gemm_kernel<4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(sizeof(ThinSmem))));
      });
      static const int thin_wc = [] {  // diagnostics: SBX_THIN_WC=2 selects the 8-warp variant
        const char* e = std::getenv("SBX_THIN_WC");
        return e && std::atoi(e) == 2 ? 2 : 4;
      }();
      KernelTimer kt("thin_gemm", s);
      void* args[] = {(void*)&d};
      const bool narrow = j.n <= 64;
      const void* fn = narrow         ? reinterpret_cast<const void*>(&thin_gemm_kernel<4, 2>)
                       : thin_wc == 2 ? reinterpret_cast<const void*>(&thin_gemm_kernel<2, 10>)
                                      : reinterpret_cast<const void*>(&thin_gemm_kernel<4, 5>);
      SBX_CUDA(cudaLaunchCooperativeKernel(fn, dim3(unsigned(j.splitk)), dim3(!narrow && thin_wc == 2 ? 256 : 512),
                                           args, sizeof(ThinSmem), s));
      SBX_LAUNCHED();
      return;
    }
  }
  // split K when a product has few output tiles but a long inner dimension
  i64 out_tiles = 0;
  for (const auto& j : js) out_tiles += i64((j.m + gTM - 1) / gTM) * ((j.n + gTN - 1) / gTN);
  i64 ptot = 0;
  std::vector<i64> poff(js.size(), 0);
  for (size_t q = 0; q < js.size(); ++q) {
    auto& j = js[q];
    const i64 t = i64((j.m + gTM - 1) / gTM) * ((j.n + gTN - 1) / gTN);
    j.splitk = 1;
    if (j.k >= 2048 && out_tiles < 2 * 148) {
      const int want = int(std::min<i64>((2 * 148 + t - 1) / std::max<i64>(t, 1), j.k / 512));
      if (want > 1) {
        j.kchunk = ((j.k + want - 1) / want + gKC - 1) / gKC * gKC;
        j.splitk = (j.k + j.kchunk - 1) / j.kchunk;
      }
    }
    if (j.splitk > 1) {
      poff[q] = ptot;
      ptot += i64(j.splitk) * j.m * j.n;
    }
  }
  if (ptot > 0) {
    parts.reserve(size_t(ptot));
    for (size_t q = 0; q < js.size(); ++q)
      if (js[q].splitk > 1) js[q].part = parts.get() + poff[q];
  }
  std::vector<int4> tiles;
  i64 mx_out = 0;
  for (size_t j = 0; j < js.size(); ++j) {
    for (int w = 0; w < js[j].splitk; ++w)
      for (int r = 0; r < js[j].m; r += gTM)
        for (int c = 0; c < js[j].n; c += gTN) tiles.push_back(make_int4(int(j), r, c, w));
    if (js[j].splitk > 1) mx_out = std::max<i64>(mx_out, i64(js[j].m) * js[j].n);
  }
  if (tiles.empty()) return;
  const GemmJob* d = tab.upload(js, s);
  const int4* dt = ttab.upload(tiles, s);
  static std::once_flag attr;
  std::call_once(attr, [] {
    SBX_CUDA(cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(GemmSmem))));
  });
  gemm_kernel<<<unsigned(tiles.size()), 256, sizeof(GemmSmem), s>>>(d, dt);
  SBX_LAUNCHED();
  if (mx_out > 0) {
    dim3 grid(unsigned(std::min<i64>((mx_out + 255) / 256, 256)), unsigned(js.size()));
    splitk_reduce_kernel<<<grid, 256, 0, s>>>(d);
    SBX_LAUNCHED();
  }
}


namespace {
void lu_blocked(const LuJob& j, cudaStream_t s) {
  const int n = j.n, lda = j.lda;
  static thread_local DevBuf<int> d_ipiv;
  static thread_local DevBuf<double> d_l1;
  d_ipiv.reserve(size_t(n));
  d_l1.reserve(1);
  static std::once_flag attr;
  std::call_once(attr, [] {
    SBX_CUDA(cudaFuncSetAttribute(panel_lu_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(kSmemCap)));
  });
  if (j.rcond) {
    SBX_CUDA(cudaMemsetAsync(d_l1.get(), 0, sizeof(double), s));
    l1norm_kernel<<<unsigned((n + 7) / 8), 256, 0, s>>>(j.a, n, lda, d_l1.get());
    SBX_LAUNCHED();
  }
  for (int j0 = 0; j0 < n; j0 += kLuNb) {
    const int nb = std::min(kLuNb, n - j0);
    const size_t need = std::min(kSmemCap, (64 + size_t(n - j0) * nb) * sizeof(double));
    panel_lu_kernel<<<1, kT, need, s>>>(j.a, n, lda, j0, nb, d_ipiv.get(), int(need / sizeof(double)));
    SBX_LAUNCHED();
    lu_swap_kernel<<<unsigned((n + 127) / 128), 128, 0, s>>>(j.a, n, lda, j0, nb, d_ipiv.get());
    SBX_LAUNCHED();
    const int rest = n - j0 - nb;
    if (rest > 0) {
      lu_diag_trsm_kernel<<<unsigned((rest + 127) / 128), 128, 0, s>>>(j.a, lda, j0, nb, j.a, lda, j0 + nb,
                                                                      rest, 1);
      SBX_LAUNCHED();
      gemm_batched({{j.a + (j0 + nb) + size_t(j0) * lda, j.a + j0 + size_t(j0 + nb) * lda,
                     j.a + (j0 + nb) + size_t(j0 + nb) * lda, rest, rest, nb, lda, lda, lda, 0, 0, -1.0, 1.0}},
                   s);
    }
  }
  ipiv_to_perm_kernel<<<1, 1, 0, s>>>(d_ipiv.get(), n, j.piv);
  SBX_LAUNCHED();
  // X = U^{-1} L^{-1} P
  double* X = j.inv;
  perm_identity_kernel<<<unsigned(std::min<i64>((i64(n) * n + 255) / 256, 148 * 16)), 256, 0, s>>>(X, n, j.piv);
  SBX_LAUNCHED();
  const unsigned cg = unsigned((n + 127) / 128);
  for (int r0 = 0; r0 < n; r0 += kLuNb) {
    const int nb = std::min(kLuNb, n - r0);
    lu_diag_trsm_kernel<<<cg, 128, 0, s>>>(j.a, lda, r0, nb, X, n, 0, n, 1);
    SBX_LAUNCHED();
    const int below = n - r0 - nb;
    if (below > 0)
      gemm_batched({{j.a + (r0 + nb) + size_t(r0) * lda, X + r0, X + r0 + nb, below, n, nb, lda, n, n, 0, 0,
                     -1.0, 1.0}},
                   s);
  }
  for (int r0 = ((n - 1) / kLuNb) * kLuNb; r0 >= 0; r0 -= kLuNb) {
    const int nb = std::min(kLuNb, n - r0);
    lu_diag_trsm_kernel<<<cg, 128, 0, s>>>(j.a, lda, r0, nb, X, n, 0, n, 0);
    SBX_LAUNCHED();
    if (r0 > 0)
      gemm_batched({{j.a + size_t(r0) * lda, X + r0, X, r0, n, nb, lda, n, n, 0, 0, -1.0, 1.0}}, s);
  }
  if (j.rcond) {
    rcond_kernel<<<1, kT, 0, s>>>(X, n, d_l1.get(), j.work, j.rcond);
    SBX_LAUNCHED();
  }
}
}  // namespace

void lu_batched(const std::vector<LuJob>& all, cudaStream_t s) {
  if (all.empty()) return;
  static const bool log = std::getenv("SBX_LU_LOG") != nullptr;  // diagnostics
  if (log) {
    std::string line;
    for (const auto& j : all) line += " " + std::to_string(j.n);
    std::fprintf(stderr, "[sbx-lu]%s\n", line.c_str());
  }
  // large blocks (few per batch) go through the blocked multi-kernel path
  std::vector<LuJob> jobs, big;
  for (const auto& j : all) (j.n >= kLuBlockedMin ? big : jobs).push_back(j);
  if (big.size() > 16) {
    jobs = all;
    big.clear();
  }
  for (const auto& j : big) {
    require(j.inv != nullptr, "lu_batched: the explicit inverse output is required");
    require(!j.rcond || j.work != nullptr, "lu_batched: rcond needs 4n scratch");
    lu_blocked(j, s);
  }
  if (jobs.empty()) return;
  static const bool no_gj = std::getenv("SBX_NO_GJ") != nullptr;  // diagnostics
  if (!no_gj) {
    std::vector<LuJob> gj[3], rest;
    for (const auto& j : jobs) (j.n <= 32 ? gj[0] : j.n <= 64 ? gj[1] : j.n <= kGjMax ? gj[2] : rest).push_back(j);
    // 64 < n <= 128 on the DMMA-tile kernel too (4 x 8 tiles per warp): 133 us at n = 96, 170 us at
    // n = 128 against 207 / 302 us of the register kernel below (SBX_GJ_DMMA128=0 restores it)
    static const bool dmma128 = [] {
      const char* e = std::getenv("SBX_GJ_DMMA128");
      return !e || std::atoi(e) != 0;
    }();
    if (dmma128 && !gj[2].empty()) {
      int nmax = 1;
      for (const auto& j : gj[2]) {
        require(j.inv != nullptr, "lu_batched: the explicit inverse output is required");
        require(!j.rcond || j.work != nullptr, "lu_batched: rcond needs 4n scratch");
        nmax = std::max(nmax, j.n);
      }
      static std::once_flag d4attr;
      std::call_once(d4attr, [] {
        SBX_CUDA(cudaFuncSetAttribute(gj_inverse_dmma_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(gj_dmma_smem<4>(kGjMax))));
      });
      static thread_local JobTable<LuJob> d4tab;
      const LuJob* d = d4tab.upload(gj[2], s);
      KernelTimer kt("gj_inverse", s);
      gj_inverse_dmma_kernel<4><<<unsigned(gj[2].size()), kGjT, gj_dmma_smem<4>(nmax), s>>>(d);
      SBX_LAUNCHED();
      gj[2].clear();
    }
    static thread_local JobTable<LuJob> gtab[3];
    static std::once_flag gattr;
    std::call_once(gattr, [] {
      SBX_CUDA(cudaFuncSetAttribute(gj_inverse_kernel<1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(gj_smem(kGjMax))));
      SBX_CUDA(cudaFuncSetAttribute(gj_inverse_kernel<2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(gj_smem(kGjMax))));
      SBX_CUDA(cudaFuncSetAttribute(gj_inverse_kernel<4, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(gj_smem(kGjMax))));
    });
    for (int c = 0; c < 3; ++c) {
      if (gj[c].empty()) continue;
      int nmax = 1;
      for (const auto& j : gj[c]) {
        require(j.inv != nullptr, "lu_batched: the explicit inverse output is required");
        require(!j.rcond || j.work != nullptr, "lu_batched: rcond needs 4n scratch");
        nmax = std::max(nmax, j.n);
      }
      const LuJob* d = gtab[c].upload(gj[c], s);
      const unsigned g = unsigned(gj[c].size());
      KernelTimer kt("gj_inverse", s);
      const size_t sm = gj_smem(nmax);
      if (c == 0)
        gj_inverse_kernel<1, 2><<<g, kT, sm, s>>>(d);
      else if (c == 1)
        gj_inverse_kernel<2, 4><<<g, kT, sm, s>>>(d);
      else
        gj_inverse_kernel<4, 8><<<g, kT, sm, s>>>(d);
      SBX_LAUNCHED();
    }
    // 128 < n <= 160: blocked Gauss-Jordan on DMMA accumulator tiles
    // (SBX_GJ_SMEM=1: the unblocked shared-memory kernel, diagnostics)
    std::vector<LuJob> mid, rest2;
    for (const auto& j : rest) (j.n <= kGjSmemMax ? mid : rest2).push_back(j);
    static const bool gj_smem_only = std::getenv("SBX_GJ_SMEM") != nullptr;
    if (!mid.empty() && !gj_smem_only) {
      int nmax = 1;
      for (const auto& j : mid) {
        require(j.inv != nullptr, "lu_batched: the explicit inverse output is required");
        require(!j.rcond || j.work != nullptr, "lu_batched: rcond needs 4n scratch");
        nmax = std::max(nmax, j.n);
      }
      static std::once_flag dattr;
      std::call_once(dattr, [] {
        SBX_CUDA(cudaFuncSetAttribute(gj_inverse_dmma_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(gj_dmma_smem<5>(kGjSmemMax))));
      });
      static thread_local JobTable<LuJob> dtab;
      const LuJob* d = dtab.upload(mid, s);
      KernelTimer kt("gj_inverse_dmma", s);
      gj_inverse_dmma_kernel<5><<<unsigned(mid.size()), kGjT, gj_dmma_smem<5>(nmax), s>>>(d);
      SBX_LAUNCHED();
      mid.clear();
    }
    if (!mid.empty()) {
      int nmax = 1;
      for (const auto& j : mid) {
        require(j.inv != nullptr, "lu_batched: the explicit inverse output is required");
        require(!j.rcond || j.work != nullptr, "lu_batched: rcond needs 4n scratch");
        nmax = std::max(nmax, j.n);
      }
      static std::once_flag mattr;
      std::call_once(mattr, [] {
        SBX_CUDA(cudaFuncSetAttribute(gj_inverse_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(gj_smem_bytes(kGjSmemMax))));
      });
      static thread_local JobTable<LuJob> mtab;
      const LuJob* d = mtab.upload(mid, s);
      gj_inverse_smem_kernel<<<unsigned(mid.size()), kT, gj_smem_bytes(nmax), s>>>(d);
      SBX_LAUNCHED();
    }
    jobs = rest2;
    if (jobs.empty()) return;
  }
  static thread_local JobTable<LuJob> tab;
  size_t need = 64 * sizeof(double);
  for (const auto& j : jobs) {
    require(j.inv != nullptr, "lu_batched: the explicit inverse output is required");
    require(!j.rcond || j.work != nullptr, "lu_batched: rcond needs 4n scratch");
    const size_t sz = (64 + size_t(j.n) * j.n) * sizeof(double);
    if (sz <= kSmemCap) need = std::max(need, sz);
  }
  static std::once_flag attr;
  std::call_once(attr, [] {
    SBX_CUDA(cudaFuncSetAttribute(lu_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(kSmemCap)));
  });
  const LuJob* d = tab.upload(jobs, s);
  lu_kernel<<<unsigned(jobs.size()), kT, need, s>>>(d, int(need / sizeof(double)));
  SBX_LAUNCHED();
}

void lu_solve(const double* lu, int n, int lda, const int* piv, double* B, int ldb, int nrhs,
              double* scratch, cudaStream_t s) {
  if (nrhs == 0 || n == 0) return;
  require(n <= 32 * kMaxRowsPerLane, "lu_solve: matrix too large for the warp solver");
  const int warps_per_block = 8;
  lu_solve_kernel<<<unsigned((nrhs + warps_per_block - 1) / warps_per_block), 32 * warps_per_block,
                    0, s>>>(lu, n, lda, piv, B, ldb, nrhs, scratch);
  SBX_LAUNCHED();
}

void copy_batched(const std::vector<CopyJob>& jobs, cudaStream_t s) {
  if (jobs.empty()) return;
  static thread_local JobTable<CopyJob> tab;
  i64 mx = 0;
  for (const auto& j : jobs) mx = std::max<i64>(mx, i64(j.rows) * j.cols);
  if (mx == 0) return;
  const CopyJob* d = tab.upload(jobs, s);
  dim3 grid(unsigned(std::min<i64>((mx + 255) / 256, 64)), unsigned(jobs.size()));
  copy_jobs_kernel<<<grid, 256, 0, s>>>(d);
  SBX_LAUNCHED();
}

void scatter_batched(const std::vector<ScatterJob>& jobs, cudaStream_t s) {
  if (jobs.empty()) return;
  static thread_local JobTable<ScatterJob> tab;
  i64 mx = 0;
  for (const auto& j : jobs) mx = std::max<i64>(mx, i64(j.rows) * j.cols);
  if (mx == 0) return;
  const ScatterJob* d = tab.upload(jobs, s);
  dim3 grid(unsigned(std::min<i64>((mx + 255) / 256, 256)), unsigned(jobs.size()));
  scatter_jobs_kernel<<<grid, 256, 0, s>>>(d);
  SBX_LAUNCHED();
}

void launch_copy2d(const double* src, i64 lds, double* dst, i64 ldd, i64 rows, i64 cols,
                   cudaStream_t s) {
  if (rows * cols == 0) return;
  const unsigned g = unsigned(std::min<i64>((rows * cols + 255) / 256, 4096));
  copy2d_kernel<<<g, 256, 0, s>>>(src, lds, dst, ldd, rows, cols);
  SBX_LAUNCHED();
}

void launch_add_identity(double* a, i64 lda, i64 n, cudaStream_t s) {
  if (n == 0) return;
  add_identity_kernel<<<unsigned(std::min<i64>((n + 255) / 256, 1024)), 256, 0, s>>>(a, lda, n);
  SBX_LAUNCHED();
}

}  // namespace sbx
