// Row-split cluster CPQR (engine 7): one tall problem per thread-block
// cluster of G <= 8 CTAs, CTA r holding the row slab [M r / G, M (r+1) / G)
// of W^T in shared memory for the whole factorisation.
//
// The other cluster engines split COLUMNS across CTAs, so every step ships a
// pivot column of M rows between CTAs and each CTA re-reads its whole slab
// (two passes over M x n/G doubles of shared memory); for the tall, narrow
// problems of the late ID rounds (M = 257..1088 functionals, n = 20..130
// candidates) the per-step latency is what sets the round's time.  Splitting
// ROWS instead keeps every per-step exchange O(n):
//   * the column norms (upd / dir) are replicated in every CTA and updated
//     identically, so the pivot is chosen redundantly (no exchange);
//   * exchange 1: each CTA's partial sum of squares of the pivot column
//     below the diagonal (+ the diagonal entry from the owner of row j) ->
//     every CTA forms the same Householder scalars (rank-ordered sums);
//   * exchange 2: each CTA's partial dot products v^T A(:, c) over its rows
//     for all live columns, and the owner's row j -> every CTA applies the
//     reflector to its rows and downdates the replicated norms identically;
//   * (rare) exchange 3: partial column norms when the xGEQPF recompute
//     rule fires.
// Each exchange is a parity-buffered slot in shared memory read by the peers
// through DSMEM after one hardware cluster barrier: two cluster barriers per
// step.  Pivot rule (first max of the downdated norms, ties to the lower
// logical position), Householder convention, stop rule, norm downdating and
// the R layout (columns never move, perm names them) are those of the other
// engines (Eigen ColPivHouseholderQR, idlib.cpp:27-51).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cfloat>
#include <functional>
#include <map>
#include <mutex>

#include "dense.hpp"

namespace cg = cooperative_groups;

namespace sbx {

namespace {

constexpr int kRT = 512;  // threads per CTA
constexpr int kRW = kRT / 32;
constexpr int kRMaxG = 8;
constexpr size_t kRowsSmemCap = 200 * 1024;

__device__ __forceinline__ double rw_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ bool rw_better(double v, int p, double bv, int bp) {
  return v > bv || (v == bv && p < bp);
}

// Shared-memory layout (doubles unless noted), n columns, ml local rows; the
// exchange slots come first so peers address them at the same offset in
// every CTA (slab heights differ by a row between CTAs).
__host__ __device__ inline size_t rows_doubles(int ml, int n, int size) {
  return 4                      // xch1[2] = {partial, cc}
         + 4 * size_t(n)        // xch2[2]: partial dots | row j
         + 2 * size_t(n)        // xch3[2]: partial norms (recompute)
         + 2 * size_t(n)        // upd, dir
         + size_t(size)         // sbeta
         + size_t(ml | 1) * n   // slab (odd leading dimension)
         + size_t(n);           // mypos + pivstep (2 ints per column)
}

#ifdef SBX_CPQR_PROF
__device__ long long g_rows_prof[64 * 8];
#define ROWS_T(ph)                                                                                      \
  do {                                                                                                  \
    if (blockIdx.x == 0 && threadIdx.x == 0 && j < 64) g_rows_prof[j * 8 + (ph)] = clock64();          \
  } while (0)
#else
#define ROWS_T(ph) \
  do {             \
  } while (0)
#endif

// Sum over the gsz lanes of a column group (groups are aligned in the warp);
// every lane of the group gets the same bits.
__device__ __forceinline__ double group_sum(double v, int gsz) {
  for (int o = 1; o < gsz; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Rank-ordered sum of one slot over the cluster's G CTAs: all G DSMEM loads
// are issued before the first add (a remote load costs hundreds of cycles).
__device__ __forceinline__ double cluster_sum(cg::cluster_group& cl, double* slot, int G) {
  double part[kRMaxG];
#pragma unroll
  for (int q = 0; q < kRMaxG; ++q) part[q] = q < G ? *cl.map_shared_rank(slot, q) : 0.0;
  double d = 0.0;
#pragma unroll
  for (int q = 0; q < kRMaxG; ++q)
    if (q < G) d += part[q];
  return d;
}

__global__ void __launch_bounds__(kRT, 1) cpqr_rows_kernel(const QrJob* __restrict__ jobs) {
  extern __shared__ __align__(16) double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int G = int(cl.num_blocks()), r = int(cl.block_rank());
  const QrJob jb = jobs[blockIdx.x / G];
  const int M = jb.M, n = jb.n, lda = jb.lda;
  const int r0 = int(i64(M) * r / G), r1 = int(i64(M) * (r + 1) / G), ml = r1 - r0, ld = ml | 1;
  const int size = min(M, n);
  const int tid = threadIdx.x, lane = tid & 31;
  double* xch1 = sm;                            // 2 x 2
  double* xch2 = xch1 + 4;                      // 2 x 2n
  double* xch3 = xch2 + 4 * size_t(n);          // 2 x n
  double* upd = xch3 + 2 * size_t(n);           // n
  double* dir = upd + n;                        // n
  double* sbeta = dir + n;                      // size
  double* S = sbeta + size;                     // ml x n, ld = ml | 1
  int* mypos = reinterpret_cast<int*>(S + size_t(ld) * n);  // n
  int* pivstep = mypos + n;                                 // n
  __shared__ int s_p, s_lp, s_flag;
  __shared__ int s_split[kRMaxG + 1];  // row split points of the cluster (no 64-bit divisions per step)
  if (tid <= G) s_split[tid] = int(i64(M) * tid / G);
  // column groups: gsz consecutive lanes per column (a power of two, gsz n <= kRT)
  int gsz = 32;
  while (gsz > 1 && gsz * n > kRT) gsz >>= 1;
  const int gc = tid / gsz, sub = tid % gsz;  // this thread's column and row phase
  const bool has_col = gc < n;
  double* col = has_col ? S + size_t(gc) * ld : S;
  // ---- load the slab, initial norms (partials exchanged once)
  for (int c = tid / 32; c < n; c += kRT / 32)
    for (int i = lane; i < ml; i += 32) S[i + size_t(c) * ld] = __ldg(jb.a + (r0 + i) + size_t(c) * lda);
  for (int c = tid; c < n; c += kRT) {
    mypos[c] = c;
    pivstep[c] = -1;
  }
  __syncthreads();
  {
    double s2 = 0.0;
    if (has_col)
      for (int i = sub; i < ml; i += gsz) s2 = fma(col[i], col[i], s2);
    s2 = group_sum(s2, gsz);
    if (has_col && sub == 0) xch3[gc] = s2;
  }
  cl.sync();
  if (has_col && sub == 0) {
    const double s2 = cluster_sum(cl, xch3 + gc, G);
    upd[gc] = dir[gc] = sqrt(s2);
  }
  cl.sync();  // peers done reading xch3[0]; upd visible CTA-wide
  const int steps_max = jb.max_steps > 0 ? min(size, jb.max_steps) : size;
  const double thr = sqrt(DBL_EPSILON);
  double r00 = 0.0;
  int done = 0;
  for (int j = 0; j < steps_max; ++j) {
    const int par = j & 1;
    const bool own_j = j >= r0 && j < r1;
    const int i0 = max(j + 1, r0) - r0;  // first local row strictly below the diagonal
    int owner = 0;                       // CTA holding row j
    while (j >= s_split[owner + 1]) ++owner;
    ROWS_T(0);
    // ---- warp 0: pivot (first max of the replicated norms) and this CTA's
    // share of the pivot column's Householder norm
    if (tid < 32) {
      double bv = -1.0;
      int bp = 0x7fffffff, bq = -1;
      for (int c = lane; c < n; c += 32) {
        const int ps = mypos[c];
        if (ps >= 0 && rw_better(upd[c], ps, bv, bp)) {
          bv = upd[c];
          bp = ps;
          bq = c;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int op = __shfl_xor_sync(0xffffffffu, bp, o);
        const int oq = __shfl_xor_sync(0xffffffffu, bq, o);
        if (rw_better(ov, op, bv, bp)) {
          bv = ov;
          bp = op;
          bq = oq;
        }
      }
      const double* pc = S + size_t(bq) * ld;
      double part = 0.0;
      for (int i = i0 + lane; i < ml; i += 32) part = fma(pc[i], pc[i], part);
      part = rw_sum(part);
      if (lane == 0) {
        s_p = bq;
        s_lp = bp;
        xch1[2 * par] = part;
        xch1[2 * par + 1] = own_j ? pc[j - r0] : 0.0;
      }
    }
    ROWS_T(1);
    cl.sync();  // #1 (also the CTA barrier for s_p)
    ROWS_T(2);
    const int p = s_p, lp = s_lp;
    // every lane: the Householder scalars from the G shares, in rank order
    double tail = 0.0, cc = 0.0;
    {
      const double x0 = lane < G ? cl.map_shared_rank(xch1, lane)[2 * par] : 0.0;
      const double x1 = lane < G ? cl.map_shared_rank(xch1, lane)[2 * par + 1] : 0.0;
      for (int q = 0; q < G; ++q) tail += __shfl_sync(0xffffffffu, x0, q);
      cc = __shfl_sync(0xffffffffu, x1, owner);
    }
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
    const double rd = denom == 0.0 ? 0.0 : 1.0 / denom;
    if (j == 0) r00 = fabs(beta);
    // logical swap: the column at position j moves to lp, p takes position j
    // (each column's mypos is touched only by its group leader from here on)
    const int myp = has_col ? mypos[gc] : -1;
    const bool live = has_col && myp >= 0 && gc != p;
    ROWS_T(3);
    __syncthreads();  // every thread has read mypos[] before it changes
    if (has_col && sub == 0) {
      if (gc == p) {
        mypos[gc] = -1;
        pivstep[gc] = j;
      } else if (myp == j) {
        mypos[gc] = lp;
      }
    }
    if (tid == 0) {
      sbeta[j] = beta;
      if (r == 0) jb.perm[j] = p;
    }
    done = j + 1;
    if (jb.stop_eps > 0.0 && !(fabs(beta) > jb.stop_eps * r00)) break;
    // ---- exchange 2: partial dots v^T A(:, c) over the local rows (v from the
    // pivot column on the fly; the owner adds row j, v_j = 1)
    const double* pc = S + size_t(p) * ld;
    double* x2 = xch2 + size_t(par) * 2 * n;
    {
      double d = 0.0;
      if (live && tau != 0.0)
#pragma unroll 4
        for (int i = i0 + sub; i < ml; i += gsz) d = fma(pc[i] * rd, col[i], d);
      d = group_sum(d, gsz);
      if (live && sub == 0) {
        const double aj = own_j ? col[j - r0] : 0.0;
        x2[gc] = d + aj;
        x2[n + gc] = aj;
      }
    }
    ROWS_T(4);
    cl.sync();  // #2
    ROWS_T(5);
    // group leaders gather their column's dot (rank order) and the owner's row j
    double tw = 0.0, rj = 0.0;
    if (live && sub == 0) {
      rj = cl.map_shared_rank(x2, owner)[n + gc];
      tw = tau * cluster_sum(cl, x2 + gc, G);
    }
    tw = __shfl_sync(0xffffffffu, tw, lane & ~(gsz - 1));
    // ---- apply the reflector to the local rows of the column
    if (live) {
      if (tw != 0.0)
#pragma unroll 4
        for (int i = i0 + sub; i < ml; i += gsz) col[i] = fma(-(pc[i] * rd), tw, col[i]);
      if (own_j && sub == 0) col[j - r0] -= tw;
    }
    ROWS_T(6);
    // ---- xGEQPF norm downdate, identical in every CTA (row j from the owner)
    if (tid == 0) s_flag = 0;
    bool recompute = false;
    if (live && sub == 0) {
      const double uu = upd[gc];
      if (uu != 0.0) {
        const double rjn = rj - tw;  // the owner's updated R(j, c), same arithmetic
        double t = fabs(rjn) / uu;
        t = (1.0 + t) * (1.0 - t);
        t = t < 0.0 ? 0.0 : t;
        const double rr = uu / dir[gc];
        if (t * rr * rr <= thr) recompute = true;
        else upd[gc] = uu * sqrt(t);
      }
    }
    recompute = __shfl_sync(0xffffffffu, recompute ? 1 : 0, lane & ~(gsz - 1)) != 0;
    __syncthreads();
    if (recompute && sub == 0) s_flag = 1;
    __syncthreads();
    if (s_flag) {  // exchange 3 (rare): partial norms of the flagged columns below row j
      double* x3 = xch3 + size_t(par) * n;
      double s2 = 0.0;
      if (recompute)
        for (int i = i0 + sub; i < ml; i += gsz) s2 = fma(col[i], col[i], s2);
      s2 = group_sum(s2, gsz);
      if (recompute && sub == 0) x3[gc] = s2;
      cl.sync();
      if (recompute && sub == 0) {
        const double t = cluster_sum(cl, x3 + gc, G);
        upd[gc] = dir[gc] = sqrt(t);
      }
      __syncthreads();
    }
    ROWS_T(7);
  }
  cl.sync();  // peers are done reading this CTA's slots
  // ---- write back: R diagonal of the pivoted columns, the slab, perm, diag
  for (int c = tid; c < n; c += kRT) {
    const int ps = pivstep[c];
    if (ps >= r0 && ps < r1) S[(ps - r0) + size_t(c) * ld] = sbeta[ps];
  }
  __syncthreads();
  for (int c = tid / 32; c < n; c += kRT / 32)
    for (int i = lane; i < ml; i += 32) jb.a[(r0 + i) + size_t(c) * lda] = S[i + size_t(c) * ld];
  if (r == 0) {
    for (int c = tid; c < n; c += kRT)
      if (mypos[c] >= 0) jb.perm[mypos[c]] = c;
    for (int l = tid; l < size; l += kRT) jb.diag[l] = l < done ? fabs(sbeta[l]) : 0.0;
    if (tid == 0 && jb.steps) *jb.steps = done;
  }
}

struct JobTableRows {
  DevBuf<QrJob> d;
  const QrJob* upload(const std::vector<QrJob>& h, cudaStream_t s) {
    d.reserve(h.size());
    SBX_CUDA(cudaMemcpyAsync(d.get(), h.data(), h.size() * sizeof(QrJob), cudaMemcpyHostToDevice, s));
    return d.get();
  }
};

size_t rows_smem(int M, int n, int G) {
  const int ml = (M + G - 1) / G;
  return rows_doubles(ml, n, std::min(M, n)) * sizeof(double);
}

}  // namespace

#ifdef SBX_CPQR_PROF
void cpqr_rows_prof_dump() {
  long long h[64 * 8];
  SBX_CUDA(cudaMemcpyFromSymbol(h, g_rows_prof, sizeof(h)));
  for (int j = 0; j < 64; ++j) {
    if (h[j * 8 + 7] == 0) break;
    std::fprintf(stderr, "rows step %2d:", j);
    for (int q = 1; q < 8; ++q) std::fprintf(stderr, " %6lld", h[j * 8 + q] - h[j * 8 + q - 1]);
    std::fprintf(stderr, "\n");
  }
}
#endif

int cpqr_rows_cluster(int M, int n) {
  if (M <= 0 || n <= 0 || M < 2 * n) return 0;  // tall problems only
  for (int G = 1; G <= kRMaxG; G <<= 1)
    if (rows_smem(M, n, G) <= kRowsSmemCap && (M + G - 1) / G >= 8) return G;
  return 0;
}

void cpqr_rows_batched(const std::vector<QrJob>& all, cudaStream_t s) {
  if (all.empty()) return;
  static std::once_flag attr;
  std::call_once(attr, [] {
    SBX_CUDA(cudaFuncSetAttribute(cpqr_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(kRowsSmemCap)));
  });
  int dev = 0, sms = 148;
  SBX_CUDA(cudaGetDevice(&dev));
  SBX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // spread few problems over more CTAs (shorter per-step work), never past
  // one wave.  The cluster size sets the rank order of every partial sum, so
  // it must depend on the batch's multiset of shapes only, not on the order
  // the rendezvous participants arrived in: problems of one (M, n) class
  // grow together, classes taken tallest first.
  std::vector<QrJob> jobs_in(all);
  std::map<std::pair<int, int>, std::pair<int, int>, std::greater<std::pair<int, int>>> cls;  // (M, n) -> (count, G)
  i64 ctas = 0;
  for (const auto& j : jobs_in) {
    const int g = cpqr_rows_cluster(j.M, j.n);
    require(g > 0, "cpqr_rows: problem does not fit one cluster");
    auto& c = cls[{j.M, j.n}];
    c.first += 1;
    c.second = g;
    ctas += g;
  }
  static const int force_g = [] {  // diagnostics: fixed cluster size
    const char* e = std::getenv("SBX_ROWS_G");
    return e ? std::atoi(e) : 0;
  }();
  for (auto& kv : cls) {
    auto& c = kv.second;
    if (force_g > 0) {
      c.second = std::max(c.second, force_g);
      continue;
    }
    while (c.second < kRMaxG && (kv.first.first / (2 * c.second)) >= 32 && ctas + i64(c.first) * c.second <= sms) {
      ctas += i64(c.first) * c.second;
      c.second *= 2;
    }
  }
  std::vector<std::pair<int, QrJob>> sized;
  for (const auto& j : jobs_in) sized.push_back({cls[{j.M, j.n}].second, j});
  std::stable_sort(sized.begin(), sized.end(), [](const auto& a, const auto& b) { return a.first > b.first; });
  std::vector<QrJob> jobs;
  for (const auto& sj : sized) jobs.push_back(sj.second);
  static thread_local JobTableRows tab;
  const QrJob* dj = tab.upload(jobs, s);
  for (size_t g0 = 0; g0 < jobs.size();) {
    const int C = sized[g0].first;
    size_t g1 = g0;
    size_t smem = 0;
    while (g1 < jobs.size() && sized[g1].first == C) {
      smem = std::max(smem, rows_smem(jobs[g1].M, jobs[g1].n, C));
      ++g1;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned((g1 - g0) * size_t(C)));
    cfg.blockDim = dim3(kRT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = unsigned(C);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const QrJob* jp = dj + g0;
    SBX_CUDA(cudaLaunchKernelEx(&cfg, cpqr_rows_kernel, jp));
    SBX_LAUNCHED();
    g0 = g1;
  }
}

}  // namespace sbx
