// One-exchange row-split cluster CPQR (engine 8): one tall problem per
// thread-block cluster of G <= 8 CTAs, CTA r holding the row slab
// [M r / G, M (r+1) / G) of W^T in shared memory for the whole factorisation.
//
// Engine 7 (cpqr_rows.cu) needs two cluster-wide exchanges per Householder
// step (the pivot column's norm, then the dot products v^T A(:, c)) plus
// pulls of remote slots after each hardware cluster barrier.  This engine
// folds them into ONE pushed exchange per step:
//   * every CTA computes, over its rows strictly below the diagonal, the
//     UNSCALED dots x^T A(:, c) of the pivot column x with every unpivoted
//     column c, the pivot column itself included (x^T x is the Householder
//     tail norm), and the owner of row j adds A(j, c);
//   * the column groups push those values into every CTA's slot with
//     st.async (remote shared-memory stores that complete a transaction count
//     on the receiver's mbarrier): no cluster barrier and no remote loads on
//     the critical path, each CTA waits on its own mbarrier for
//     (n - j) (8 G + 8) bytes;
//   * every CTA then forms the same Householder scalars and
//     w_c = tau (A(j, c) + (x^T A(:, c)) / (x_j - beta)) from the G partials
//     summed in rank order, applies the reflector to its rows and downdates
//     the replicated column norms identically, and picks the next pivot
//     redundantly (one CTA barrier per step).
// The xGEQPF recompute (rare) pulls partial norms after a cluster barrier.
// Pivot rule (first max of the downdated norms, ties to the lower logical
// position), Householder convention, stop rule, norm downdating and the R
// layout (columns never move, perm names them) are those of the other
// engines (Eigen ColPivHouseholderQR, reference idlib.cpp:27-51); the dot
// products are scaled by 1/(x_j - beta) after the sum instead of before it
// (same value in exact arithmetic).
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "dense.hpp"

namespace cg = cooperative_groups;

namespace sbx {

namespace {

constexpr int kPT = 512;  // threads per CTA
constexpr int kPW = kPT / 32;
constexpr int kPMaxG = 8;
constexpr size_t kPushSmemCap = 220 * 1024;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ unsigned mapa_u32(unsigned a, int rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void push_f64(unsigned raddr, double v, unsigned rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
               :
               : "r"(raddr), "l"(__double_as_longlong(v)), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void push_f64x2(unsigned raddr, double a, double b, unsigned rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];"
               :
               : "r"(raddr), "l"(__double_as_longlong(a)), "l"(__double_as_longlong(b)), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" : : "r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" : : "r"(bar), "r"(bytes) : "memory");
}
// Wait for the phase with the given parity; traps (instead of hanging the
// GPU) if it never completes.
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  unsigned done = 0;
  for (long long it = 0;; ++it) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    if (it > (1ll << 26)) __trap();
  }
}

// Sum over the gsz lanes of a column group (groups are aligned in the warp);
// every lane of the group gets the same bits.
__device__ __forceinline__ double grp_sum(double v, int gsz) {
  for (int o = 1; o < gsz; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Candidate order: larger norm, then lower logical position (key = pos << 16 | column).
__device__ __forceinline__ bool cand_better(double v, unsigned k, double bv, unsigned bk) {
  return v > bv || (v == bv && k < bk);
}
__device__ __forceinline__ void warp_argmax(double& v, unsigned& k) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const unsigned ok = __shfl_xor_sync(0xffffffffu, k, o);
    if (cand_better(ov, ok, v, k)) {
      v = ov;
      k = ok;
    }
  }
}

#ifdef SBX_CPQR_PROF
__device__ long long g_push_prof[64 * 8];
__device__ unsigned long long g_push_cta[4096 * 4];  // per CTA: start, end (globaltimer ns), M | n << 16 | G << 28, steps
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PUSH_T(ph)                                                                                      \
  do {                                                                                                  \
    if (blockIdx.x == 0 && threadIdx.x == 0 && j < 64) g_push_prof[j * 8 + (ph)] = clock64();          \
  } while (0)
#else
#define PUSH_T(ph) \
  do {             \
  } while (0)
#endif

struct PushLayout {
  // byte offsets of the per-CTA shared-memory regions (identical in every
  // CTA of a cluster: remote addresses are the local ones mapped by rank)
  size_t bar, cand, slot, rowj, x3, slab, total;
  int ld;
};
__host__ __device__ inline PushLayout push_layout(int ml_max, int n, int G) {
  PushLayout L{};
  L.bar = 0;                                              // 2 mbarriers
  L.cand = 16;                                            // 2 x n doubles (norms) + 2 x n keys
  L.slot = L.cand + ((2 * size_t(n) * 12 + 15) / 16) * 16;  // 2 x G x n x double2 {dot, sum of squares}
  L.rowj = L.slot + 2 * size_t(G) * n * 16;               // 2 x n doubles: row j from its owner
  L.x3 = L.rowj + 2 * size_t(n) * 8;                      // 2 x n doubles
  L.slab = L.x3 + 2 * size_t(n) * 8;                      // ld x n doubles
  L.ld = ml_max | 1;
  L.total = L.slab + size_t(L.ld) * n * 8;
  return L;
}

__global__ void __launch_bounds__(kPT, 1) cpqr_push_kernel(const QrJob* __restrict__ jobs) {
  extern __shared__ __align__(16) unsigned char smraw[];
  cg::cluster_group cl = cg::this_cluster();
  const int G = int(cl.num_blocks()), r = int(cl.block_rank());
  const QrJob jb = jobs[blockIdx.x / G];
  const int M = jb.M, n = jb.n, lda = jb.lda;
  const int r0 = int(i64(M) * r / G), r1 = int(i64(M) * (r + 1) / G), ml = r1 - r0;
  const PushLayout L = push_layout((M + G - 1) / G, n, G);
  const int ld = L.ld;
  const int size = min(M, n);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef SBX_CPQR_PROF
  if (tid == 0 && blockIdx.x < 4096) g_push_cta[blockIdx.x * 4] = gtimer();
#endif
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smraw + L.bar);
  double* cand_v = reinterpret_cast<double*>(smraw + L.cand);                   // [2][n] norms
  unsigned* cand_k = reinterpret_cast<unsigned*>(smraw + L.cand + 2 * size_t(n) * 8);  // [2][n] keys
  double2* slot = reinterpret_cast<double2*>(smraw + L.slot);             // [2][G][n]
  double* rowj = reinterpret_cast<double*>(smraw + L.rowj);               // [2][n]
  double* x3 = reinterpret_cast<double*>(smraw + L.x3);                   // [2][n]
  double* S = reinterpret_cast<double*>(smraw + L.slab);                  // ld x n
  __shared__ int s_split[kPMaxG + 1];
  if (tid <= G) s_split[tid] = int(i64(M) * tid / G);
  // mbarrier q counts the pushes of the steps j = q (mod 2); each use is
  // armed (arrive + expected bytes) before any peer can push into it: at
  // initialisation for steps 0 and 1, and for step j + 2 right after step
  // j's phase completed (a peer pushes step j + 2 only after it has received
  // this CTA's step j + 1 values, which leave after that point).
  if (tid == 0) {
    mbar_init(smem_u32(&bars[0]), 1);
    mbar_init(smem_u32(&bars[1]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int q = 0; q < 2 && q < n; ++q) mbar_arrive_expect(smem_u32(&bars[q]), unsigned((n - q) * (16 * G + 8)));
  }
  // column groups: gsz consecutive lanes per column (a power of two, gsz n <= kPT)
  int gsz = 32;
  while (gsz > 1 && gsz * n > kPT) gsz >>= 1;
  const int gc = tid / gsz, sub = tid % gsz;
  const bool has_col = gc < n;
  double* col = S + size_t(has_col ? gc : 0) * ld;
  // ---- load the slab
  for (int c = warp; c < n; c += kPW)
    for (int i = lane; i < ml; i += 32) S[i + size_t(c) * ld] = __ldg(jb.a + (r0 + i) + size_t(c) * lda);
  __syncthreads();
  // per-column state, replicated in every lane of the column's group
  double upd = 0.0, mybeta = 0.0;
  int myp = has_col ? gc : -1, pivstep = -1;
  {  // initial norms: partials through x3[1] (pulled after a cluster barrier)
    double s2 = 0.0;
    if (has_col)
      for (int i = sub; i < ml; i += gsz) s2 = fma(col[i], col[i], s2);
    s2 = grp_sum(s2, gsz);
    if (has_col && sub == 0) x3[n + gc] = s2;
  }
  cl.sync();  // also publishes the mbarrier initialisation cluster-wide
  if (has_col) {
    double part[kPMaxG];
#pragma unroll
    for (int q = 0; q < kPMaxG; ++q) part[q] = q < G ? *cl.map_shared_rank(x3 + n + gc, q) : 0.0;
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < kPMaxG; ++q)
      if (q < G) t += part[q];
    upd = sqrt(t);
  }
  // argmax of the replicated norms over the CTA; every thread gets the pivot:
  // the column leaders publish (norm, pos << 16 | column), one CTA barrier
  // (which also ORs the recompute flags), then every warp scans all n
  auto pick = [&](int par, bool flag, int& p, int& lp, bool& anyflag) {
    if (has_col && sub == 0) {
      cand_v[par * n + gc] = myp >= 0 ? upd : -1.0;
      cand_k[par * n + gc] = myp >= 0 ? ((unsigned(myp) << 16) | unsigned(gc)) : 0xffffffffu;
    }
    anyflag = __syncthreads_or(flag ? 1 : 0) != 0;
    double bv = -1.0;
    unsigned bk = 0xffffffffu;
    for (int c = lane; c < n; c += 32) {
      const double v = cand_v[par * n + c];
      const unsigned k = cand_k[par * n + c];
      if (cand_better(v, k, bv, bk)) {
        bv = v;
        bk = k;
      }
    }
    warp_argmax(bv, bk);
    p = int(bk & 0xffffu);
    lp = int(bk >> 16);
  };
  int p = 0, lp = 0;
  {
    bool af = false;
    pick(1, false, p, lp, af);
  }
  const int steps_max = jb.max_steps > 0 ? min(size, jb.max_steps) : size;
  const double thr = sqrt(DBL_EPSILON);
  double r00 = 0.0;
  int done = 0, owner = 0;
  const unsigned slot_u32 = smem_u32(slot);
  const unsigned bar_u32 = smem_u32(bars);
  const unsigned rowj_u32 = smem_u32(rowj);
  for (int j = 0; j < steps_max; ++j) {
    const int par = j & 1;
    PUSH_T(0);
    while (j >= s_split[owner + 1]) ++owner;
    const bool own_j = owner == r;
    const int i0 = max(j + 1, r0) - r0;  // first local row strictly below the diagonal
    const double* pc = S + size_t(p) * ld;
    // ---- unscaled partial dots with the pivot column and partial squared
    // norms over the rows below the diagonal (+ row j from its owner), pushed
    const bool alive = has_col && myp >= 0;
    double d0 = 0.0, d1 = 0.0, s0 = 0.0, s1 = 0.0;
    if (alive) {
      int i = i0 + sub;
#pragma unroll 2
      for (; i + gsz < ml; i += 2 * gsz) {
        const double a0 = col[i], a1 = col[i + gsz];
        const double x0 = pc[i], x1 = pc[i + gsz];
        d0 = fma(x0, a0, d0);
        s0 = fma(a0, a0, s0);
        d1 = fma(x1, a1, d1);
        s1 = fma(a1, a1, s1);
      }
      if (i < ml) {
        const double a0 = col[i];
        d0 = fma(pc[i], a0, d0);
        s0 = fma(a0, a0, s0);
      }
    }
    const double d = grp_sum(d0 + d1, gsz);  // whole warp: groups of dead columns too
    const double sq = grp_sum(s0 + s1, gsz);
    PUSH_T(1);
    if (alive) {
      const unsigned off = unsigned(((par * G + r) * n + gc) * 16);
      const unsigned boff = unsigned(par * 8);
      for (int q = sub; q < G; q += gsz) push_f64x2(mapa_u32(slot_u32 + off, q), d, sq, mapa_u32(bar_u32 + boff, q));
      if (own_j) {
        const double aj = col[j - r0];
        const unsigned roff = unsigned((par * n + gc) * 8);
        for (int q = sub; q < G; q += gsz) push_f64(mapa_u32(rowj_u32 + roff, q), aj, mapa_u32(bar_u32 + boff, q));
      }
    }
    mbar_wait(bar_u32 + unsigned(par * 8), unsigned((j >> 1) & 1));
    if (tid == 0 && j + 2 < n) mbar_arrive_expect(bar_u32 + unsigned(par * 8), unsigned((n - j - 2) * (16 * G + 8)));
    PUSH_T(2);
    // ---- Householder scalars (every thread, same bits in every CTA)
    const double2* sl = slot + size_t(par) * G * n;
    const double* rj = rowj + size_t(par) * n;
    double tail = 0.0;
    {
      double part[kPMaxG];
#pragma unroll
      for (int q = 0; q < kPMaxG; ++q) part[q] = q < G ? sl[size_t(q) * n + p].x : 0.0;
#pragma unroll
      for (int q = 0; q < kPMaxG; ++q)
        if (q < G) tail += part[q];
    }
    const double cc = rj[p];
    double tau, beta, rd;
    if (tail <= DBL_MIN) {
      tau = 0.0;
      beta = cc;
      rd = 0.0;
    } else {
      beta = sqrt(fma(cc, cc, tail));
      if (cc >= 0.0) beta = -beta;
      const double den = cc - beta;
      rd = 1.0 / den;  // the two divisions are independent
      tau = -den / beta;
    }
    if (j == 0) r00 = fabs(beta);
    if (r == 0 && tid == 0) {
      jb.perm[j] = p;
      jb.diag[j] = fabs(beta);
    }
    // logical swap: p takes position j, the column at position j moves to lp
    const bool is_piv = has_col && gc == p;
    if (is_piv) {
      myp = -1;
      pivstep = j;
      mybeta = beta;
    } else if (alive && myp == j) {
      myp = lp;
    }
    done = j + 1;
    if (jb.stop_eps > 0.0 && !(fabs(beta) > jb.stop_eps * r00)) break;
    PUSH_T(3);
    // ---- apply the reflector to this CTA's rows; the column's new norm below
    // row j from its FRESH norm over rows >= j (a reflection keeps it) minus
    // R(j, c)^2, with a direct recomputation when that cancels below
    // sqrt(eps) (the xGEQPF rule, applied to one step's drop)
    bool recompute = false;
    unsigned long long kb = 0ull;
    if (alive && !is_piv) {
      double part[kPMaxG], pars[kPMaxG];
#pragma unroll
      for (int q = 0; q < kPMaxG; ++q) {
        const double2 v = q < G ? sl[size_t(q) * n + gc] : make_double2(0.0, 0.0);
        part[q] = v.x;
        pars[q] = v.y;
      }
      double dsum = 0.0, ssum = 0.0;
#pragma unroll
      for (int q = 0; q < kPMaxG; ++q)
        if (q < G) {
          dsum += part[q];
          ssum += pars[q];
        }
      const double aj = rj[gc];
      const double tw = tau * (aj + dsum * rd);
      if (tw != 0.0) {
        const double sc = tw * rd;
        for (int i = i0 + sub; i < ml; i += gsz) col[i] = fma(-pc[i], sc, col[i]);
        if (own_j && sub == 0) col[j - r0] = aj - tw;
      }
      const double rjn = aj - tw;  // R(j, c) in every CTA
      const double full = fma(aj, aj, ssum);
      const double n2 = fma(-rjn, rjn, full);
      if (!(n2 > thr * full)) recompute = full > 0.0;
      else upd = sqrt(n2);
      if (!(full > 0.0)) upd = 0.0;
    }
    PUSH_T(4);
    bool anyflag = false;
    pick(par, recompute, p, lp, anyflag);
    PUSH_T(5);
    if (anyflag) {  // rare: exact norms of the flagged columns below row j
      double* xr = x3 + size_t(par) * n;
      double s2 = 0.0;
      if (recompute)
        for (int i = i0 + sub; i < ml; i += gsz) s2 = fma(col[i], col[i], s2);
      s2 = grp_sum(s2, gsz);
      if (recompute && sub == 0) xr[gc] = s2;
      cl.sync();
      if (recompute) {
        double part[kPMaxG];
#pragma unroll
        for (int q = 0; q < kPMaxG; ++q) part[q] = q < G ? *cl.map_shared_rank(xr + gc, q) : 0.0;
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < kPMaxG; ++q)
          if (q < G) t += part[q];
        upd = sqrt(t);
      }
      bool af2 = false;
      pick(par, false, p, lp, af2);
    }
    PUSH_T(6);
  }
  cl.sync();  // peers are done with this CTA's slots and x3
  // ---- write back: R diagonal of the pivoted columns, the slab, perm, diag
  if (has_col && sub == 0 && pivstep >= r0 && pivstep < r1) S[(pivstep - r0) + size_t(gc) * ld] = mybeta;
  __syncthreads();
  for (int c = warp; c < n; c += kPW)
    for (int i = lane; i < ml; i += 32) jb.a[(r0 + i) + size_t(c) * lda] = S[i + size_t(c) * ld];
  if (r == 0) {
    if (has_col && sub == 0 && myp >= 0) jb.perm[myp] = gc;
    for (int l = done + tid; l < size; l += kPT) jb.diag[l] = 0.0;
    if (tid == 0 && jb.steps) *jb.steps = done;
  }
#ifdef SBX_CPQR_PROF
  if (tid == 0 && blockIdx.x < 4096) {
    g_push_cta[blockIdx.x * 4 + 1] = gtimer();
    g_push_cta[blockIdx.x * 4 + 2] = (unsigned long long)M | ((unsigned long long)n << 16) | ((unsigned long long)G << 28);
    g_push_cta[blockIdx.x * 4 + 3] = (unsigned long long)done;
  }
#endif
}

// ---------------------------------------------------------------- engine 9
// Register-resident variant: the same row split and pushed exchange, but
// each thread keeps its column's rows sub + t gsz (t < RPT) in REGISTERS,
// and no step has a serial section: every column group forms the (same)
// Householder scalars and its own column's w_c, R(j, c) (written straight
// to global memory by the owner of row j) and new squared norm from the
// exchanged sums, applies the reflector to its rows at once, and bids for
// the next pivot with one shared-memory atomicMax of a packed key (norm's
// leading 48 bits, then the lower logical position); one CTA barrier later
// every thread knows the pivot, whose group publishes its column into the
// broadcast buffer XV for the next step's dots (second CTA barrier).
// Norms are tracked squared; keys compare them to 2^-36 relative (well
// inside the 1e-8 the fresh-norm formula guarantees, and Eigen's own
// downdated norms carry), ties going to the lower position.
constexpr int kRRXv = 1024;  // XV doubles per parity (>= RPT * gsz)
__host__ __device__ inline size_t rr_smem(int /*ml_max*/, int n, int G) {
  return 16                        // 2 mbarriers
         + 2 * size_t(G) * n * 16  // slots {dot, sum of squares}
         + 2 * size_t(n) * 8       // row j received
         + 2 * size_t(n) * 8       // x3 (initial norms, recompute)
         + 2 * size_t(kRRXv) * 8   // XV: pivot column, two parities
         + size_t(n) * 8 + 16;     // rowbuf
}

// pivot bid: squared norm's leading 48 bits, then the lower logical
// position (n <= 256), then the column
__device__ __forceinline__ unsigned long long rr_key(double n2, int pos, int col) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(n2 > 0.0 ? n2 : 0.0));
  return ((b >> 16) << 16) | ((255ull - unsigned(pos)) << 8) | unsigned(col);
}
__device__ __forceinline__ int rr_key_col(unsigned long long k) { return int(k & 0xffull); }
// warp max of a 64-bit key with two 32-bit REDUX steps (every lane gets it)
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long k) {
  const unsigned hi = unsigned(k >> 32), lo = unsigned(k);
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  return (static_cast<unsigned long long>(mhi) << 32) | mlo;
}
__device__ __forceinline__ int rr_key_pos(unsigned long long k) { return 255 - int((k >> 8) & 0xffull); }

template <int RPT, int gsz>
__global__ void __launch_bounds__(kPT, 1) cpqr_regrows_kernel(const QrJob* __restrict__ jobs) {
  extern __shared__ __align__(16) unsigned char smraw[];
  cg::cluster_group cl = cg::this_cluster();
  const int G = int(cl.num_blocks()), r = int(cl.block_rank());
  const QrJob jb = jobs[blockIdx.x / G];
  const int M = jb.M, n = jb.n, lda = jb.lda;
  const int r0 = int(i64(M) * r / G), r1 = int(i64(M) * (r + 1) / G), ml = r1 - r0;
  const int size = min(M, n);
  const int tid = threadIdx.x, nt = int(blockDim.x), lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
#ifdef SBX_CPQR_PROF
  if (tid == 0 && blockIdx.x < 4096) g_push_cta[blockIdx.x * 4] = gtimer();
#endif
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smraw);
  size_t off = 16;
  double2* slot = reinterpret_cast<double2*>(smraw + off);  // [2][G][n]
  off += 2 * size_t(G) * n * 16;
  double* rowin = reinterpret_cast<double*>(smraw + off);  // [2][n] row j (from its owner)
  off += 2 * size_t(n) * 8;
  double* x3 = reinterpret_cast<double*>(smraw + off);  // [2][n]
  off += 2 * size_t(n) * 8;
  double* XV = reinterpret_cast<double*>(smraw + off);  // [2][kRRXv]
  off += 2 * size_t(kRRXv) * 8;
  double* rowbuf = reinterpret_cast<double*>(smraw + off);  // [n] this CTA's row j (if owned)
  __shared__ int s_split[kPMaxG + 1];
  __shared__ unsigned long long s_bid[2][kPW];  // per-warp pivot bids, two parities
  __shared__ double s_sc[4];                    // tau, rd, beta (warp 0 -> all), stop flag
  if (tid <= G) s_split[tid] = int(i64(M) * tid / G);
  if (tid == 0) {
    mbar_init(smem_u32(&bars[0]), 1);
    mbar_init(smem_u32(&bars[1]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int q = 0; q < 2 && q < n; ++q) mbar_arrive_expect(smem_u32(&bars[q]), unsigned((n - q) * (16 * G + 8)));
  }
  const int gc = tid / gsz, sub = tid % gsz;  // gsz lanes per column (host-chosen, blockDim >= gsz n)
  const bool has_col = gc < n;
  // ---- the column slab in registers: rows sub + t gsz (zero beyond the slab)
  double a[RPT];
#pragma unroll
  for (int t = 0; t < RPT; ++t) {
    const int i = sub + t * gsz;
    a[t] = (has_col && i < ml) ? __ldg(jb.a + (r0 + i) + size_t(gc) * lda) : 0.0;
  }
  {
    double s2 = 0.0;
#pragma unroll
    for (int t = 0; t < RPT; ++t) s2 = fma(a[t], a[t], s2);
    s2 = grp_sum(s2, gsz);
    if (has_col && sub == 0) x3[n + gc] = s2;
  }
  // Rows at and above the current diagonal are ZERO in the registers (their
  // R values go to global memory as they become final), so the per-step
  // passes need no row predicates.  Row 0: staged for the first push, zeroed.
  if (r == 0 && has_col && sub == 0) {
    rowbuf[gc] = a[0];
    a[0] = 0.0;
  }
  auto tree8 = [](const double* v) { return ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7])); };
  auto bid = [&](unsigned long long k, unsigned long long* slots) {
    k = warp_max_u64(k);
    if (lane == 0) slots[warp] = k;
  };
  auto bids_max = [&](const unsigned long long* slots) { return warp_max_u64(lane < nw ? slots[lane] : 0ull); };
  int myp = has_col ? gc : -1;  // logical position (-1: pivoted), same in every lane of the group
  cl.sync();                    // also publishes the mbarrier initialisation cluster-wide
  {
    unsigned long long kb = 0ull;
    if (has_col && sub == 0) {
      double v[kPMaxG];
#pragma unroll
      for (int q = 0; q < kPMaxG; ++q) v[q] = q < G ? *cl.map_shared_rank(x3 + n + gc, q) : 0.0;
      kb = rr_key(tree8(v), myp, gc);
    }
    bid(kb, s_bid[0]);
  }
  __syncthreads();
  unsigned long long key = bids_max(s_bid[0]);
  int p = rr_key_col(key), lp = rr_key_pos(key);
  if (has_col && gc == p) {
#pragma unroll
    for (int t = 0; t < RPT; ++t) XV[sub + t * gsz] = a[t];
  }
  __syncthreads();
  const int steps_max = jb.max_steps > 0 ? min(size, jb.max_steps) : size;
  const double thr = sqrt(DBL_EPSILON);
  double r00 = 0.0;
  int done = 0, owner = 0;
  const unsigned slot_u32 = smem_u32(slot);
  const unsigned bar_u32 = smem_u32(bars);
  const unsigned rowin_u32 = smem_u32(rowin);
  for (int j = 0; j < steps_max; ++j) {
    const int par = j & 1;
    PUSH_T(0);
    while (j >= s_split[owner + 1]) ++owner;
    const bool own_j = owner == r;
    const double* xv = XV + size_t(par) * kRRXv;
    const bool alive = has_col && myp >= 0;
    // ---- dots with the pivot column and sums of squares below the diagonal
    double d0 = 0.0, d1 = 0.0, q0 = 0.0, q1 = 0.0;
#pragma unroll
    for (int t = 0; t < RPT; t += 2) {
      d0 = fma(xv[sub + t * gsz], a[t], d0);
      q0 = fma(a[t], a[t], q0);
      if (t + 1 < RPT) {
        d1 = fma(xv[sub + (t + 1) * gsz], a[t + 1], d1);
        q1 = fma(a[t + 1], a[t + 1], q1);
      }
    }
    const double d = grp_sum(d0 + d1, gsz);
    const double sq = grp_sum(q0 + q1, gsz);
    PUSH_T(1);
    if (alive) {
      const unsigned so = unsigned(((par * G + r) * n + gc) * 16);
      const unsigned bo = unsigned(par * 8);
      for (int q = sub; q < G; q += gsz) push_f64x2(mapa_u32(slot_u32 + so, q), d, sq, mapa_u32(bar_u32 + bo, q));
      if (own_j) {
        const double aj = rowbuf[gc];
        const unsigned ro = unsigned((par * n + gc) * 8);
        for (int q = sub; q < G; q += gsz) push_f64(mapa_u32(rowin_u32 + ro, q), aj, mapa_u32(bar_u32 + bo, q));
      }
    }
    const double2* sl = slot + size_t(par) * G * n;
    const double* rj = rowin + size_t(par) * n;
    if (warp == 0) {
      // ---- warp 0: the exchange, then the Householder scalars (same bits in every CTA)
      // (re-arming below cannot complete the next phase before this CTA's
      // step j + 2 pushes, which follow B2)
      mbar_wait(bar_u32 + unsigned(par * 8), unsigned((j >> 1) & 1));
      if (lane == 0) {
        if (j + 2 < n) mbar_arrive_expect(bar_u32 + unsigned(par * 8), unsigned((n - j - 2) * (16 * G + 8)));
        double v[kPMaxG];
#pragma unroll
        for (int q = 0; q < kPMaxG; ++q) v[q] = q < G ? sl[size_t(q) * n + p].x : 0.0;
        const double tail = tree8(v);
        const double cc = rj[p];
        double tau, beta, rd;
        if (tail <= DBL_MIN) {
          tau = 0.0;
          beta = cc;
          rd = 0.0;
        } else {
          beta = sqrt(fma(cc, cc, tail));
          if (cc >= 0.0) beta = -beta;
          const double den = cc - beta;
          rd = 1.0 / den;
          tau = -den / beta;
        }
        if (j == 0) r00 = fabs(beta);
        const bool stop = jb.stop_eps > 0.0 && !(fabs(beta) > jb.stop_eps * r00);
        s_sc[0] = tau;
        s_sc[1] = rd;
        s_sc[2] = stop ? 1.0 : 0.0;
        if (r == 0) {
          jb.perm[j] = p;
          jb.diag[j] = fabs(beta);
        }
        if (own_j) jb.a[j + size_t(p) * lda] = beta;
      }
    }
    __syncthreads();  // B0
    PUSH_T(2);
    const double tau = s_sc[0], rd = s_sc[1];
    const bool stop = s_sc[2] != 0.0;
    // logical swap: p takes position j, the column at position j moves to lp
    const bool is_piv = has_col && gc == p;
    if (is_piv) myp = -1;
    else if (alive && myp == j) myp = lp;
    done = j + 1;
    if (stop) break;
    PUSH_T(3);
    // ---- this column: w_c, R(j, c), the reflector on its rows, new norm
    bool recompute = false;
    unsigned long long kb = 0ull;
    if (alive && !is_piv) {
      double vx[kPMaxG], vy[kPMaxG];
#pragma unroll
      for (int q = 0; q < kPMaxG; ++q) {
        const double2 v = q < G ? sl[size_t(q) * n + gc] : make_double2(0.0, 0.0);
        vx[q] = v.x;
        vy[q] = v.y;
      }
      const double aj = rj[gc];
      const double tw = tau * (aj + tree8(vx) * rd);
      const double rjn = aj - tw;  // R(j, c)
      const double sc = tw * rd;
      if (own_j && sub == 0) jb.a[j + size_t(gc) * lda] = rjn;
#pragma unroll
      for (int t = 0; t < RPT; ++t) a[t] = fma(-xv[sub + t * gsz], sc, a[t]);
      const double full = fma(aj, aj, tree8(vy));
      const double n2 = fma(-rjn, rjn, full);
      if (full > 0.0 && !(n2 > thr * full)) recompute = true;
      else if (sub == 0) kb = rr_key(full > 0.0 ? n2 : 0.0, myp, gc);
    }
    bid(kb, s_bid[par ^ 1]);
    const bool anyflag = __syncthreads_or(recompute ? 1 : 0) != 0;  // B1
    PUSH_T(4);
    if (anyflag) {  // rare: exact squared norms of the flagged columns below row j
      double s2 = 0.0;
      if (recompute) {
#pragma unroll
        for (int t = 0; t < RPT; ++t) s2 = fma(a[t], a[t], s2);
      }
      s2 = grp_sum(s2, gsz);
      double* xr = x3 + size_t(par) * n;
      if (recompute && sub == 0) xr[gc] = s2;
      cl.sync();  // (also: every warp is past B1)
      unsigned long long k2 = 0ull;
      if (recompute && sub == 0) {
        double v[kPMaxG];
#pragma unroll
        for (int q = 0; q < kPMaxG; ++q) v[q] = q < G ? *cl.map_shared_rank(xr + gc, q) : 0.0;
        k2 = rr_key(tree8(v), myp, gc);
      }
      const unsigned long long k1 = bids_max(s_bid[par ^ 1]);
      __syncthreads();
      bid(k2 > k1 ? k2 : k1, s_bid[par ^ 1]);
      __syncthreads();
    }
    key = bids_max(s_bid[par ^ 1]);
    p = rr_key_col(key);
    lp = rr_key_pos(key);
    // ---- stage row j + 1 for the next push and zero it; publish the next pivot column
    {
      const int jn = j + 1;
      if (jn >= r0 && jn < r1 && has_col) {
        const int ln = jn - r0, tn = ln / gsz;
        if (sub == ln % gsz) {
          double v = 0.0;
#pragma unroll
          for (int t = 0; t < RPT; ++t)
            if (t == tn) {
              v = a[t];
              a[t] = 0.0;
            }
          rowbuf[gc] = v;
        }
      }
    }
    if (has_col && gc == p) {
      double* xn = XV + size_t(par ^ 1) * kRRXv;
#pragma unroll
      for (int t = 0; t < RPT; ++t) xn[sub + t * gsz] = a[t];
    }
    __syncthreads();  // B2
    PUSH_T(5);
    PUSH_T(6);
  }
  cl.sync();  // peers are done with this CTA's slots and x3
  // ---- write back the rows below the last step (rows above it were written
  // as R rows step by step; the pivoted columns keep their Householder
  // vectors below their diagonal)
  if (has_col) {
#pragma unroll
    for (int t = 0; t < RPT; ++t) {
      const int i = sub + t * gsz;
      if (i < ml && r0 + i >= done) jb.a[(r0 + i) + size_t(gc) * lda] = a[t];
    }
  }
  if (r == 0) {
    if (has_col && sub == 0 && myp >= 0) jb.perm[myp] = gc;
    for (int l = done + tid; l < size; l += nt) jb.diag[l] = 0.0;
    if (tid == 0 && jb.steps) *jb.steps = done;
  }
#ifdef SBX_CPQR_PROF
  if (tid == 0 && blockIdx.x < 4096) {
    g_push_cta[blockIdx.x * 4 + 1] = gtimer();
    g_push_cta[blockIdx.x * 4 + 2] = (unsigned long long)M | ((unsigned long long)n << 16) | ((unsigned long long)G << 28);
    g_push_cta[blockIdx.x * 4 + 3] = (unsigned long long)done;
  }
#endif
}

struct JobTablePush {
  DevBuf<QrJob> d;
  const QrJob* upload(const std::vector<QrJob>& h, cudaStream_t s) {
    d.reserve(h.size());
    SBX_CUDA(cudaMemcpyAsync(d.get(), h.data(), h.size() * sizeof(QrJob), cudaMemcpyHostToDevice, s));
    return d.get();
  }
};

size_t push_smem(int M, int n, int G) { return push_layout((M + G - 1) / G, n, G).total; }

}  // namespace

#ifdef SBX_CPQR_PROF
void cpqr_push_prof_dump() {
  long long h[64 * 8];
  SBX_CUDA(cudaMemcpyFromSymbol(h, g_push_prof, sizeof(h)));
  for (int j = 0; j < 64; ++j) {
    if (h[j * 8 + 6] == 0) break;
    std::fprintf(stderr, "push step %2d:", j);
    for (int q = 1; q < 7; ++q) std::fprintf(stderr, " %6lld", h[j * 8 + q] - h[j * 8 + q - 1]);
    std::fprintf(stderr, "\n");
  }
  static std::vector<unsigned long long> c(4096 * 4);
  SBX_CUDA(cudaMemcpyFromSymbol(c.data(), g_push_cta, c.size() * 8));
  unsigned long long t0 = ~0ull;
  for (int b = 0; b < 4096; ++b)
    if (c[b * 4 + 2]) t0 = std::min(t0, c[b * 4]);
  std::map<std::string, std::vector<double>> cls;
  for (int b = 0; b < 4096; ++b) {
    const unsigned long long d = c[b * 4 + 2];
    if (!d) continue;
    char k[96];
    std::snprintf(k, sizeof(k), "%llux%llu G%llu", d & 0xffff, (d >> 16) & 0xfff, d >> 28);
    cls[k].push_back(double(c[b * 4] - t0) * 1e-3);
    cls[k].push_back(double(c[b * 4 + 1] - c[b * 4]) * 1e-3);
    cls[k].push_back(double(c[b * 4 + 3]));
  }
  for (const auto& kv : cls) {
    double st = 1e30, en = 0, dmax = 0, smax = 0;
    for (size_t i = 0; i < kv.second.size(); i += 3) {
      st = std::min(st, kv.second[i]);
      en = std::max(en, kv.second[i] + kv.second[i + 1]);
      dmax = std::max(dmax, kv.second[i + 1]);
      smax = std::max(smax, kv.second[i + 2]);
    }
    std::fprintf(stderr, "  %-18s ctas %4zu start %8.1f end %8.1f us, max CTA %7.1f us, max steps %3.0f\n", kv.first.c_str(),
                 kv.second.size() / 3, st, en, dmax, smax);
  }
  void* ptr = nullptr;
  SBX_CUDA(cudaGetSymbolAddress(&ptr, g_push_cta));
  SBX_CUDA(cudaMemset(ptr, 0, 4096 * 4 * 8));
}
#endif

int cpqr_push_cluster(int M, int n) {
  if (M <= 0 || n <= 0 || M < 2 * n || n > kPT) return 0;  // tall problems only
  for (int G = 1; G <= kPMaxG; G <<= 1)
    if (push_smem(M, n, G) <= kPushSmemCap && (M + G - 1) / G >= 8) return G;
  return 0;
}

void cpqr_push_batched(const std::vector<QrJob>& all, cudaStream_t s) {
  if (all.empty()) return;
  static std::once_flag attr;
  std::call_once(attr, [] {
    SBX_CUDA(cudaFuncSetAttribute(cpqr_push_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(kPushSmemCap)));
  });
  int dev = 0, sms = 148;
  SBX_CUDA(cudaGetDevice(&dev));
  SBX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  static const int min_rows = [] {  // rows per CTA below which a class stops growing its cluster
    const char* e = std::getenv("SBX_PUSH_MINROWS");
    return e ? std::atoi(e) : 32;
  }();
  static const int force_g = [] {  // diagnostics: fixed cluster size
    const char* e = std::getenv("SBX_PUSH_G");
    return e ? std::atoi(e) : 0;
  }();
  // Few problems are spread over more CTAs (shorter per-step work), never
  // past one wave.  The cluster size sets the rank order of every partial
  // sum, so it depends on the batch's multiset of shapes only: problems of
  // one (M, n) class grow together, classes taken tallest first.
  std::map<std::pair<int, int>, std::pair<int, int>, std::greater<std::pair<int, int>>> cls;  // (M, n) -> (count, G)
  i64 ctas = 0;
  for (const auto& j : all) {
    const int g = cpqr_push_cluster(j.M, j.n);
    require(g > 0, "cpqr_push: problem does not fit one cluster");
    auto& c = cls[{j.M, j.n}];
    c.first += 1;
    c.second = g;
    ctas += g;
  }
  for (auto& kv : cls) {
    auto& c = kv.second;
    if (force_g > 0) {
      c.second = std::max(c.second, std::min(force_g, kPMaxG));
      continue;
    }
    while (c.second < kPMaxG && (kv.first.first / (2 * c.second)) >= min_rows &&
           ctas + i64(c.first) * c.second <= sms &&
           push_smem(kv.first.first, kv.first.second, 2 * c.second) <= kPushSmemCap) {
      ctas += i64(c.first) * c.second;
      c.second *= 2;
    }
  }
  std::vector<std::pair<int, QrJob>> sized;
  for (const auto& j : all) sized.push_back({cls[{j.M, j.n}].second, j});
  std::stable_sort(sized.begin(), sized.end(), [](const auto& a, const auto& b) { return a.first > b.first; });
  std::vector<QrJob> jobs;
  for (const auto& sj : sized) jobs.push_back(sj.second);
  static thread_local JobTablePush tab;
  const QrJob* dj = tab.upload(jobs, s);
  for (size_t g0 = 0; g0 < jobs.size();) {
    const int C = sized[g0].first;
    size_t g1 = g0;
    size_t smem = 0;
    while (g1 < jobs.size() && sized[g1].first == C) {
      smem = std::max(smem, push_smem(jobs[g1].M, jobs[g1].n, C));
      ++g1;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned((g1 - g0) * size_t(C)));
    cfg.blockDim = dim3(kPT);
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
    SBX_CUDA(cudaLaunchKernelEx(&cfg, cpqr_push_kernel, jp));
    SBX_LAUNCHED();
    g0 = g1;
  }
}


// ---------------------------------------------------------------- engine 9 host side
namespace {
constexpr int kRRMaxRpt = 32;
int rr_gsz(int n) {
  int g = 32;
  while (g > 1 && g * n > kPT) g >>= 1;
  return g;
}
int rr_rpt(int M, int n, int G) {
  const int ml = (M + G - 1) / G, g = rr_gsz(n);
  return (ml + g - 1) / g;
}
constexpr size_t kRRSmemCap = 200 * 1024;
using RRKernel = void (*)(const QrJob*);
template <int R>
RRKernel rr_kernel_g(int g) {  // gsz
  switch (g) {
    case 2: return cpqr_regrows_kernel<R, 2>;
    case 4: return cpqr_regrows_kernel<R, 4>;
    case 8: return cpqr_regrows_kernel<R, 8>;
    case 16: return cpqr_regrows_kernel<R, 16>;
    default: return cpqr_regrows_kernel<R, 32>;
  }
}
RRKernel rr_kernel(int rpt, int g) {
  switch (rpt) {
    case 8: return rr_kernel_g<8>(g);
    case 12: return rr_kernel_g<12>(g);
    case 16: return rr_kernel_g<16>(g);
    case 24: return rr_kernel_g<24>(g);
    default: return rr_kernel_g<32>(g);
  }
}
int rr_rpt_t(int rpt) { return rpt <= 8 ? 8 : rpt <= 12 ? 12 : rpt <= 16 ? 16 : rpt <= 24 ? 24 : 32; }
}  // namespace

int cpqr_regrows_cluster(int M, int n) {
  if (M <= 0 || n <= 0 || n > 256) return 0;  // at least two lanes per column (keys hold 8-bit positions)
  for (int G = 1; G <= kPMaxG; G <<= 1)
    if (rr_rpt(M, n, G) <= kRRMaxRpt && rr_smem((M + G - 1) / G, n, G) <= kRRSmemCap) return G;
  return 0;
}

void cpqr_regrows_batched(const std::vector<QrJob>& all, cudaStream_t s) {
  if (all.empty()) return;
  static std::once_flag attr;
  std::call_once(attr, [] {
    for (int r : {8, 12, 16, 24, 32})
      for (int g : {2, 4, 8, 16, 32})
        SBX_CUDA(cudaFuncSetAttribute(rr_kernel(r, g), cudaFuncAttributeMaxDynamicSharedMemorySize, int(kRRSmemCap)));
  });
  int dev = 0, sms = 148;
  SBX_CUDA(cudaGetDevice(&dev));
  SBX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  static const int min_rpt = [] {  // rows per thread below which a class stops growing its cluster
    const char* e = std::getenv("SBX_RR_MINRPT");
    return e ? std::atoi(e) : 4;
  }();
  static const int force_g = [] {  // diagnostics: fixed cluster size
    const char* e = std::getenv("SBX_RR_G");
    return e ? std::atoi(e) : 0;
  }();
  // cluster size per (M, n) class (a function of the batch's multiset of
  // shapes only: it sets the rank order of every partial sum)
  std::map<std::pair<int, int>, std::pair<int, int>, std::greater<std::pair<int, int>>> cls;
  i64 ctas = 0;
  for (const auto& j : all) {
    const int g = cpqr_regrows_cluster(j.M, j.n);
    require(g > 0, "cpqr_regrows: problem does not fit one cluster");
    auto& c = cls[{j.M, j.n}];
    c.first += 1;
    c.second = g;
    ctas += g;
  }
  for (auto& kv : cls) {
    auto& c = kv.second;
    const int M = kv.first.first, n = kv.first.second;
    if (force_g > 0) {
      while (c.second < std::min(force_g, kPMaxG) && rr_smem((M + 2 * c.second - 1) / (2 * c.second), n, 2 * c.second) <= kRRSmemCap)
        c.second *= 2;
      continue;
    }
    while (c.second < kPMaxG && rr_rpt(M, n, 2 * c.second) >= min_rpt && ctas + i64(c.first) * c.second <= sms &&
           rr_smem((M + 2 * c.second - 1) / (2 * c.second), n, 2 * c.second) <= kRRSmemCap) {
      ctas += i64(c.first) * c.second;
      c.second *= 2;
    }
  }
  // launch groups: (G, RPT); groups run side by side on forked streams
  std::map<std::pair<int, int>, std::vector<QrJob>, std::greater<std::pair<int, int>>> groups;  // (G, RPT | gsz << 8)
  for (const auto& j : all) {
    const int G = cls[{j.M, j.n}].second;
    groups[{G, rr_rpt_t(rr_rpt(j.M, j.n, G)) | (rr_gsz(j.n) << 8)}].push_back(j);
  }
  std::vector<QrJob> jobs;
  std::vector<std::pair<size_t, size_t>> spans;
  for (const auto& kv : groups) {
    spans.push_back({jobs.size(), jobs.size() + kv.second.size()});
    jobs.insert(jobs.end(), kv.second.begin(), kv.second.end());
  }
  static thread_local JobTablePush tab;
  const QrJob* dj = tab.upload(jobs, s);
  // every (G, RPT, gsz) group launches on its own stream forked from s, so
  // the groups run side by side
  const size_t ng = groups.size();
  std::vector<std::unique_ptr<SideStream>> side;
  for (size_t g = 0; g < ng; ++g) side.emplace_back(new SideStream(s));
  size_t gi = 0;
  for (const auto& kv : groups) {
    const int C = kv.first.first, R = kv.first.second & 0xff;
    const auto sp = spans[gi];
    cudaStream_t st = side[gi]->get();
    size_t smem = 0;
    int threads = 32;
    for (size_t q = sp.first; q < sp.second; ++q) {
      smem = std::max(smem, rr_smem((jobs[q].M + C - 1) / C, jobs[q].n, C));
      threads = std::max(threads, (rr_gsz(jobs[q].n) * jobs[q].n + 31) / 32 * 32);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned((sp.second - sp.first) * size_t(C)));
    cfg.blockDim = dim3(unsigned(threads));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = unsigned(C);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const QrJob* jp = dj + sp.first;
    SBX_CUDA(cudaLaunchKernelEx(&cfg, rr_kernel(R, rr_gsz(jobs[sp.first].n)), jp));
    SBX_LAUNCHED();
    side[gi]->join(s);
    ++gi;
  }
}

}  // namespace sbx
