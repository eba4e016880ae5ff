// HBS inverse / forward apply sweeps on sm_100a (reference hbs.cpp:511-625).
//
// The whole up- and down-sweep is ONE persistent dataflow launch
// (sweep_flow_kernel): every box product D = A*B (+P) is cut into row-tile
// work items taken in tree order, each waiting only for the items that
// produce its inputs, so tree levels overlap instead of meeting at kernel
// boundaries (SBX_SWEEP_LEVELS=1 restores one launch per level):
//   * nrhs == 1 : HBM-bound GEMV (sweep_gemv_kernel).  Factors are read once,
//     coalesced along columns, with 8 independent loads in flight per thread;
//     the input vector segment is staged in shared memory.
//   * nrhs >= 2 : FP64 tensor-core tiles (sweep_dmma_kernel) issuing
//     mma.sync.m8n8k4.f64 (SASS DMMA), operands staged in shared memory.
// The leaf products g*b and d*v that only depend on the input are folded
// into the first (leaf) up-level, so the down-sweep streams e / u only.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "dense.hpp"
#include "hbs.hpp"

#include <type_traits>

namespace sbx {

namespace {

constexpr int kTM = 64;       // rows per work item
constexpr int kThreads = 256;

// ---------------------------------------------------------------- item bodies
// One work item = rows [row0, row0 + kTM) (x one 64-column tile for nrhs > 1)
// of one task's product D = A B (+ P).  Inputs produced inside the same
// launch are read with L2 loads (__ldcg): the producer published them with
// a fence before bumping its completion counter.

// nrhs == 1: HBM-bound GEMV over 64-row items, 4 K-slices per item, 8
// independent loads in flight per thread.  The first batch of the item's
// factor block is loaded BEFORE the dependency wait, so on the critical
// path of the sweep the producers' output and the factor stream overlap.
constexpr int kGR = 64;                // rows per GEMV item (throughput levels)
constexpr int kGRs = 16;               // rows per GEMV item on latency-bound levels

// Rows-per-item GR: 64 rows x 4 K-slices streams the big levels with 8
// loads in flight per thread; 16 rows x 16 K-slices on the short upper
// levels holds a whole K <= 256 item in registers before the dependency
// wait, so the critical path only pays the input-vector fetch.
// One register set serves both shapes (only kGV of the 16 slots are used by
// the 64-row shape), so the kernel holds a single copy.
template <int GR>
struct GemvShape {
  static constexpr int kGS = kThreads / GR;      // K slices
  static constexpr int kGV = 16;                 // columns prefetched per thread
};
struct GemvRegs {
  double av[16];
  int j0, j1;
};

template <int GR>
__device__ __forceinline__ void gemv_prefetch(const double* __restrict__ fac, const SweepTask& t,
                                              int row0, int kb, int ke, GemvRegs& g) {
  constexpr int kGS = GemvShape<GR>::kGS, kGV = GemvShape<GR>::kGV;
  const int r = threadIdx.x % GR, slice = threadIdx.x / GR;
  const int row = row0 + r;
  const int per = (ke - kb + kGS - 1) / kGS;
  g.j0 = kb + slice * per;
  g.j1 = min(ke, g.j0 + per);
  const double* a = fac + t.a_off + row;
#pragma unroll
  for (int q = 0; q < kGV; ++q) {
    const int j = g.j0 + q;
    g.av[q] = (row < t.m && j < g.j1) ? __ldg(a + size_t(j) * t.lda) : 0.0;
  }
}

// partial != null: write the item's partial row sums there instead of the
// final rows (split-K).
template <int GR>
__device__ __forceinline__ void gemv_finish(const double* __restrict__ fac, double* __restrict__ ws,
                                            const SweepTask& t, int row0, int kb, int ke, const GemvRegs& g,
                                            double* sm, double* partial, const SweepDirectIo& io) {
  constexpr int kGS = GemvShape<GR>::kGS, kGV = GemvShape<GR>::kGV;
  const int K = t.K;
  double* xs = sm;                    // K doubles
  double* red = sm + ((K + 1) & ~1);  // kThreads partial sums
  const int r = threadIdx.x % GR, slice = threadIdx.x / GR;
  const int row = row0 + r;
  // the P row is fetched together with the input vector (one round trip on
  // the critical path instead of two)
  const double pv = (slice == 0 && row < t.m && t.p_row >= 0 && !partial) ? __ldcg(ws + t.p_row + row) : 0.0;
  {
    // the caller's vector stands in for the workspace's input region
    const bool direct = io.in && t.b_row >= io.in_row && t.b_row < io.in_row + io.n;
    const double* xsrc = direct ? io.in + (t.b_row - io.in_row) : ws + t.b_row;
    for (int j = kb + threadIdx.x; j < ke; j += kThreads) xs[j] = __ldcg(xsrc + j);
  }
  __syncthreads();
  double acc = 0.0, acc1 = 0.0;
#pragma unroll
  for (int q = 0; q < kGV; q += 2) {
    const int j = g.j0 + q;
    if (j < g.j1) acc = fma(g.av[q], xs[j], acc);
    if (j + 1 < g.j1) acc1 = fma(g.av[q + 1], xs[j + 1], acc1);
  }
  if (row < t.m) {
    const double* a = fac + t.a_off + row;
    int j = g.j0 + kGV;
    for (; j + 16 <= g.j1; j += 16) {  // 16 loads in flight per thread
      double v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = __ldg(a + size_t(j + q) * t.lda);
#pragma unroll
      for (int q = 0; q < 16; q += 2) {
        acc = fma(v[q], xs[j + q], acc);
        acc1 = fma(v[q + 1], xs[j + q + 1], acc1);
      }
    }
    for (; j + 8 <= g.j1; j += 8) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = __ldg(a + size_t(j + q) * t.lda);
#pragma unroll
      for (int q = 0; q < 8; q += 2) {
        acc = fma(v[q], xs[j + q], acc);
        acc1 = fma(v[q + 1], xs[j + q + 1], acc1);
      }
    }
    for (; j < g.j1; ++j) acc = fma(__ldg(a + size_t(j) * t.lda), xs[j], acc);
  }
  red[threadIdx.x] = acc + acc1;
  __syncthreads();
  if (slice == 0 && row < t.m) {
    double s = red[r];
#pragma unroll
    for (int q = 1; q < kGS; ++q) s += red[r + q * GR];
    if (partial) {
      partial[r] = s;
      return;
    }
    if (t.p_row >= 0) s += pv;
    const i64 dst = row < t.split ? t.d1_row + row : t.d2_row + (row - t.split);
    if (io.out && dst >= io.out_row && dst < io.out_row + io.n)
      io.out[dst - io.out_row] = s;
    else
      ws[dst] = s;
  }
}

// nrhs >= 2: C tile 64 x 64 on FP64 tensor cores (mma.sync.m8n8k4.f64 ->
// SASS DMMA), 8 warps with 16 x 32 warp tiles.  K moves through a 4-stage
// cp.async pipeline: A (read-only factors, 8-byte .ca copies: factor
// columns need not be 16-byte aligned) and B (workspace rows produced by
// other CTAs of the launch: 16-byte .cg copies that bypass L1, whose lines
// could hold stale neighbours of a just-published row).
#ifndef SBX_DMMA_KC
#define SBX_DMMA_KC 16
#endif
#ifndef SBX_DMMA_STAGES
#define SBX_DMMA_STAGES 4
#endif
constexpr int kKC = SBX_DMMA_KC;
constexpr int kStages = SBX_DMMA_STAGES;
constexpr int kPad = 8;  // row stride 72 doubles

// TN: columns per tile (64, or 32 to halve the work per item on the
// latency-bound upper levels of the tree)
template <int TN>
struct DmmaSmem {
  double As[kStages][kKC][kTM + kPad];
  double Bs[kStages][kKC][TN + kPad];
};

__device__ __forceinline__ void dmma_m8n8k4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool pred) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const int sz = pred ? 8 : 0;  // zero-fill when out of range
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(sz));
}
__device__ __forceinline__ void cp_async16_cg(double* dst, const double* src, int bytes) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int TN, int TM = kTM>
__device__ __forceinline__ void dmma_issue_a(const double* __restrict__ fac, const SweepTask& t, int row0,
                                             int stage, int k0, int ke, DmmaSmem<TN>& S) {
  const double* A = fac + t.a_off;
  static_assert((TM * kKC) % kThreads == 0, "A chunk split");
#pragma unroll
  for (int q = 0; q < TM * kKC / kThreads; ++q) {
    const int idx = threadIdx.x + q * kThreads;  // TM x kKC
    const int kk = idx / TM, rr = idx % TM;
    const int grow = row0 + rr, gk = k0 + kk;
    const bool pa = grow < t.m && gk < ke;
    cp_async8(&S.As[stage][kk][rr], pa ? A + grow + size_t(gk) * t.lda : A, pa);
  }
}

template <int TN>
__device__ __forceinline__ void dmma_issue_b(const double* __restrict__ ws, const SweepTask& t, int col0,
                                             int nrhs, int ldw, int stage, int k0, int ke, DmmaSmem<TN>& S) {
  const double* B = ws + t.b_row * ldw;
  constexpr int kPairs = TN / 2;  // 16-byte pairs per B row
  static_assert((kKC * kPairs) % kThreads == 0, "B chunk split");
#pragma unroll
  for (int q = 0; q < kKC * kPairs / kThreads; ++q) {
    const int idx = threadIdx.x + q * kThreads;  // kKC rows x kPairs pairs
    const int kk = idx / kPairs, pr = (idx % kPairs) * 2;
    const int gk = k0 + kk, gcol = col0 + pr;
    int bytes = 0;
    if (gk < ke) bytes = gcol + 1 < nrhs ? 16 : (gcol < nrhs ? 8 : 0);
    cp_async16_cg(&S.Bs[stage][kk][pr], bytes ? B + size_t(gk) * ldw + gcol : B, bytes);
  }
}

// Issues the A parts of the first kStages-1 chunks (call before waiting on
// the producers of B); they join the first commit group.
template <int TN, int TM = kTM>
__device__ __forceinline__ void dmma_prefetch(const double* __restrict__ fac, const SweepTask& t, int row0,
                                              int kb, int ke, DmmaSmem<TN>& S) {
  const int nchunks = (ke - kb + kKC - 1) / kKC;
#pragma unroll
  for (int c = 0; c < kStages - 1; ++c)
    if (c < nchunks) dmma_issue_a<TN, TM>(fac, t, row0, c, kb + c * kKC, ke, S);
}

// partial != null: write the raw 64 x 64 tile there (row-major) instead of
// the final rows (split-K).
template <int TN, int TM = kTM>
__device__ __forceinline__ void dmma_item(const double* __restrict__ fac, double* __restrict__ ws,
                                          const SweepTask& t, int row0, int col0, int nrhs, int ldw,
                                          int kb, int ke, DmmaSmem<TN>& S, double* partial) {
  constexpr int RG = TM / 16;      // warp row groups (16 rows each)
  constexpr int CG = 8 / RG;       // warp column groups
  constexpr int NB = TN / CG / 8;  // 8-column blocks per warp
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int wm = (warp % RG) * 16;
  const int wn = (warp / RG) * (TN / CG);
  double c[2][NB][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < NB; ++b) c[a][b][0] = c[a][b][1] = 0.0;
  const int nchunks = (ke - kb + kKC - 1) / kKC;
  // the P block (produced long before, by the up-sweep) is loaded now so its
  // latency hides behind the K loop
  double pv[2][NB][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int row = row0 + wm + a * 8 + gid, col = col0 + wn + b * 8 + 2 * tig;
      const bool ok = !partial && t.p_row >= 0 && row < t.m;
      pv[a][b][0] = ok && col < nrhs ? __ldcg(ws + (t.p_row + row) * ldw + col) : 0.0;
      pv[a][b][1] = ok && col + 1 < nrhs ? __ldcg(ws + (t.p_row + row) * ldw + col + 1) : 0.0;
    }
#pragma unroll
  for (int ch = 0; ch < kStages - 1; ++ch) {  // B of the prologue chunks (A already issued)
    if (ch < nchunks) dmma_issue_b(ws, t, col0, nrhs, ldw, ch, kb + ch * kKC, ke, S);
    cp_async_commit();
  }
  for (int ch = 0; ch < nchunks; ++ch) {
    const int st = ch % kStages;
    cp_async_wait<kStages - 2>();
    __syncthreads();  // chunk ch visible; stage (ch-1) % kStages is free
    const int nx = ch + kStages - 1;
    if (nx < nchunks) {
      dmma_issue_a<TN, TM>(fac, t, row0, nx % kStages, kb + nx * kKC, ke, S);
      dmma_issue_b(ws, t, col0, nrhs, ldw, nx % kStages, kb + nx * kKC, ke, S);
    }
    cp_async_commit();
#pragma unroll
    for (int k4 = 0; k4 < kKC; k4 += 4) {
      double af[2], bf[NB];
#pragma unroll
      for (int a = 0; a < 2; ++a) af[a] = S.As[st][k4 + tig][wm + a * 8 + gid];
#pragma unroll
      for (int b = 0; b < NB; ++b) bf[b] = S.Bs[st][k4 + tig][wn + b * 8 + gid];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < NB; ++b) dmma_m8n8k4(c[a][b][0], c[a][b][1], af[a], bf[b]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // smem free for the next item
  if (partial) {
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int r = wm + a * 8 + gid, cc = wn + b * 8 + 2 * tig;
        partial[r * TN + cc] = c[a][b][0];
        partial[r * TN + cc + 1] = c[a][b][1];
      }
    return;
  }
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int row = row0 + wm + a * 8 + gid;
    if (row >= t.m) continue;
    const i64 dst = row < t.split ? t.d1_row + row : t.d2_row + (row - t.split);
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int col = col0 + wn + b * 8 + 2 * tig;
      double v0 = c[a][b][0], v1 = c[a][b][1];
      if (t.p_row >= 0) {
        v0 += pv[a][b][0];
        v1 += pv[a][b][1];
      }
      if (col < nrhs) ws[dst * ldw + col] = v0;
      if (col + 1 < nrhs) ws[dst * ldw + col + 1] = v1;
    }
  }
}

// ---------------------------------------------------------------- dataflow sweep
// The whole up/down sweep is ONE persistent launch.  CTAs take work items
// in plan order from a ticket counter; an item first waits until every item
// of the tasks it reads from (same column tile) has completed, then computes
// and publishes (fence + counter bump).  Items are taken in dependency order
// and a CTA only waits after taking a ticket, so every awaited item is held
// by a running CTA: no deadlock, and levels overlap instead of meeting at
// kernel boundaries.
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <bool kDmma, int TN>
__global__ void __launch_bounds__(kThreads, kDmma ? 3 : 4)
    sweep_flow_kernel(const double* __restrict__ fac, double* __restrict__ ws,
                      const SweepTask* __restrict__ tasks, const FlowItem* __restrict__ items,
                      int n_items, int* __restrict__ counters, int ncol, int nrhs, int ldw,
                      double* __restrict__ partials, int* __restrict__ tile_cnt,
                      unsigned long long* __restrict__ trace, const ItemDesc* __restrict__ descs,
                      SweepDirectIo io, int ncount) {
  extern __shared__ __align__(16) double dsm[];
  __shared__ int s_last;
  __shared__ __align__(16) ItemDesc sdesc[2];
  constexpr int tile_elems = kDmma ? kTM * TN : kGR;
  constexpr int kDescChunks = int(sizeof(ItemDesc) / 16);
  static_assert(sizeof(ItemDesc) % 16 == 0, "descriptor copies are 16-byte chunks");
  // Static round-robin schedule: CTA b takes items b, b + G, ...  Items are
  // in dependency order, a CTA waits only on items that precede its own and
  // every CTA is resident, so the lowest unfinished item always has its
  // producers done and its CTA working on it (no deadlock).  The descriptor
  // of the next item is fetched asynchronously while the current one
  // computes (no ticket atomics, no dependent descriptor loads).
  const int G = int(gridDim.x);
  if (threadIdx.x < kDescChunks && int(blockIdx.x) < n_items)
    cp_async16_cg(reinterpret_cast<double*>(&sdesc[0]) + 2 * threadIdx.x,
                  reinterpret_cast<const double*>(descs + blockIdx.x) + 2 * threadIdx.x, 16);
  cp_async_commit();
  for (int r = 0, idx = int(blockIdx.x);; ++r, idx += G) {
    cp_async_wait<0>();
    __syncthreads();
    if (idx >= n_items) break;
    if (threadIdx.x < kDescChunks && idx + G < n_items)
      cp_async16_cg(reinterpret_cast<double*>(&sdesc[(r + 1) & 1]) + 2 * threadIdx.x,
                    reinterpret_cast<const double*>(descs + idx + G) + 2 * threadIdx.x, 16);
    cp_async_commit();
    unsigned long long t0 = 0, t1 = 0;
    if (trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    const ItemDesc& D = sdesc[r & 1];
    // DMMA items keep the descriptor in registers (their K loop reads it per
    // chunk); GEMV items read it from shared memory on use
    using ItT = std::conditional_t<kDmma, const FlowItem, const FlowItem&>;
    using TaskT = std::conditional_t<kDmma, const SweepTask, const SweepTask&>;
    ItT it = D.it;
    TaskT t = D.t;
    GemvRegs g;
    const bool small = it.tile != (kDmma ? kTM : kGR);
    if constexpr (kDmma) {
      if (small)
        dmma_prefetch<TN, 32>(fac, t, it.row0, it.kb, it.ke, *reinterpret_cast<DmmaSmem<TN>*>(dsm));
      else
        dmma_prefetch<TN>(fac, t, it.row0, it.kb, it.ke, *reinterpret_cast<DmmaSmem<TN>*>(dsm));
    } else if (small)
      gemv_prefetch<kGRs>(fac, t, it.row0, it.kb, it.ke, g);
    else
      gemv_prefetch<kGR>(fac, t, it.row0, it.kb, it.ke, g);
    if (threadIdx.x < D.t.ndep) {  // from the shared descriptor (dynamic index)
      const int d = D.t.dep[threadIdx.x];
      const int need = D.need[threadIdx.x];
      const int* p = counters + 1 + d * ncol + it.ct;
      while (ld_acquire(p) < need) __nanosleep(32);
    }
    __syncthreads();
    if (trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    double* part = it.nsplit > 1 ? partials + it.poff + i64(it.ks) * tile_elems : nullptr;
    if constexpr (kDmma) {
      if (small)
        dmma_item<TN, 32>(fac, ws, t, it.row0, it.ct * TN, nrhs, ldw, it.kb, it.ke,
                          *reinterpret_cast<DmmaSmem<TN>*>(dsm), part);
      else
        dmma_item<TN>(fac, ws, t, it.row0, it.ct * TN, nrhs, ldw, it.kb, it.ke,
                      *reinterpret_cast<DmmaSmem<TN>*>(dsm), part);
    }
    else if (small)
      gemv_finish<kGRs>(fac, ws, t, it.row0, it.kb, it.ke, g, dsm, part, io);
    else
      gemv_finish<kGR>(fac, ws, t, it.row0, it.kb, it.ke, g, dsm, part, io);
    __syncthreads();  // the item's stores happen-before thread 0's release below
    bool done = true;
    if (it.nsplit > 1) {  // last split of the tile reduces the partials in split order
      if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(tile_cnt + it.cidx, 1) == it.nsplit - 1;
      }
      __syncthreads();
      done = s_last != 0;
      if (done) {
        __threadfence();
        const double* pb = partials + it.poff;
        if constexpr (kDmma) {
          for (int e = threadIdx.x; e < it.tile * TN; e += kThreads) {
            const int r = e / TN, cc = e % TN;
            const int row = it.row0 + r, col = it.ct * TN + cc;
            if (row >= t.m || col >= nrhs) continue;
            double v = 0.0;
            for (int q = 0; q < it.nsplit; ++q) v += __ldcg(pb + i64(q) * tile_elems + e);
            if (t.p_row >= 0) v += __ldcg(ws + (t.p_row + row) * ldw + col);
            const i64 dst = row < t.split ? t.d1_row + row : t.d2_row + (row - t.split);
            ws[dst * ldw + col] = v;
          }
        } else {
          for (int r = threadIdx.x; r < it.tile; r += kThreads) {
            const int row = it.row0 + r;
            if (row >= t.m) continue;
            double v = 0.0;
            for (int q = 0; q < it.nsplit; ++q) v += __ldcg(pb + i64(q) * tile_elems + r);
            if (t.p_row >= 0) v += __ldcg(ws + t.p_row + row);
            const i64 dst = row < t.split ? t.d1_row + row : t.d2_row + (row - t.split);
            if (io.out && dst >= io.out_row && dst < io.out_row + io.n)
              io.out[dst - io.out_row] = v;
            else
              ws[dst] = v;
          }
        }
        __syncthreads();
      }
    }
    if (threadIdx.x == 0) {
      if (done) {
        __threadfence();  // cumulative: covers every thread's stores ordered by the barrier
        atomicAdd(counters + 1 + it.task * ncol + it.ct, 1);
      }
      if (trace) {
        unsigned long long t2;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2));
        trace[4 * idx] = t0;
        trace[4 * idx + 1] = t1;
        trace[4 * idx + 2] = t2;
        trace[4 * idx + 3] = blockIdx.x;
      }
    }
  }
  // The last CTA out zeroes the counters for the next launch on this stream's
  // scratch (every other CTA has passed its last wait): no memset per call.
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(counters, 1) == G - 1;
  }
  __syncthreads();
  if (s_last)
    for (int i = threadIdx.x; i < ncount; i += kThreads) counters[i] = 0;
}

// Per-level launches (diagnostic path, SBX_SWEEP_LEVELS=1).
__global__ void __launch_bounds__(kThreads)
    sweep_gemv_kernel(const double* __restrict__ fac, double* __restrict__ ws,
                      const SweepTask* __restrict__ tasks, const FlowItem* __restrict__ items) {
  extern __shared__ __align__(16) double dsm[];
  const FlowItem f = items[blockIdx.x];
  const int4 it = make_int4(f.task, f.row0, f.ct, 0);
  const SweepTask t = tasks[it.x];
  GemvRegs g;
  gemv_prefetch<kGR>(fac, t, it.y, 0, t.K, g);
  gemv_finish<kGR>(fac, ws, t, it.y, 0, t.K, g, dsm, nullptr, SweepDirectIo{});
}

template <int TN>
__global__ void __launch_bounds__(kThreads)
    sweep_dmma_kernel(const double* __restrict__ fac, double* __restrict__ ws,
                      const SweepTask* __restrict__ tasks, const FlowItem* __restrict__ items,
                      int nrhs, int ldw) {
  extern __shared__ __align__(16) double dsm[];
  const FlowItem f = items[blockIdx.x];
  const int4 it = make_int4(f.task, f.row0, f.ct, 0);
  const SweepTask t = tasks[it.x];
  DmmaSmem<TN>& S = *reinterpret_cast<DmmaSmem<TN>*>(dsm);
  dmma_prefetch<TN>(fac, t, it.y, 0, t.K, S);
  dmma_item<TN>(fac, ws, t, it.y, it.z * TN, nrhs, ldw, 0, t.K, S, nullptr);
}

// ---------------------------------------------------------------- layout moves
// Layout conversions between the caller's column-major blocks and the
// row-major sweep workspace (RHS fastest), with an optional row map.  Blocks
// of several RHS go through 32 x 32 shared-memory tiles, so the column-major
// side moves along its rows and the row-major side along its RHS (both
// coalesced, no 64-bit index divisions); a single RHS is a plain (gathered)
// copy.
template <bool kToRm>
__global__ void __launch_bounds__(256) transpose_tiles_kernel(const double* __restrict__ src, i64 lds,
                                                              double* __restrict__ dst, i64 ldd, i64 n, i64 nrhs,
                                                              const i64* __restrict__ map) {
  __shared__ double t[32][33];
  const i64 i0 = i64(blockIdx.x) * 32, c0 = i64(blockIdx.y) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  if (kToRm) {  // src column-major (i, c); dst row map(i), column c
#pragma unroll
    for (int k = ty; k < 32; k += 8) {
      const i64 c = c0 + k, i = i0 + tx;
      if (i < n && c < nrhs) t[k][tx] = src[i + c * lds];
    }
    __syncthreads();
#pragma unroll
    for (int k = ty; k < 32; k += 8) {
      const i64 i = i0 + k, c = c0 + tx;
      if (i < n && c < nrhs) dst[(map ? map[i] : i) * ldd + c] = t[tx][k];
    }
  } else {  // src row map(i), column c; dst column-major (i, c)
#pragma unroll
    for (int k = ty; k < 32; k += 8) {
      const i64 i = i0 + k, c = c0 + tx;
      if (i < n && c < nrhs) t[k][tx] = src[(map ? map[i] : i) * lds + c];
    }
    __syncthreads();
#pragma unroll
    for (int k = ty; k < 32; k += 8) {
      const i64 c = c0 + k, i = i0 + tx;
      if (i < n && c < nrhs) dst[i + c * ldd] = t[tx][k];
    }
  }
}

template <bool kToRm>
__global__ void copy_rows_kernel(const double* __restrict__ src, i64 lds, double* __restrict__ dst, i64 ldd, i64 n,
                                 const i64* __restrict__ map) {
  for (i64 i = blockIdx.x * i64(blockDim.x) + threadIdx.x; i < n; i += i64(gridDim.x) * blockDim.x) {
    const i64 r = map ? map[i] : i;
    if (kToRm) dst[r * ldd] = src[i];
    else dst[i] = src[r * lds];
  }
}

int grid_for(i64 total) {
  return int(std::min<i64>((total + 255) / 256, 148 * 16));
}

}  // namespace

void launch_cm_to_rm(const double* src, i64 ld, i64 n, i64 nrhs, double* dst, i64 ldw, const i64* map,
                     cudaStream_t s) {
  if (n * nrhs == 0) return;
  if (nrhs == 1)
    copy_rows_kernel<true><<<grid_for(n), 256, 0, s>>>(src, ld, dst, ldw, n, map);
  else
    transpose_tiles_kernel<true><<<dim3(unsigned((n + 31) / 32), unsigned((nrhs + 31) / 32)), 256, 0, s>>>(
        src, ld, dst, ldw, n, nrhs, map);
  SBX_LAUNCHED();
}

void launch_rm_to_cm(const double* src, i64 ldw, i64 n, i64 nrhs, double* dst, i64 ld, const i64* map,
                     cudaStream_t s) {
  if (n * nrhs == 0) return;
  if (nrhs == 1)
    copy_rows_kernel<false><<<grid_for(n), 256, 0, s>>>(src, ldw, dst, ld, n, map);
  else
    transpose_tiles_kernel<false><<<dim3(unsigned((n + 31) / 32), unsigned((nrhs + 31) / 32)), 256, 0, s>>>(
        src, ldw, dst, ld, n, nrhs, map);
  SBX_LAUNCHED();
}

namespace {

// Work items in level order; per level: column tile, then task, then row
// tile, then K split.  Levels with too few tiles to fill the GPU split K so
// the short upper levels of the tree (the sweep's critical path) spread
// over more CTAs.  Returns per-level [first, count).
std::vector<FlowItem> make_items(SweepPlan& plan, int tile0, int ncol, int tile_elems, int target,
                                 std::vector<int2>* ranges, i64* partial_elems, int* n_tile_cnt,
                                 std::vector<int>* needs, int small_tile, i64 small_below, int kcap) {
  std::vector<FlowItem> fi;
  needs->assign(size_t(plan.n_tasks), 0);
  i64 poff = 0;
  int cidx = 0;
  for (auto& L : plan.levels) {
    const i64 first = i64(fi.size());
    i64 base = 0;
    for (const auto& tk : L.tasks) base += (tk.m + tile0 - 1) / tile0;
    base *= ncol;
    // short levels (the tree's critical path) take smaller row tiles; a
    // level with a forced K split (the collapsed top) is cut into K chunks
    // of at most kcap (a GEMV item then holds its whole block in registers
    // before the dependency wait)
    const int tile = L.ksplit > 0 ? (kcap > 128 && small_tile > 0 ? small_tile : tile0)
                     : (small_tile > 0 && base < small_below) ? small_tile : tile0;
    const int lsplit_ok = tile == tile0;
    const int lsplit = L.ksplit > 0 ? int((L.max_k + kcap - 1) / kcap)
                       : lsplit_ok && target > 0 && base > 0 ? int(std::min<i64>(8, (target + base - 1) / base))
                                                               : 1;
    // (column tiles innermost: the items reading the same factor rows run
    // side by side, so the second column tile finds them in L2)
    for (size_t t = 0; t < L.tasks.size(); ++t)
      for (int r0 = 0; r0 < L.tasks[t].m; r0 += tile)
        for (int ct = 0; ct < ncol; ++ct) {
        const auto& tk = L.tasks[t];
        const int ns = L.ksplit > 0 ? lsplit : std::max(1, std::min(lsplit, tk.K / 32));
        // split boundaries on multiples of 16 (the DMMA K chunk)
        const int per = ((tk.K + ns - 1) / ns + 15) / 16 * 16;
        const int nsplit = std::max(1, (tk.K + per - 1) / std::max(per, 1));
        (*needs)[size_t(L.first_task + i64(t))] = (tk.m + tile - 1) / tile;
        {
          for (int ks = 0; ks < nsplit; ++ks) {
            FlowItem f{};
            f.task = int(L.first_task + i64(t));
            f.row0 = r0;
            f.ct = ct;
            f.ks = ks;
            f.nsplit = nsplit;
            f.kb = ks * per;
            f.ke = std::min(tk.K, (ks + 1) * per);
            f.cidx = nsplit > 1 ? cidx : -1;
            f.poff = nsplit > 1 ? poff : 0;
            f.tile = tile;
            fi.push_back(f);
          }
          if (nsplit > 1) {
            ++cidx;
            poff += i64(nsplit) * tile_elems;
          }
        }
      }
    if (ranges) ranges->push_back(make_int2(int(first), int(i64(fi.size()) - first)));
  }
  *partial_elems = poff;
  *n_tile_cnt = cidx;
  return fi;
}

// Dependencies of the dataflow sweep: every workspace row is written by
// exactly one task per sweep; a task depends on the writers of the rows it
// reads (its B rows and its P rows).  Rows written before the launch (the
// input region) have no writer.
void finalize(SweepPlan& plan) {
  std::vector<SweepTask> all;
  for (auto& L : plan.levels) {
    L.first_task = i64(all.size());
    for (const auto& tk : L.tasks) L.max_k = std::max(L.max_k, tk.K);
    all.insert(all.end(), L.tasks.begin(), L.tasks.end());
  }
  std::vector<int> writer(size_t(plan.ws_rows), -1);
  for (size_t ti = 0; ti < all.size(); ++ti) {
    auto& t = all[ti];
    t.ndep = 0;
    auto add_reads = [&](i64 r0, i64 nr) {
      for (i64 r = r0; r < r0 + nr; ++r) {
        const int w = writer[size_t(r)];
        if (w < 0) continue;
        bool seen = false;
        for (int q = 0; q < t.ndep; ++q) seen |= t.dep[q] == w;
        if (seen) continue;
        require(t.ndep < kMaxDep, "sweep plan: task reads from too many producers");
        t.dep[t.ndep++] = w;
      }
    };
    add_reads(t.b_row, t.K);
    if (t.p_row >= 0) add_reads(t.p_row, t.m);
    for (int r = 0; r < t.m; ++r) {
      const i64 dst = r < t.split ? t.d1_row + r : t.d2_row + (r - t.split);
      writer[size_t(dst)] = int(ti);
    }
  }
  plan.n_tasks = int(all.size());
  plan.flows.clear();
  const cudaStream_t st = cur_stream();
  plan.d_tasks.upload(all, st);
  plan.h_tasks = all;
  SBX_CUDA(cudaStreamSynchronize(st));
  plan.built = true;
}

SweepTask mk(i64 a_off, i64 lda, i64 m, i64 K, i64 b_row, i64 p_row, i64 d1, i64 d2, i64 split) {
  SweepTask t;
  t.a_off = a_off;
  t.lda = int(std::max<i64>(lda, 1));
  t.m = int(m);
  t.K = int(K);
  t.b_row = b_row;
  t.p_row = p_row;
  t.d1_row = d1;
  t.d2_row = d2;
  t.split = int(split);
  t.ndep = 0;
  for (int& d : t.dep) d = -1;
  return t;
}

}  // namespace

namespace {
// Workspace rows of the solve: IN, OUT, HAT (k_i), PP (c_i), INC (k_i).
struct SolveLayout {
  std::vector<i64> hat, pp, inc;
  i64 in_row = 0, out_row = 0, ws_rows = 0;
};

SolveLayout solve_layout(const HbsOp& op) {
  const size_t nn = op.nodes.size();
  SolveLayout Y;
  Y.hat.assign(nn, 0);
  Y.pp.assign(nn, 0);
  Y.inc.assign(nn, 0);
  i64 row = 0;
  Y.in_row = row;
  row += op.n;
  Y.out_row = row;
  row += op.n;
  for (size_t i = 1; i < nn; ++i) {
    Y.hat[i] = row;
    row += op.nodes[i].k;
  }
  for (size_t i = 1; i < nn; ++i) {
    Y.pp[i] = row;
    row += op.nodes[i].c;
  }
  for (size_t i = 1; i < nn; ++i) {
    Y.inc[i] = row;
    row += op.nodes[i].k;
  }
  Y.ws_rows = row;
  return Y;
}

// Solve tasks: up-sweep of the nodes in up_sel (deepest level first), the
// root product when `root`, down-sweep of the nodes in down_sel.
void build_solve_tasks(const HbsOp& op, const SolveLayout& Y, const std::vector<char>& up_sel, bool root,
                       const std::vector<char>& down_sel, SweepPlan& P, int top = 0) {
  P.levels.clear();
  P.in_row = Y.in_row;
  P.out_row = Y.out_row;
  P.ws_rows = Y.ws_rows;
  const size_t nn = op.nodes.size();
  if (nn == 1) {  // single leaf: x = root_g b (hbs.cpp:592)
    if (root) {
      SweepLevel L;
      const i64 c = op.nodes[0].c;
      L.tasks.push_back(mk(op.o_root_g, c, c, c, Y.in_row, -1, Y.out_row, 0, c));
      P.levels.push_back(std::move(L));
    }
    finalize(P);
    return;
  }
  for (int d = op.max_depth; d >= std::max(top, 1); --d) {  // up
    SweepLevel L;
    for (size_t i = 1; i < nn; ++i) {
      const auto& nd = op.nodes[i];
      if (nd.depth != d || !up_sel[i]) continue;
      const i64 b = nd.is_leaf() ? Y.in_row + 2 * nd.begin : Y.hat[size_t(nd.left)];
      L.tasks.push_back(mk(nd.o_fg, nd.k + nd.c, nd.k + nd.c, nd.c, b, -1, Y.hat[i], Y.pp[i], nd.k));
    }
    if (!L.tasks.empty()) P.levels.push_back(std::move(L));
  }
  if (root && top > 0) {  // collapsed top: inc(depth-top boxes) = T * hat(depth-top boxes)
    size_t first = 0;
    while (op.nodes[first].depth != top) ++first;
    SweepLevel L;
    const i64 K = op.top_K;
    L.tasks.push_back(mk(op.o_top, K, K, K, Y.hat[first], -1, Y.inc[first], 0, K));
    L.ksplit = int(std::min<i64>(8, std::max<i64>(1, (K + 127) / 128)));
    P.levels.push_back(std::move(L));
  } else if (root) {
    SweepLevel L;
    const auto& nd = op.nodes[0];
    L.tasks.push_back(mk(op.o_root_g, nd.c, nd.c, nd.c, Y.hat[size_t(nd.left)], -1, Y.inc[size_t(nd.left)], 0,
                         nd.c));
    P.levels.push_back(std::move(L));
  }
  for (int d = std::max(top, 1); d <= op.max_depth; ++d) {  // down
    SweepLevel L;
    for (size_t i = 1; i < nn; ++i) {
      const auto& nd = op.nodes[i];
      if (nd.depth != d || !down_sel[i]) continue;
      const i64 dst = nd.is_leaf() ? Y.out_row + 2 * nd.begin : Y.inc[size_t(nd.left)];
      L.tasks.push_back(mk(nd.o_e, nd.c, nd.c, nd.k, Y.inc[i], Y.pp[i], dst, 0, nd.c));
    }
    if (!L.tasks.empty()) P.levels.push_back(std::move(L));
  }
  finalize(P);
}
}  // namespace

namespace {
// Depth at which the solve's top collapses (0: none).  Every box above it
// must be internal, the depth-L boxes feed one task (2^L <= kMaxDep
// producers) and the dense map stays small next to the factors.
int choose_top(const HbsOp& op) {
  static const int env = [] {
    const char* e = std::getenv("SBX_SWEEP_TOP");  // depth, 0 disables
    return e ? std::atoi(e) : -1;
  }();
  static const i64 kmax = [] {
    const char* e = std::getenv("SBX_SWEEP_TOP_KMAX");
    return e ? std::atoll(e) : 1280;
  }();
  if (op.nodes.size() < 3 || env == 0) return 0;
  int min_leaf = 1 << 30;
  for (const auto& nd : op.nodes)
    if (nd.is_leaf()) min_leaf = std::min(min_leaf, nd.depth);
  if (env < 0 && op.max_depth < 7) return 0;  // shallow trees: few levels to save
  static const double min_rcond = [] {
    const char* e = std::getenv("SBX_SWEEP_TOP_RCOND");
    return e ? std::atof(e) : 1e-6;
  }();
  static const bool log = std::getenv("SBX_SWEEP_TOP_LOG") != nullptr;  // diagnostics
  if (log && op.node_rcond.size() == op.nodes.size()) {
    std::vector<double> mn(size_t(op.max_depth + 1), 1.0);
    for (size_t i = 0; i < op.nodes.size(); ++i)
      mn[size_t(op.nodes[i].depth)] = std::min(mn[size_t(op.nodes[i].depth)], op.node_rcond[i]);
    std::fprintf(stderr, "[sbx-top] n=%lld min rcond by depth:", (long long)op.n);
    for (double r : mn) std::fprintf(stderr, " %.1e", r);
    std::fprintf(stderr, "\n");
  }
  int best = 0;
  for (int L = 2; L < min_leaf && (1 << L) <= kMaxDep; ++L) {
    if (env < 0) {  // every block above depth L must be well conditioned (and known)
      bool ok = op.node_rcond.size() == op.nodes.size();
      for (size_t i = 0; ok && i < op.nodes.size(); ++i)
        if (op.nodes[i].depth < L && !(op.node_rcond[i] >= min_rcond)) ok = false;
      if (!ok) break;
    }
    i64 K = 0;
    for (const auto& nd : op.nodes)
      if (nd.depth == L) K += nd.k;
    if (env > 0) {
      if (L == env) best = L;
      continue;
    }
    if (K <= kmax) best = L;
  }
  return best;
}

// T_L by the recursion over the top levels (d = 1 .. L-1):
//   M_1 = root_g,  M_{d+1} = blockdiag(e_p) M_d blockdiag(f_p) + blockdiag(g_p)
// over the depth-d boxes p in BFS order (their children are the depth-(d+1)
// boxes, in order), which is the map the up-sweep, root product and
// down-sweep of those levels apply to the stacked depth-(d+1) hats.  The
// transposed solve sees M^T (same recursion over the transposed factors).
void hbs_build_top(HbsOp& op, int L, cudaStream_t s) {
  std::vector<std::vector<size_t>> lev(size_t(L + 1));
  for (size_t i = 0; i < op.nodes.size(); ++i)
    if (op.nodes[i].depth <= L) lev[size_t(op.nodes[i].depth)].push_back(i);
  auto ksum = [&](int d) {
    i64 K = 0;
    for (size_t i : lev[size_t(d)]) K += op.nodes[i].k;
    return K;
  };
  const double* A = op.arena.get();
  i64 Kd = op.nodes[0].c;
  DevBuf<double> M(static_cast<size_t>(Kd * Kd));
  SBX_CUDA(cudaMemcpyAsync(M.get(), A + op.o_root_g, size_t(Kd * Kd) * 8, cudaMemcpyDeviceToDevice, s));
  for (int d = 1; d < L; ++d) {
    const i64 Kn = ksum(d + 1);
    DevBuf<double> Z(static_cast<size_t>(Kd * Kn)), Mn(static_cast<size_t>(Kn * Kn));
    SBX_CUDA(cudaMemsetAsync(Mn.get(), 0, size_t(Kn * Kn) * 8, s));
    std::vector<GemmJob> zj, ej;
    std::vector<CopyJob> gj;
    i64 ko = 0, co = 0;
    for (size_t i : lev[size_t(d)]) {
      const auto& p = op.nodes[i];
      const int k = int(p.k), c = int(p.c);
      if (k > 0) {
        zj.push_back({M.get() + ko * Kd, A + p.o_fg, Z.get() + co * Kd, int(Kd), c, k, int(Kd), k + c, int(Kd), 0, 0,
                      1.0, 0.0});
        ej.push_back({A + p.o_e, Z.get() + ko, Mn.get() + co, c, int(Kn), k, c, int(Kd), int(Kn), 0, 0, 1.0, 1.0});
      }
      gj.push_back({A + p.o_fg + k, Mn.get() + co + co * Kn, c, c, k + c, int(Kn), 0, 0});
      ko += k;
      co += c;
    }
    require(ko == Kd && co == Kn, "sweep top: level sizes inconsistent");
    copy_batched(gj, s);
    if (!zj.empty()) {
      SBX_CUDA(cudaMemsetAsync(Z.get(), 0, size_t(Kd * Kn) * 8, s));
      gemm_batched(zj, s);
      gemm_batched(ej, s);
    }
    SBX_CUDA(cudaStreamSynchronize(s));  // job tables are reused by the next level
    M = std::move(Mn);
    Kd = Kn;
  }
  if (op.o_top < 0 || op.top_cap < Kd * Kd) {  // grow the arena by the map
    const i64 off = (op.arena_used + 31) / 32 * 32;
    DevBuf<double> grown(static_cast<size_t>(off + Kd * Kd));
    SBX_CUDA(cudaMemcpyAsync(grown.get(), op.arena.get(), size_t(op.arena_used) * 8, cudaMemcpyDeviceToDevice, s));
    // the old arena may still be read by sweeps in flight on other streams
    // (an apply on a caller stream): drain the device before it is recycled
    SBX_CUDA(cudaDeviceSynchronize());
    op.arena = std::move(grown);
    op.o_top = off;
    op.top_cap = Kd * Kd;
    op.t_solve = op.t_apply = false;  // the transposed arena is rebuilt on next use
  }
  SBX_CUDA(cudaMemcpyAsync(op.arena.get() + op.o_top, M.get(), size_t(Kd * Kd) * 8, cudaMemcpyDeviceToDevice, s));
  SBX_CUDA(cudaStreamSynchronize(s));
  op.top_L = L;
  op.top_K = Kd;
}
}  // namespace

void hbs_build_solve_plan(HbsOp& op) {
  require(op.has_inverse, "hbs_solve: inverse not built");
  const SolveLayout Y = solve_layout(op);
  const std::vector<char> all(op.nodes.size(), 1);
  const int L = choose_top(op);
  if (L > 0) hbs_build_top(op, L, cur_stream());
  build_solve_tasks(op, Y, all, true, all, op.solve_plan, L);
}

ShardPlans& hbs_shard(HbsOp& op, int G, int p) {
  std::lock_guard<std::recursive_mutex> lk(op.mu);
  require(op.has_inverse, "hbs_solve: inverse not built");
  require(!op.sharded() || (op.shard_G == G && op.shard_p == p),
          "shard: a subtree-sharded operator solves only on the partition it was built for");
  require(G >= 1 && (G & (G - 1)) == 0, "shard: rank count must be a power of two");
  require(p >= 0 && p < G, "shard: rank out of range");
  if (op.shard && op.shard->G == G && op.shard->p == p) return *op.shard;
  // the previous plans' tables may still be read by kernels in flight on
  // another stream: drain before they return to the pool
  if (op.shard) SBX_CUDA(cudaDeviceSynchronize());
  auto S = std::make_unique<ShardPlans>();
  S->G = G;
  S->p = p;
  int g = 0;
  while ((1 << g) < G) ++g;
  S->g = g;
  const size_t nn = op.nodes.size();
  // subtree roots: BFS nodes of depth g, in order; every leaf must lie at depth >= g
  for (size_t i = 0; i < nn; ++i) {
    if (op.nodes[i].depth == g) S->roots.push_back(i64(i));
    if (op.nodes[i].is_leaf())
      require(op.nodes[i].depth >= g, "shard: tree has a leaf above the partition depth");
  }
  require(i64(S->roots.size()) == G, "shard: tree has fewer subtrees than ranks at that depth");
  std::vector<i64> owner(nn, -1);  // subtree index of every node at depth >= g
  for (size_t q = 0; q < S->roots.size(); ++q) owner[size_t(S->roots[q])] = i64(q);
  for (size_t i = 0; i < nn; ++i)  // BFS order: parents come first
    if (op.nodes[i].depth > g) owner[i] = owner[size_t(op.nodes[i].parent)];
  const auto& sr = op.nodes[size_t(S->roots[size_t(p)])];
  S->row0 = 2 * sr.begin;
  S->row1 = 2 * sr.end;
  for (i64 r : S->roots) S->kmax = std::max(S->kmax, op.nodes[size_t(r)].k);
  const SolveLayout Y = solve_layout(op);
  std::vector<char> mine(nn, 0), above(nn, 0), none(nn, 0);
  for (size_t i = 1; i < nn; ++i) {
    mine[i] = owner[i] == p;
    above[i] = op.nodes[i].depth >= 1 && op.nodes[i].depth < g;
  }
  if (g == 0) {  // one rank: the subtree is the whole tree, the root product is "top"
    build_solve_tasks(op, Y, mine, false, none, S->up);
    build_solve_tasks(op, Y, none, true, none, S->top);
    build_solve_tasks(op, Y, none, false, mine, S->down);
  } else {
    build_solve_tasks(op, Y, mine, false, none, S->up);
    build_solve_tasks(op, Y, above, true, above, S->top);
    build_solve_tasks(op, Y, none, false, mine, S->down);
  }
  op.shard = std::move(S);
  return *op.shard;
}

void hbs_solve_shard_up(HbsOp& op, int G, int p, const double* b_local, i64 ldb, i64 nrhs, double* hat_out,
                        bool dev, cudaStream_t s) {
  // the shard plans are replaced when (G, p) changes: one shard call at a time per handle
  std::lock_guard<std::recursive_mutex> lk(op.mu);
  ShardPlans& S = hbs_shard(op, G, p);
  const i64 rows = S.row1 - S.row0;
  require(nrhs >= 1 && ldb >= rows, "shard_up: bad sizes");
  const i64 ldw = sweep_ld(nrhs);
  SweepScratch& sc = op.scratch_for(s);
  {
    StreamScope ss(s);
    sc.ws.reserve(size_t(S.up.ws_rows * ldw));
    if (!dev) sc.io.reserve(size_t(rows * nrhs));
  }
  double* ws = sc.ws.get();
  const double* bd = b_local;
  if (!dev) {
    SBX_CUDA(cudaMemcpy2DAsync(sc.io.get(), size_t(rows) * 8, b_local, size_t(ldb) * 8, size_t(rows) * 8,
                               size_t(nrhs), cudaMemcpyHostToDevice, s));
    bd = sc.io.get();
  }
  launch_cm_to_rm(bd, dev ? ldb : rows, rows, nrhs, ws + (S.up.in_row + S.row0) * ldw, ldw, nullptr, s);
  hbs_run_plan(op, S.up, ws, nrhs, s);
  // pack hat of the subtree root: k rows (x nrhs, row-major), zero-padded to kmax
  const auto& sr = op.nodes[size_t(S.roots[size_t(p)])];
  const i64 hat_row = solve_layout(op).hat[size_t(S.roots[size_t(p)])];
  const auto kind = dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  if (S.kmax > 0) {
    if (dev) SBX_CUDA(cudaMemsetAsync(hat_out, 0, size_t(S.kmax * nrhs) * 8, s));
    else std::memset(hat_out, 0, size_t(S.kmax * nrhs) * 8);
    if (sr.k > 0 && S.g > 0)
      SBX_CUDA(cudaMemcpy2DAsync(hat_out, size_t(nrhs) * 8, ws + hat_row * ldw, size_t(ldw) * 8,
                                 size_t(nrhs) * 8, size_t(sr.k), kind, s));
  }
  if (!dev) SBX_CUDA(cudaStreamSynchronize(s));
}

void hbs_solve_shard_down(HbsOp& op, int G, int p, const double* hats, i64 nrhs, double* x_local, i64 ldx,
                          bool dev, cudaStream_t s) {
  std::lock_guard<std::recursive_mutex> lk(op.mu);
  ShardPlans& S = hbs_shard(op, G, p);
  const i64 rows = S.row1 - S.row0;
  require(nrhs >= 1 && ldx >= rows, "shard_down: bad sizes");
  const i64 ldw = sweep_ld(nrhs);
  SweepScratch& sc = op.scratch_for(s);
  require(sc.ws.size() >= size_t(S.up.ws_rows * ldw), "shard_down: call shard_up first (on the same stream)");
  double* ws = sc.ws.get();
  const SolveLayout Y = solve_layout(op);
  const auto kind = dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  if (S.g > 0)
    for (int q = 0; q < G; ++q) {  // the other ranks' subtree-root hats
      if (q == p) continue;
      const i64 r = S.roots[size_t(q)];
      const i64 k = op.nodes[size_t(r)].k;
      if (k > 0)
        SBX_CUDA(cudaMemcpy2DAsync(ws + Y.hat[size_t(r)] * ldw, size_t(ldw) * 8, hats + i64(q) * S.kmax * nrhs,
                                   size_t(nrhs) * 8, size_t(nrhs) * 8, size_t(k), kind, s));
    }
  hbs_run_plan(op, S.top, ws, nrhs, s);
  hbs_run_plan(op, S.down, ws, nrhs, s);
  if (dev) {
    launch_rm_to_cm(ws + (S.down.out_row + S.row0) * ldw, ldw, rows, nrhs, x_local, ldx, nullptr, s);
  } else {
    {
      StreamScope ss(s);
      sc.io.reserve(size_t(rows * nrhs));
    }
    launch_rm_to_cm(ws + (S.down.out_row + S.row0) * ldw, ldw, rows, nrhs, sc.io.get(), rows, nullptr, s);
    SBX_CUDA(cudaMemcpy2DAsync(x_local, size_t(ldx) * 8, sc.io.get(), size_t(rows) * 8, size_t(rows) * 8,
                               size_t(nrhs), cudaMemcpyDeviceToHost, s));
    SBX_CUDA(cudaStreamSynchronize(s));
  }
  sc.mark.record(s);
}

void hbs_build_apply_plan(HbsOp& op) {
  require(op.has_apply, "hbs_apply: operator has no forward factors");
  SweepPlan& P = op.apply_plan;
  P.levels.clear();
  const size_t nn = op.nodes.size();
  std::vector<i64> hat(nn, 0), pp(nn, 0), S(nn, 0), inc(nn, 0);
  i64 row = 0;
  P.in_row = row;
  row += op.n;
  P.out_row = row;
  row += op.n;
  for (size_t i = 1; i < nn; ++i) {
    hat[i] = row;
    row += op.nodes[i].k;
  }
  for (size_t i = 1; i < nn; ++i) {
    if (op.nodes[i].is_leaf()) {
      pp[i] = row;
      row += op.nodes[i].c;
    }
  }
  for (size_t i = 1; i < nn; ++i) {
    inc[i] = row;
    row += op.nodes[i].k;
  }
  for (size_t i = 1; i < nn; ++i) {
    if (!op.nodes[i].is_leaf()) {
      S[i] = row;
      row += op.nodes[i].c;
    }
  }
  if (nn > 1) S[0] = inc[size_t(op.nodes[0].left)];  // root's couplings are its children's inc
  P.ws_rows = row;
  if (nn == 1) {  // single leaf: y = d v (hbs.cpp:513)
    SweepLevel L;
    const i64 c = op.nodes[0].c;
    L.tasks.push_back(mk(op.nodes[0].o_vd, c, c, c, P.in_row, -1, P.out_row, 0, c));
    P.levels.push_back(std::move(L));
    finalize(P);
    return;
  }
  for (int d = op.max_depth; d >= 0; --d) {  // up: hats of depth d, couplings S of depth d
    SweepLevel L;
    for (size_t i = 0; i < nn; ++i) {
      const auto& nd = op.nodes[i];
      if (nd.depth != d) continue;
      if (i != 0) {
        if (nd.is_leaf())
          L.tasks.push_back(mk(nd.o_vd, nd.k + nd.c, nd.k + nd.c, nd.c, P.in_row + 2 * nd.begin, -1,
                               hat[i], pp[i], nd.k));
        else
          L.tasks.push_back(mk(nd.o_vd, nd.k, nd.k, nd.c, hat[size_t(nd.left)], -1, hat[i], 0, nd.k));
      }
      if (!nd.is_leaf()) {
        const size_t l = size_t(nd.left), r = size_t(nd.right);
        const auto& L_ = op.nodes[l];
        const auto& R_ = op.nodes[r];
        // inc_l = b_sib_l hat_r, inc_r = b_sib_r hat_l (hbs.cpp:527-528)
        L.tasks.push_back(mk(L_.o_b, L_.k, L_.k, R_.k, hat[r], -1, S[i], 0, L_.k));
        L.tasks.push_back(mk(R_.o_b, R_.k, R_.k, L_.k, hat[l], -1, S[i] + L_.k, 0, R_.k));
      }
    }
    // couplings of depth d need hats of depth d+1 only, so they share the level
    if (!L.tasks.empty()) P.levels.push_back(std::move(L));
  }
  for (int d = 1; d <= op.max_depth; ++d) {  // down
    SweepLevel L;
    for (size_t i = 1; i < nn; ++i) {
      const auto& nd = op.nodes[i];
      if (nd.depth != d) continue;
      if (!nd.is_leaf())
        L.tasks.push_back(mk(nd.o_u, nd.c, nd.c, nd.k, inc[i], S[i], inc[size_t(nd.left)], 0, nd.c));
      else
        L.tasks.push_back(mk(nd.o_u, nd.c, nd.c, nd.k, inc[i], pp[i], P.out_row + 2 * nd.begin, 0, nd.c));
    }
    if (!L.tasks.empty()) P.levels.push_back(std::move(L));
  }
  finalize(P);
}

namespace {
template <int TN>
void run_flow(HbsOp& op, SweepPlan& plan, double* ws, i64 nrhs, cudaStream_t s, const double* fac,
              const SweepDirectIo* dio, bool build_only) {
  const bool dmma = nrhs > 1;
  static const bool per_level = std::getenv("SBX_SWEEP_LEVELS") != nullptr;  // diagnostics
  int max_k = 0;
  for (auto& L : plan.levels) max_k = std::max(max_k, L.max_k);
  const size_t gemv_smem = size_t(((max_k + 1) & ~1) + kThreads) * sizeof(double);
  const size_t smem = dmma ? sizeof(DmmaSmem<TN>) : gemv_smem;
  static std::once_flag attr;
  std::call_once(attr, [] {
    SBX_CUDA(cudaFuncSetAttribute(sweep_flow_kernel<true, TN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(sizeof(DmmaSmem<TN>))));
    SBX_CUDA(cudaFuncSetAttribute(sweep_dmma_kernel<TN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(sizeof(DmmaSmem<TN>))));
  });
  const int ncol = dmma ? int((nrhs + TN - 1) / TN) : 1;
  const int tile = dmma ? kTM : kGR;
  int dev = 0, sms = 148, per_sm = 1;
  SBX_CUDA(cudaGetDevice(&dev));
  SBX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (dmma)
    SBX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_flow_kernel<true, TN>, kThreads, smem));
  else
    SBX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_flow_kernel<false, TN>, kThreads, smem));
  per_sm = std::max(per_sm, 1);
  static const int split_env = [] {
    // split-K of the short upper levels: measured slower on cfg2/cfg3 (the
    // partial-tile round trip costs more than the shorter K loop saves), so
    // it is off unless SBX_SWEEP_SPLIT=1
    const char* e = std::getenv("SBX_SWEEP_SPLIT");
    return e ? std::atoi(e) : 0;
  }();
  static const int split_target = [] {
    const char* e = std::getenv("SBX_SWEEP_SPLIT_TARGET");
    return e ? std::atoi(e) : 64;
  }();
  const int target = (per_level || split_env == 0) ? 0 : split_target;
  static const int dmma_small = [] {  // 32-row DMMA tiles on short levels (SBX_SWEEP_DMMA_SMALL=0 disables)
    const char* e = std::getenv("SBX_SWEEP_DMMA_SMALL");
    return (e && std::atoi(e) == 0) ? 0 : 32;
  }();
  static const int small_below_dmma = [] {
    const char* e = std::getenv("SBX_SWEEP_DMMA_SMALL_BELOW");
    return e ? std::atoi(e) : 300;
  }();
  static const int small_below_gemv = [] {
    const char* e = std::getenv("SBX_SWEEP_GEMV_SMALL_BELOW");
    return e ? std::atoi(e) : 300;
  }();
  const int key = ((ncol * 2 + (dmma ? 1 : 0)) * 2 + (target > 0 ? 1 : 0)) * 128 + TN;
  // the flow items of this width are built once per plan under op.mu (they
  // are immutable afterwards and shared by every stream)
  std::unique_lock<std::recursive_mutex> lk(op.mu);
  auto& slot = plan.flows[key];
  const bool fresh = !slot;
  if (fresh) slot = std::make_unique<FlowCache>();
  FlowCache& F = *slot;
  if (fresh) {
    std::vector<int> needs;
    const std::vector<FlowItem> fi =
        make_items(plan, tile, ncol, dmma ? kTM * TN : kGR, target, &F.level_items, &F.partial_elems,
                   &F.n_tile_cnt, &needs, per_level ? 0 : (dmma ? dmma_small : kGRs),
                   dmma ? small_below_dmma : small_below_gemv, dmma ? 128 : kGRs * GemvShape<kGRs>::kGV);
    F.d_flow_items.upload(fi, s);
    F.d_needs.upload(needs, s);
    std::vector<ItemDesc> descs(fi.size());
    for (size_t q = 0; q < fi.size(); ++q) {
      ItemDesc& D = descs[q];
      D.it = fi[q];
      D.t = plan.h_tasks[size_t(fi[q].task)];
      for (int d = 0; d < kMaxDep; ++d) D.need[d] = d < D.t.ndep ? needs[size_t(D.t.dep[d])] : 0;
    }
    F.d_descs.upload(descs, s);
    F.n_flow_items = i64(fi.size());
    SBX_CUDA(cudaStreamSynchronize(s));  // other streams may launch over these tables next
  }
  lk.unlock();
  if (build_only) return;  // hbs_prebuild_flow: the item tables of this width now exist
  if (per_level) {
    for (const int2 rg : F.level_items) {
      if (rg.y == 0) continue;
      const FlowItem* items = F.d_flow_items.get() + rg.x;
      if (!dmma)
        sweep_gemv_kernel<<<unsigned(rg.y), kThreads, gemv_smem, s>>>(fac, ws, plan.d_tasks.get(), items);
      else
        sweep_dmma_kernel<TN><<<unsigned(rg.y), kThreads, smem, s>>>(fac, ws, plan.d_tasks.get(), items,
                                                                      int(nrhs), int(sweep_ld(nrhs)));
      SBX_LAUNCHED();
    }
    return;
  }
  if (F.n_flow_items == 0) return;
  // completion counters and split-K partials are per call: the stream's scratch
  SweepScratch& sc = op.scratch_for(s);
  const size_t ncount = size_t(1 + plan.n_tasks * ncol + F.n_tile_cnt);
  {
    StreamScope ss(s);
    sc.counters.reserve(ncount);
    sc.partials.reserve(size_t(std::max<i64>(F.partial_elems, 1)));
  }
  if (sc.counters_zeroed != sc.counters.get() || sc.counters_zeroed_n < ncount) {
    // fresh (or regrown) memory; afterwards every launch leaves its counters zero
    SBX_CUDA(cudaMemsetAsync(sc.counters.get(), 0, sc.counters.size() * sizeof(int), s));
    sc.counters_zeroed = sc.counters.get();
    sc.counters_zeroed_n = sc.counters.size();
  }
  int* counters = sc.counters.get();
  int* tile_cnt = counters + 1 + plan.n_tasks * ncol;
  double* partials = sc.partials.get();
  const int grid = int(std::min<i64>(F.n_flow_items, i64(sms) * per_sm));
  static const char* trace_path = std::getenv("SBX_SWEEP_TRACE");  // diagnostics: per-item timeline
  DevBuf<unsigned long long> trace;
  if (trace_path) trace.resize(size_t(4 * F.n_flow_items));
  unsigned long long* tr = trace.get();
  const SweepTask* tasks = plan.d_tasks.get();
  const FlowItem* items = F.d_flow_items.get();
  const ItemDesc* descs = F.d_descs.get();
  int n_items = int(F.n_flow_items), nr = int(nrhs), ldw = dmma ? int(sweep_ld(nrhs)) : 1;
  SweepDirectIo io = (dio && !dmma) ? *dio : SweepDirectIo{};
  int ncount_i = int(ncount);
  void* args[] = {(void*)&fac, (void*)&ws, (void*)&tasks, (void*)&items, (void*)&n_items, (void*)&counters,
                  (void*)&ncol, (void*)&nr, (void*)&ldw, (void*)&partials, (void*)&tile_cnt, (void*)&tr,
                  (void*)&descs, (void*)&io, (void*)&ncount_i};
  // Cooperative launch: the static round-robin item schedule spin-waits on
  // items held by other CTAs, which is only deadlock-free when the whole
  // grid is co-resident -- guaranteed here even when other streams' kernels
  // (a concurrent solve on the same handle) occupy part of the chip.
  KernelTimer kt(dmma ? "sweep_flow_dmma" : "sweep_flow_gemv", s);
  const void* fn = dmma ? reinterpret_cast<const void*>(&sweep_flow_kernel<true, TN>)
                        : reinterpret_cast<const void*>(&sweep_flow_kernel<false, TN>);
  SBX_CUDA(cudaLaunchCooperativeKernel(fn, dim3(unsigned(grid)), dim3(kThreads), args, smem, s));
  SBX_LAUNCHED();
  if (trace_path) {
    std::vector<unsigned long long> h(size_t(4 * F.n_flow_items));
    std::vector<FlowItem> fi(size_t(F.n_flow_items));
    trace.download(h.data(), h.size(), s);
    F.d_flow_items.download(fi.data(), fi.size(), s);
    SBX_CUDA(cudaStreamSynchronize(s));
    std::vector<int> level_of(size_t(plan.n_tasks), 0);
    for (size_t l = 0; l < plan.levels.size(); ++l)
      for (size_t t = 0; t < plan.levels[l].tasks.size(); ++t)
        level_of[size_t(plan.levels[l].first_task) + t] = int(l);
    if (FILE* f = std::fopen(trace_path, "a")) {
      std::fprintf(f, "# nrhs %lld items %lld grid %d\n", (long long)nrhs, (long long)F.n_flow_items, grid);
      for (i64 i = 0; i < F.n_flow_items; ++i) {
        const auto& it = fi[size_t(i)];
        const auto& tk = plan.levels[size_t(level_of[size_t(it.task)])];
        (void)tk;
        std::fprintf(f, "%lld %d %d %d %d %d %llu %llu %llu %llu\n", (long long)i, level_of[size_t(it.task)],
                     it.task, it.nsplit, it.ke - it.kb, it.row0, h[size_t(4 * i)], h[size_t(4 * i + 1)],
                     h[size_t(4 * i + 2)], h[size_t(4 * i + 3)]);
      }
      std::fclose(f);
    }
  }
}

}  // namespace

void hbs_ensure_solve_plan(HbsOp& op) {
  require(!op.sharded(), "hbs_solve: a subtree-sharded operator solves through sbx_hbs_solve_sharded");
  if (op.solve_plan.built.load(std::memory_order_acquire)) return;
  std::lock_guard<std::recursive_mutex> lk(op.mu);
  if (!op.solve_plan.built) hbs_build_solve_plan(op);
}

void hbs_ensure_apply_plan(HbsOp& op) {
  require(!op.sharded(), "hbs_apply: a subtree-sharded operator holds only its subtree's factors");
  if (op.apply_plan.built.load(std::memory_order_acquire)) return;
  std::lock_guard<std::recursive_mutex> lk(op.mu);
  if (!op.apply_plan.built) hbs_build_apply_plan(op);
}

void hbs_sweep_rows(HbsOp& op, SweepPlan& plan, const double* in, i64 ldi, i64 rows, i64 nrhs, double* out,
                    i64 ldo, const i64* map, bool transposed, cudaStream_t s) {
  if (nrhs == 0 || rows == 0) return;
  const i64 ldw = sweep_ld(nrhs);
  SweepScratch& sc = op.scratch_for(s);
  {
    StreamScope ss(s);
    sc.ws.reserve(size_t(plan.ws_rows * ldw));
  }
  double* ws = sc.ws.get();
  // one right-hand side in natural order: the leaf items read the caller's
  // vector and the last items write the caller's result (no layout kernels)
  static const bool no_direct = std::getenv("SBX_SWEEP_NO_DIRECT") != nullptr ||
                                std::getenv("SBX_SWEEP_LEVELS") != nullptr;  // diagnostics
  const bool disjoint = in + rows <= out || out + rows <= in;
  if (nrhs == 1 && !map && !no_direct && disjoint && rows == op.n) {
    SweepDirectIo io;
    io.in = in;
    io.out = out;
    io.in_row = plan.in_row;
    io.out_row = plan.out_row;
    io.n = rows;
    hbs_run_plan(op, plan, ws, nrhs, s, transposed ? op.arena_t.get() : nullptr, &io);
    sc.mark.record(s);
    return;
  }
  launch_cm_to_rm(in, ldi, rows, nrhs, ws + plan.in_row * ldw, ldw, map, s);
  hbs_run_plan(op, plan, ws, nrhs, s, transposed ? op.arena_t.get() : nullptr);
  launch_rm_to_cm(ws + plan.out_row * ldw, ldw, rows, nrhs, out, ldo, map, s);
  sc.mark.record(s);
}

void hbs_sweep_rm(HbsOp& op, bool apply, bool transpose, const double* b, i64 ldb, i64 nrhs, double* x, i64 ldx,
                  cudaStream_t s) {
  require(nrhs >= 0 && ldb >= std::max<i64>(nrhs, 1) && ldx >= std::max<i64>(nrhs, 1),
          "sweep: row-major leading dimension smaller than nrhs");
  if (apply) hbs_ensure_apply_plan(op);
  else hbs_ensure_solve_plan(op);
  if (transpose) hbs_ensure_transpose(op, !apply, apply, s);
  if (nrhs == 0) return;
  SweepPlan& plan = apply ? op.apply_plan : op.solve_plan;
  const i64 ldw = sweep_ld(nrhs);
  SweepScratch& sc = op.scratch_for(s);
  {
    StreamScope ss(s);
    sc.ws.reserve(size_t(plan.ws_rows * ldw));
  }
  double* ws = sc.ws.get();
  {
    // one dense right-hand side: the sweep reads b and writes x in place of
    // the workspace's input / output regions (no copies)
    static const bool no_direct = std::getenv("SBX_SWEEP_NO_DIRECT") != nullptr ||
                                  std::getenv("SBX_SWEEP_LEVELS") != nullptr;  // diagnostics
    const bool disjoint = b + op.n <= x || x + op.n <= b;
    if (nrhs == 1 && ldb == 1 && ldx == 1 && disjoint && !no_direct) {
      SweepDirectIo io;
      io.in = b;
      io.out = x;
      io.in_row = plan.in_row;
      io.out_row = plan.out_row;
      io.n = op.n;
      hbs_run_plan(op, plan, ws, nrhs, s, transpose ? op.arena_t.get() : nullptr, &io);
      sc.mark.record(s);
      return;
    }
  }
  // dense rows (ld == nrhs == the workspace pitch): one linear copy; a 2D
  // copy of 8-byte rows runs at a fraction of the bandwidth
  if (ldb == nrhs && ldw == nrhs)
    SBX_CUDA(cudaMemcpyAsync(ws + plan.in_row * ldw, b, size_t(op.n * nrhs) * 8, cudaMemcpyDeviceToDevice, s));
  else
    SBX_CUDA(cudaMemcpy2DAsync(ws + plan.in_row * ldw, size_t(ldw) * 8, b, size_t(ldb) * 8, size_t(nrhs) * 8,
                               size_t(op.n), cudaMemcpyDeviceToDevice, s));
  hbs_run_plan(op, plan, ws, nrhs, s, transpose ? op.arena_t.get() : nullptr);
  if (ldx == nrhs && ldw == nrhs)
    SBX_CUDA(cudaMemcpyAsync(x, ws + plan.out_row * ldw, size_t(op.n * nrhs) * 8, cudaMemcpyDeviceToDevice, s));
  else
    SBX_CUDA(cudaMemcpy2DAsync(x, size_t(ldx) * 8, ws + plan.out_row * ldw, size_t(ldw) * 8, size_t(nrhs) * 8,
                               size_t(op.n), cudaMemcpyDeviceToDevice, s));
  sc.mark.record(s);
}

namespace {
void run_plan(HbsOp& op, SweepPlan& plan, double* ws, i64 nrhs, cudaStream_t s, const double* fac,
              const SweepDirectIo* io, bool build_only);
}

void hbs_run_plan(HbsOp& op, SweepPlan& plan, double* ws, i64 nrhs, cudaStream_t s, const double* fac,
                  const SweepDirectIo* io) {
  run_plan(op, plan, ws, nrhs, s, fac, io, false);
}

void hbs_prebuild_flow(HbsOp& op, SweepPlan& plan, i64 nrhs, cudaStream_t s) {
  if (nrhs >= 1) run_plan(op, plan, nullptr, nrhs, s, nullptr, nullptr, true);
}

namespace {
void run_plan(HbsOp& op, SweepPlan& plan, double* ws, i64 nrhs, cudaStream_t s, const double* fac,
              const SweepDirectIo* io, bool build_only) {
  if (!fac) fac = op.arena.get();
  // column tile: 32 when the block is narrow enough that the tree depth
  // (not the tensor throughput) bounds the sweep (SBX_SWEEP_TN overrides)
  static const int tn_env = [] {
    const char* e = std::getenv("SBX_SWEEP_TN");
    return e ? std::atoi(e) : 0;
  }();
  const int tn = tn_env == 32 || tn_env == 64 ? tn_env : (nrhs <= 192 ? 32 : 64);
  if (tn == 32)
    run_flow<32>(op, plan, ws, nrhs, s, fac, io, build_only);
  else
    run_flow<64>(op, plan, ws, nrhs, s, fac, io, build_only);
}
}  // namespace

namespace {
void run_sweep(HbsOp& op, SweepPlan& plan, const double* b, i64 ldb, i64 nrhs, double* x, i64 ldx,
               bool dev, cudaStream_t s, bool transposed = false) {
  require(nrhs >= 0, "sweep: negative nrhs");
  require(ldb >= op.n && ldx >= op.n, "sweep: leading dimension smaller than n");
  if (nrhs == 0) return;
  const double* bd = b;
  double* xd = x;
  if (!dev) {
    SweepScratch& sc = op.scratch_for(s);
    {
      StreamScope ss(s);
      sc.io.reserve(size_t(2 * op.n * nrhs));
    }
    double* hb = sc.io.get();
    SBX_CUDA(cudaMemcpy2DAsync(hb, size_t(op.n) * 8, b, size_t(ldb) * 8, size_t(op.n) * 8,
                               size_t(nrhs), cudaMemcpyHostToDevice, s));
    bd = hb;
    xd = hb + op.n * nrhs;
  }
  hbs_sweep_rows(op, plan, bd, dev ? ldb : op.n, op.n, nrhs, xd, dev ? ldx : op.n, nullptr, transposed, s);
  if (!dev) {
    SBX_CUDA(cudaMemcpy2DAsync(x, size_t(ldx) * 8, xd, size_t(op.n) * 8, size_t(op.n) * 8,
                               size_t(nrhs), cudaMemcpyDeviceToHost, s));
    SBX_CUDA(cudaStreamSynchronize(s));
  }
}
}  // namespace

void hbs_solve(HbsOp& op, const double* b, i64 ldb, i64 nrhs, double* x, i64 ldx, bool dev,
               cudaStream_t s) {
  hbs_ensure_solve_plan(op);
  run_sweep(op, op.solve_plan, b, ldb, nrhs, x, ldx, dev, s);
}

void hbs_apply(HbsOp& op, const double* v, i64 ldv, i64 nrhs, double* y, i64 ldy, bool dev,
               cudaStream_t s) {
  hbs_ensure_apply_plan(op);
  run_sweep(op, op.apply_plan, v, ldv, nrhs, y, ldy, dev, s);
}

void hbs_ensure_transpose(HbsOp& op, bool solve, bool apply, cudaStream_t s) {
  std::lock_guard<std::recursive_mutex> lk(op.mu);
  solve = solve && !op.t_solve;
  apply = apply && !op.t_apply;
  if (!solve && !apply) return;
  if (!op.arena_t.get() || op.arena_t.size() < op.arena.size()) {
    require(!op.t_solve && !op.t_apply, "transposed arena: layout changed after build");
    op.arena_t.resize(op.arena.size());
  }
  const double* A = op.arena.get();
  double* T = op.arena_t.get();
  std::vector<CopyJob> jobs;
  auto tr = [&](i64 src, int lds, i64 dst, int ldd, int rows, int cols, int trans) {
    if (rows > 0 && cols > 0) jobs.push_back({A + src, T + dst, rows, cols, lds, ldd, trans, 0});
  };
  const size_t nn = op.nodes.size();
  if (solve) {
    require(op.has_inverse, "hbs_solve_t: inverse not built");
    const i64 c0 = op.nodes[0].c;
    tr(op.o_root_g, int(c0), op.o_root_g, int(c0), int(c0), int(c0), 1);
    if (op.top_L > 0) tr(op.o_top, int(op.top_K), op.o_top, int(op.top_K), int(op.top_K), int(op.top_K), 1);
    for (size_t i = 1; i < nn; ++i) {
      const auto& nd = op.nodes[i];
      const int k = int(nd.k), c = int(nd.c), ld = k + c;
      tr(nd.o_e, c, nd.o_fg, ld, k, c, 1);                  // [e^T; .]
      tr(nd.o_fg + k, ld, nd.o_fg + k, ld, c, c, 1);        // [.; g^T]
      tr(nd.o_fg, ld, nd.o_e, c, c, k, 1);                  // f^T
    }
  }
  if (apply) {
    require(op.has_apply, "hbs_apply_t: operator has no forward factors");
    if (nn == 1) {
      const int c = int(op.nodes[0].c);
      tr(op.nodes[0].o_vd, c, op.nodes[0].o_vd, c, c, c, 1);  // d^T
    }
    for (size_t i = 1; i < nn; ++i) {
      const auto& nd = op.nodes[i];
      const int k = int(nd.k), c = int(nd.c);
      const int ld = k + (nd.is_leaf() ? c : 0);
      tr(nd.o_u, c, nd.o_vd, ld, k, c, 1);                                    // [u^T; .]
      if (nd.is_leaf()) tr(nd.o_vd + k, ld, nd.o_vd + k, ld, c, c, 1);        // [.; d^T]
      tr(nd.o_v, c, nd.o_u, c, c, k, 0);                                      // u <- v
      const auto& sb = op.nodes[size_t(op.sib(i64(i)))];
      tr(sb.o_b, int(sb.k), nd.o_b, k, k, int(sb.k), 1);                      // b_i <- b_sib^T
    }
  }
  for (size_t q = 0; q < jobs.size(); q += 60000)  // grid.y limit of the copy kernel
    copy_batched(std::vector<CopyJob>(jobs.begin() + q, jobs.begin() + std::min(jobs.size(), q + 60000)), s);
  SBX_CUDA(cudaStreamSynchronize(s));  // job tables and the arena are shared state
  if (solve) op.t_solve = true;
  if (apply) op.t_apply = true;
}

void hbs_solve_t(HbsOp& op, const double* b, i64 ldb, i64 nrhs, double* x, i64 ldx, bool dev,
                 cudaStream_t s) {
  hbs_ensure_solve_plan(op);
  hbs_ensure_transpose(op, true, false, s);
  run_sweep(op, op.solve_plan, b, ldb, nrhs, x, ldx, dev, s, true);
}

void hbs_apply_t(HbsOp& op, const double* v, i64 ldv, i64 nrhs, double* y, i64 ldy, bool dev,
                 cudaStream_t s) {
  hbs_ensure_apply_plan(op);
  hbs_ensure_transpose(op, false, true, s);
  run_sweep(op, op.apply_plan, v, ldv, nrhs, y, ldy, dev, s, true);
}

}  // namespace sbx
