// HBS inverse / forward apply sweeps on sm_100a (reference hbs.cpp:511-625).
//
// Every level of the up- and down-sweep is one launch of a batched,
// variable-size product D = A*B (+P) over all boxes of that level, row-tiled
// so large boxes spread over several CTAs:
//   * nrhs == 1 : HBM-bound GEMV (sweep_gemv_kernel).  Factors are read once,
//     coalesced along columns, with 8 independent loads in flight per thread;
//     the input vector segment is staged in shared memory.
//   * nrhs >= 2 : FP64 tensor-core tiles (sweep_dmma_kernel) issuing
//     mma.sync.m8n8k4.f64 (SASS DMMA), operands staged in shared memory.
// The leaf products g*b and d*v that only depend on the input are folded
// into the first (leaf) up-level, so the down-sweep streams e / u only.
#include <algorithm>

#include "hbs.hpp"

namespace sbx {

namespace {

constexpr int kTM = 64;       // rows per work item
constexpr int kThreads = 256;

// ---------------------------------------------------------------- nrhs == 1
__global__ void __launch_bounds__(kThreads)
    sweep_gemv_kernel(const double* __restrict__ fac, double* __restrict__ ws,
                      const SweepTask* __restrict__ tasks, const int2* __restrict__ items) {
  extern __shared__ double sm[];
  const int2 it = items[blockIdx.x];
  const SweepTask t = tasks[it.x];
  const int K = t.K;
  double* xs = sm;                   // K doubles
  double* red = sm + ((K + 1) & ~1); // kThreads partial sums
  for (int j = threadIdx.x; j < K; j += kThreads) xs[j] = ws[t.b_row + j];
  __syncthreads();
  const int r = threadIdx.x % kTM;
  const int slice = threadIdx.x / kTM;
  constexpr int kSlices = kThreads / kTM;
  const int row = it.y + r;
  double acc = 0.0;
  if (row < t.m) {
    const double* a = fac + t.a_off + row;
    const int per = (K + kSlices - 1) / kSlices;
    const int j0 = slice * per;
    const int j1 = min(K, j0 + per);
    int j = j0;
    double acc1 = 0.0;
    for (; j + 8 <= j1; j += 8) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = __ldg(a + size_t(j + q) * t.lda);
#pragma unroll
      for (int q = 0; q < 8; q += 2) {
        acc = fma(v[q], xs[j + q], acc);
        acc1 = fma(v[q + 1], xs[j + q + 1], acc1);
      }
    }
    for (; j < j1; ++j) acc = fma(__ldg(a + size_t(j) * t.lda), xs[j], acc);
    acc += acc1;
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  if (slice == 0 && row < t.m) {
    double s = red[r];
#pragma unroll
    for (int q = 1; q < kSlices; ++q) s += red[r + q * kTM];
    if (t.p_row >= 0) s += ws[t.p_row + row];
    const i64 dst = row < t.split ? t.d1_row + row : t.d2_row + (row - t.split);
    ws[dst] = s;
  }
}

// ---------------------------------------------------------------- nrhs >= 2
// C tile 64 x 64, 8 warps, warp tile 16 x 32 = 2 x 4 m8n8 blocks.
constexpr int kTN = 64;
constexpr int kKC = 16;
constexpr int kPad = 8;  // row stride 72 doubles = 16 banks mod 32: 2 wavefronts

__device__ __forceinline__ void dmma_m8n8k4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(kThreads)
    sweep_dmma_kernel(const double* __restrict__ fac, double* __restrict__ ws,
                      const SweepTask* __restrict__ tasks, const int2* __restrict__ items,
                      int nrhs) {
  __shared__ double As[2][kKC][kTM + kPad];
  __shared__ double Bs[2][kKC][kTN + kPad];
  const int2 it = items[blockIdx.x];
  const SweepTask t = tasks[it.x];
  const int col0 = blockIdx.y * kTN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int wm = (warp & 3) * 16;  // warp row offset in tile
  const int wn = (warp >> 2) * 32; // warp col offset
  double c[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) c[a][b][0] = c[a][b][1] = 0.0;

  const double* A = fac + t.a_off;
  const double* B = ws + t.b_row * nrhs;
  const int K = t.K;
  const int nchunks = (K + kKC - 1) / kKC;

  // loaders: A chunk 16 x 64 (4 per thread), B chunk 16 x 64 (4 per thread)
  auto load = [&](int buf, int k0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = threadIdx.x + q * kThreads;  // 0..1023
      const int kk = idx >> 6, rr = idx & 63;
      const int grow = it.y + rr, gk = k0 + kk;
      As[buf][kk][rr] = (grow < t.m && gk < K) ? __ldg(A + grow + size_t(gk) * t.lda) : 0.0;
      const int gcol = col0 + rr;
      Bs[buf][kk][rr] = (gk < K && gcol < nrhs) ? B[size_t(gk) * nrhs + gcol] : 0.0;
    }
  };

  if (nchunks > 0) load(0, 0);
  __syncthreads();
  for (int ch = 0; ch < nchunks; ++ch) {
    const int buf = ch & 1;
    if (ch + 1 < nchunks) load(buf ^ 1, (ch + 1) * kKC);
#pragma unroll
    for (int k4 = 0; k4 < kKC; k4 += 4) {
      double af[2], bf[4];
#pragma unroll
      for (int a = 0; a < 2; ++a) af[a] = As[buf][k4 + tig][wm + a * 8 + gid];
#pragma unroll
      for (int b = 0; b < 4; ++b) bf[b] = Bs[buf][k4 + tig][wn + b * 8 + gid];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma_m8n8k4(c[a][b][0], c[a][b][1], af[a], bf[b]);
    }
    __syncthreads();
  }
  // epilogue: rows wm + a*8 + gid, cols wn + b*8 + 2*tig + {0,1}
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int row = it.y + wm + a * 8 + gid;
    if (row >= t.m) continue;
    const i64 dst = row < t.split ? t.d1_row + row : t.d2_row + (row - t.split);
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = col0 + wn + b * 8 + 2 * tig + h;
        if (col >= nrhs) continue;
        double v = c[a][b][h];
        if (t.p_row >= 0) v += ws[(t.p_row + row) * nrhs + col];
        ws[dst * nrhs + col] = v;
      }
  }
}

// ---------------------------------------------------------------- layout moves
__global__ void cm_to_rm_kernel(const double* __restrict__ src, i64 ld, i64 n, i64 nrhs,
                                double* __restrict__ dst, const i64* __restrict__ map) {
  const i64 total = n * nrhs;
  for (i64 idx = blockIdx.x * i64(blockDim.x) + threadIdx.x; idx < total;
       idx += i64(gridDim.x) * blockDim.x) {
    const i64 i = idx % n, c = idx / n;  // coalesced read along columns
    const i64 r = map ? map[i] : i;
    dst[r * nrhs + c] = src[i + c * ld];
  }
}

__global__ void rm_to_cm_kernel(const double* __restrict__ src, i64 n, i64 nrhs,
                                double* __restrict__ dst, i64 ld, const i64* __restrict__ map) {
  const i64 total = n * nrhs;
  for (i64 idx = blockIdx.x * i64(blockDim.x) + threadIdx.x; idx < total;
       idx += i64(gridDim.x) * blockDim.x) {
    const i64 i = idx % n, c = idx / n;
    const i64 r = map ? map[i] : i;
    dst[i + c * ld] = src[r * nrhs + c];
  }
}

int grid_for(i64 total) {
  return int(std::min<i64>((total + 255) / 256, 148 * 16));
}

}  // namespace

void launch_cm_to_rm(const double* src, i64 ld, i64 n, i64 nrhs, double* dst, const i64* map,
                     cudaStream_t s) {
  if (n * nrhs == 0) return;
  cm_to_rm_kernel<<<grid_for(n * nrhs), 256, 0, s>>>(src, ld, n, nrhs, dst, map);
  SBX_LAUNCHED();
}

void launch_rm_to_cm(const double* src, i64 n, i64 nrhs, double* dst, i64 ld, const i64* map,
                     cudaStream_t s) {
  if (n * nrhs == 0) return;
  rm_to_cm_kernel<<<grid_for(n * nrhs), 256, 0, s>>>(src, n, nrhs, dst, ld, map);
  SBX_LAUNCHED();
}

namespace {

void add_items(SweepLevel& L, std::vector<int2>& items, i64 task_base) {
  L.first_item = i64(items.size());
  for (size_t t = 0; t < L.tasks.size(); ++t) {
    const auto& tk = L.tasks[t];
    L.max_k = std::max(L.max_k, tk.K);
    for (int r0 = 0; r0 < tk.m; r0 += kTM) items.push_back(make_int2(int(task_base + i64(t)), r0));
  }
  L.n_items = i64(items.size()) - L.first_item;
}

void finalize(SweepPlan& plan) {
  std::vector<SweepTask> all;
  std::vector<int2> items;
  for (auto& L : plan.levels) {
    L.first_task = i64(all.size());
    add_items(L, items, L.first_task);
    all.insert(all.end(), L.tasks.begin(), L.tasks.end());
  }
  const cudaStream_t st = cur_stream();
  plan.d_tasks.upload(all, st);
  plan.d_items.upload(items, st);
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
  t.pad = 0;
  return t;
}

}  // namespace

void hbs_build_solve_plan(HbsOp& op) {
  require(op.has_inverse, "hbs_solve: inverse not built");
  SweepPlan& P = op.solve_plan;
  P.levels.clear();
  const size_t nn = op.nodes.size();
  // workspace rows: IN, OUT, HAT (k_i), PP (c_i), INC (k_i); node order
  std::vector<i64> hat(nn, 0), pp(nn, 0), inc(nn, 0);
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
    pp[i] = row;
    row += op.nodes[i].c;
  }
  for (size_t i = 1; i < nn; ++i) {
    inc[i] = row;
    row += op.nodes[i].k;
  }
  P.ws_rows = row;
  if (nn == 1) {  // single leaf: x = root_g b (hbs.cpp:592)
    SweepLevel L;
    const i64 c = op.nodes[0].c;
    L.tasks.push_back(mk(op.o_root_g, c, c, c, P.in_row, -1, P.out_row, 0, c));
    P.levels.push_back(std::move(L));
    finalize(P);
    return;
  }
  for (int d = op.max_depth; d >= 1; --d) {  // up
    SweepLevel L;
    for (size_t i = 1; i < nn; ++i) {
      const auto& nd = op.nodes[i];
      if (nd.depth != d) continue;
      const i64 b = nd.is_leaf() ? P.in_row + 2 * nd.begin : hat[size_t(nd.left)];
      L.tasks.push_back(mk(nd.o_fg, nd.k + nd.c, nd.k + nd.c, nd.c, b, -1, hat[i], pp[i], nd.k));
    }
    if (!L.tasks.empty()) P.levels.push_back(std::move(L));
  }
  for (int d = 0; d <= op.max_depth; ++d) {  // down
    SweepLevel L;
    for (size_t i = 0; i < nn; ++i) {
      const auto& nd = op.nodes[i];
      if (nd.depth != d) continue;
      if (i == 0) {
        const i64 c = nd.c;
        L.tasks.push_back(mk(op.o_root_g, c, c, c, hat[size_t(nd.left)], -1, inc[size_t(nd.left)], 0, c));
      } else if (!nd.is_leaf()) {
        L.tasks.push_back(mk(nd.o_e, nd.c, nd.c, nd.k, inc[i], pp[i], inc[size_t(nd.left)], 0, nd.c));
      } else {
        L.tasks.push_back(mk(nd.o_e, nd.c, nd.c, nd.k, inc[i], pp[i], P.out_row + 2 * nd.begin, 0, nd.c));
      }
    }
    if (!L.tasks.empty()) P.levels.push_back(std::move(L));
  }
  finalize(P);
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

void hbs_run_plan(HbsOp& op, SweepPlan& plan, double* ws, i64 nrhs, cudaStream_t s) {
  const double* fac = op.arena.get();
  for (auto& L : plan.levels) {
    if (L.n_items == 0) continue;
    const SweepTask* tasks = plan.d_tasks.get();
    const int2* items = plan.d_items.get() + L.first_item;
    if (nrhs == 1) {
      const size_t smem = size_t(((L.max_k + 1) & ~1) + kThreads) * sizeof(double);
      sweep_gemv_kernel<<<unsigned(L.n_items), kThreads, smem, s>>>(fac, ws, tasks, items);
    } else {
      dim3 grid(unsigned(L.n_items), unsigned((nrhs + kTN - 1) / kTN));
      sweep_dmma_kernel<<<grid, kThreads, 0, s>>>(fac, ws, tasks, items, int(nrhs));
    }
    SBX_LAUNCHED();
  }
}

namespace {
void run_sweep(HbsOp& op, SweepPlan& plan, const double* b, i64 ldb, i64 nrhs, double* x, i64 ldx,
               bool dev, cudaStream_t s) {
  require(nrhs >= 0, "sweep: negative nrhs");
  require(ldb >= op.n && ldx >= op.n, "sweep: leading dimension smaller than n");
  if (nrhs == 0) return;
  op.ws.reserve(size_t(plan.ws_rows * nrhs));
  double* ws = op.ws.get();
  const double* bd = b;
  double* xd = x;
  if (!dev) {
    op.io.reserve(size_t(2 * op.n * nrhs));
    double* hb = op.io.get();
    SBX_CUDA(cudaMemcpy2DAsync(hb, size_t(op.n) * 8, b, size_t(ldb) * 8, size_t(op.n) * 8,
                               size_t(nrhs), cudaMemcpyHostToDevice, s));
    bd = hb;
    xd = hb + op.n * nrhs;
  }
  launch_cm_to_rm(bd, dev ? ldb : op.n, op.n, nrhs, ws + plan.in_row * nrhs, nullptr, s);
  hbs_run_plan(op, plan, ws, nrhs, s);
  launch_rm_to_cm(ws + plan.out_row * nrhs, op.n, nrhs, xd, dev ? ldx : op.n, nullptr, s);
  if (!dev) {
    SBX_CUDA(cudaMemcpy2DAsync(x, size_t(ldx) * 8, xd, size_t(op.n) * 8, size_t(op.n) * 8,
                               size_t(nrhs), cudaMemcpyDeviceToHost, s));
    SBX_CUDA(cudaStreamSynchronize(s));
  }
}
}  // namespace

void hbs_solve(HbsOp& op, const double* b, i64 ldb, i64 nrhs, double* x, i64 ldx, bool dev,
               cudaStream_t s) {
  if (!op.solve_plan.built) hbs_build_solve_plan(op);
  run_sweep(op, op.solve_plan, b, ldb, nrhs, x, ldx, dev, s);
}

void hbs_apply(HbsOp& op, const double* v, i64 ldv, i64 nrhs, double* y, i64 ldy, bool dev,
               cudaStream_t s) {
  if (!op.apply_plan.built) hbs_build_apply_plan(op);
  run_sweep(op, op.apply_plan, v, ldv, nrhs, y, ldy, dev, s);
}

}  // namespace sbx
