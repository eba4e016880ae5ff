// Device-resident HBS operator (reference HbsOperator, hbs.hpp:48-74).
//
// The tree topology and skeleton index lists stay on the host (they drive
// launch plans); every factor lives in one device arena, packed level-major
// so each sweep level streams one contiguous range of HBM:
//   fg_i = [f_i; g_i]   (k_i + c_i) x c_i   up-sweep of the solve (one GEMV)
//   e_i                  c_i x k_i           down-sweep of the solve
//   vd_i = [v_i^T; d_i]  (k_i + c_i) x c_i   up-sweep of the apply (leaves;
//                                            internal nodes store v_i^T only)
//   u_i                  c_i x k_i           down-sweep of the apply
//   b_sib_i              k_i x k_sib         sibling coupling
//   root_g               c_0 x c_0
// All blocks are column-major (Eigen order) so HBS1 files map 1:1.
#pragma once

#include <atomic>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "common.hpp"

namespace sbx {

struct HbsNodeH {
  i64 begin = 0, end = 0, parent = -1, left = -1, right = -1;
  int depth = 0;
  i64 k = 0;
  i64 c = 0;  // candidate count: 2*(end-begin) at a leaf, k_l + k_r above
  std::vector<i64> row_skel, col_skel;
  bool is_leaf() const { return left < 0; }
  // arena offsets (doubles), -1 when absent
  i64 o_fg = -1, o_e = -1, o_vd = -1, o_u = -1, o_b = -1, o_dhat = -1, o_v = -1;
};

// One row-tiled product  D[rows] = A * B (+ P)  inside a sweep level.
// Offsets are in doubles (A, into the factor arena) or in rows of the
// row-major sweep workspace (B, P, D1, D2; one row = nrhs doubles).
// Producers one sweep task may wait on (the collapsed top of the tree reads
// the hats of up to 2^5 boxes).
constexpr int kMaxDep = 32;

struct SweepTask {
  i64 a_off;
  int lda, m, K;
  i64 b_row, p_row, d1_row, d2_row;
  int split;  // rows < split go to D1, the rest to D2 (row - split)
  int ndep;   // tasks whose outputs this task reads (dataflow sweep)
  int dep[kMaxDep];
};

// One work item of the dataflow sweep: rows [row0, row0 + tile) x column
// tile ct of task `task`, over the K range [kb, ke).  Items of a split-K
// tile (nsplit > 1) write partial tiles at `poff` (+ ks * tile size); the
// last one to finish (tile counter cidx) sums them in split order.
struct FlowItem {
  int task, row0, ct, ks;
  int nsplit, cidx, kb, ke;
  long long poff;
  int tile, pad;  // rows of this item
};

// Everything one dataflow item needs, denormalised so a CTA can prefetch the
// descriptor of its next item with one asynchronous copy.
struct alignas(16) ItemDesc {
  FlowItem it;
  SweepTask t;
  int need[kMaxDep];  // completed items awaited per producer task (same column tile)
};

struct SweepLevel {
  std::vector<SweepTask> tasks;
  i64 first_task = 0;  // index into the flattened device task table
  int max_k = 0;       // largest K in the level (smem sizing)
  int ksplit = 0;      // > 0: split K of this level's full row tiles this many ways
};

struct SweepPlan {
  std::vector<SweepLevel> levels;  // launch order
  i64 ws_rows = 0;                 // workspace rows (x nrhs doubles)
  i64 in_row = 0, out_row = 0;     // input / output vector regions
  int n_tasks = 0;
  DevBuf<SweepTask> d_tasks;
  std::vector<SweepTask> h_tasks;  // host copy of the flattened task table
  // work items (task, row0, col tile), per-level ranges, and the per-(task,
  // col tile) completion counters of the dataflow sweep, one set per
  // (tile, column-tile count) key: a step alternates block widths (the
  // Woodbury build's u columns, the solve's RHS) without rebuilding them
  std::map<int, std::unique_ptr<struct FlowCache>> flows;
  std::atomic<bool> built{false};
};

struct FlowCache {
  std::vector<int2> level_items;
  DevBuf<FlowItem> d_flow_items;
  DevBuf<ItemDesc> d_descs;  // per flow item (dataflow kernel)
  DevBuf<int> d_needs;       // items per task and column tile (dependency counts)
  i64 partial_elems = 0;     // split-K partial tiles (doubles)
  int n_tile_cnt = 0;
  i64 n_flow_items = 0;
};

// Mutable per-call state of a sweep: the row-major workspace, host-pointer
// staging, the dataflow completion counters and split-K partial tiles.  One
// set per stream (HbsOp::scratch), so concurrent solves on distinct streams
// against one operator never share any of it.
struct SweepScratch {
  DevBuf<double> ws, io, partials;
  DevBuf<int> counters;
  // the dataflow kernel zeroes the counters it used before it exits, so a
  // memset is only needed for memory it has not run over yet
  const int* counters_zeroed = nullptr;
  size_t counters_zeroed_n = 0;
  StreamMark mark;  // end of the last sweep on this stream
};

struct ShardPlans;
class Collective;

struct HbsOp {
  i64 n = 0, leaf_nodes = 64;
  double eps = 0.0;
  bool has_inverse = false;
  bool has_apply = false;
  i64 max_block_drawn = 0;
  int max_depth = 0;
  std::vector<HbsNodeH> nodes;
  std::vector<std::string> notes;
  i64 o_root_g = -1;
  // Collapsed top of the tree (sweep.cu hbs_build_top): the solve's levels
  // above depth top_L fold into one dense K x K map (at o_top in the arena)
  // from the stacked up-sweep hats of the depth-top_L boxes to their
  // down-sweep inputs; top_L == 0 runs every level.
  int top_L = 0;
  i64 o_top = -1, top_K = 0, top_cap = 0;
  // smallest reciprocal condition number of each node's x and skeleton
  // blocks seen by the inverse (hbs.cpp:429 gates); empty when unknown
  // (an inverse loaded from HBS1).  The top only collapses over
  // well-conditioned levels: an explicit product of ill-conditioned
  // factors loses the accuracy the level-by-level sweep keeps.
  std::vector<double> node_rcond;
  DevBuf<double> arena;
  i64 arena_used = 0;
  SweepPlan solve_plan, apply_plan;
  // Transposed factors in the SAME layout (hbs_solve_t / hbs_apply_t run the
  // unchanged plans over this arena): fg <- [e^T; g^T], e <- f^T,
  // root_g <- root_g^T; vd <- [u^T; d^T], u <- v, b_l <- b_r^T.  Built on
  // first use.
  DevBuf<double> arena_t;
  bool t_solve = false, t_apply = false;
  std::unique_ptr<struct ShardPlans> shard;  // subtree-partitioned solve (multi-GPU)
  // Subtree-sharded build and storage (multi-GPU): rank
  // shard_p of shard_G = 2^shard_g compresses and inverts the nodes of its
  // subtree (depth >= shard_g) and, redundantly, the top levels; `stored`
  // marks the nodes whose factors live in this arena (its subtree, the top,
  // and the G subtree roots' coupling / dhat blocks the top inverse reads).
  // Empty: an unsharded operator.  `comm` carries the build's exchanges.
  int shard_G = 1, shard_p = 0, shard_g = 0;
  std::vector<char> stored;
  Collective* comm = nullptr;
  bool sharded() const { return !stored.empty(); }
  bool has(size_t i) const { return stored.empty() || stored[i] != 0; }
  // Lazily built shared state (plans, flow items, transposed arena,
  // collapsed top, shard plans) is created under `mu`; everything a call
  // mutates lives in its stream's scratch.  After the first call on a
  // handle, concurrent calls on distinct streams only contend for `mu`
  // while enqueueing.
  std::recursive_mutex mu;
  PerStream<SweepScratch> scratch;
  SweepScratch& scratch_for(cudaStream_t s) { return scratch.get(s); }
  // Waits for every call still in flight on any stream (handle destruction).
  void drain() {
    scratch.for_each([](SweepScratch& x) { x.mark.wait(); });
  }

  i64 total_skeleton() const {
    i64 t = 0;
    for (const auto& nd : nodes) t += nd.k;
    return t;
  }
  i64 sib(i64 id) const {
    const auto& p = nodes[size_t(nodes[size_t(id)].parent)];
    return p.left == id ? p.right : p.left;
  }
  // Algorithmic bytes of one solve sweep: factor doubles.
  i64 solve_factor_doubles() const;
  i64 apply_factor_doubles() const;
};

// Computes node candidate sizes c and the level-major arena layout, then
// allocates the arena (contents undefined).
void hbs_layout(HbsOp& op);

// HBS1 (hbs.cpp:681-808) <-> device arena.
std::unique_ptr<HbsOp> hbs_load_hbs1(const std::string& path, cudaStream_t s);
void hbs_save_hbs1(const HbsOp& op, const std::string& path, cudaStream_t s);

// Sweeps.  b/x are column-major n x nrhs with leading dimensions; `dev`
// says whether they are device pointers.
void hbs_solve(HbsOp& op, const double* b, i64 ldb, i64 nrhs, double* x, i64 ldx, bool dev,
               cudaStream_t s);
void hbs_apply(HbsOp& op, const double* v, i64 ldv, i64 nrhs, double* y, i64 ldy, bool dev,
               cudaStream_t s);

// Row-major workspace form, for callers that already hold the sweep input
// in `ws` row layout (the ELS path): runs the planned levels only.
// One right-hand side may be read from / written to the caller's vectors
// directly (no copy into the workspace's input / output regions).
struct SweepDirectIo {
  const double* in = nullptr;
  double* out = nullptr;
  i64 in_row = 0, out_row = 0, n = 0;
};
void hbs_run_plan(HbsOp& op, SweepPlan& plan, double* ws, i64 nrhs, cudaStream_t s,
                  const double* fac = nullptr,
                  const SweepDirectIo* io = nullptr);
// Builds (and uploads) the dataflow item tables of `plan` for blocks of nrhs
// right-hand sides ahead of the first sweep of that width.
void hbs_prebuild_flow(HbsOp& op, SweepPlan& plan, i64 nrhs, cudaStream_t s);
// Column-major rows x nrhs block through `plan` on the stream's scratch:
// input row i goes to sweep row map[i] (identity when map is null), output
// row i comes from sweep row map[i]; `transposed` sweeps the transposed
// arena (hbs_ensure_transpose first).
void hbs_sweep_rows(HbsOp& op, SweepPlan& plan, const double* in, i64 ldi, i64 rows, i64 nrhs, double* out,
                    i64 ldo, const i64* map, bool transposed, cudaStream_t s);
// Device blocks already in the workspace layout (n x nrhs row-major, row
// stride ldb / ldx >= nrhs): solve (apply = false) or apply, plain or
// transposed, with strided copies in and out (sbx.h SBX_ROW_MAJOR).
void hbs_sweep_rm(HbsOp& op, bool apply, bool transpose, const double* b, i64 ldb, i64 nrhs, double* x, i64 ldx,
                  cudaStream_t s);
// hbs.cpp:627-664 / :546-587: transposed solve and apply.
void hbs_solve_t(HbsOp& op, const double* b, i64 ldb, i64 nrhs, double* x, i64 ldx, bool dev, cudaStream_t s);
void hbs_apply_t(HbsOp& op, const double* v, i64 ldv, i64 nrhs, double* y, i64 ldy, bool dev, cudaStream_t s);
// Builds the transposed arena parts (solve and/or apply) if missing.
void hbs_ensure_transpose(HbsOp& op, bool solve, bool apply, cudaStream_t s);
void hbs_build_solve_plan(HbsOp& op);
void hbs_build_apply_plan(HbsOp& op);
// The same, built once under op.mu on first use (thread safe).
void hbs_ensure_solve_plan(HbsOp& op);
void hbs_ensure_apply_plan(HbsOp& op);

// Subtree-partitioned solve: rank p of G = 2^g owns the
// subtree rooted at the p-th BFS node of depth g, i.e. old-mesh scalar rows
// [row0, row1).  shard_up runs the local up-sweep and packs the subtree
// root's hat (k_p x nrhs, zero-padded to kmax rows, row-major) into hat_out;
// after the caller all-gathers the G hats, shard_down runs the top g levels
// redundantly and the local down-sweep into x_local.
struct ShardPlans {
  int G = 0, p = -1, g = 0;
  i64 row0 = 0, row1 = 0, kmax = 0;
  std::vector<i64> roots;  // BFS ids of the G subtree roots
  SweepPlan up, top, down;
};
ShardPlans& hbs_shard(HbsOp& op, int G, int p);
void hbs_solve_shard_up(HbsOp& op, int G, int p, const double* b_local, i64 ldb, i64 nrhs, double* hat_out,
                        bool dev, cudaStream_t s);
void hbs_solve_shard_down(HbsOp& op, int G, int p, const double* hats, i64 nrhs, double* x_local, i64 ldx,
                          bool dev, cudaStream_t s);

// Row stride (doubles) of the row-major sweep workspace for nrhs columns:
// even above one column so 64-column B tiles move as 16-byte cp.async.cg.
inline i64 sweep_ld(i64 nrhs) { return nrhs > 1 ? (nrhs + 1) & ~i64(1) : 1; }

// Column-major (ld) <-> row-major (nrhs fastest, row stride ldw) with an
// optional row map: dst_row(i) = map ? map[i] : i.
void launch_cm_to_rm(const double* src, i64 ld, i64 n, i64 nrhs, double* dst, i64 ldw, const i64* map,
                     cudaStream_t s);
void launch_rm_to_cm(const double* src, i64 ldw, i64 n, i64 nrhs, double* dst, i64 ld, const i64* map,
                     cudaStream_t s);

}  // namespace sbx
