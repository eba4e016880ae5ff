/*
 * sbx.h — C-ABI of the B200-native refined-wall Stokes solver.
 *
 * Drop-in boundary for the reference's C++ solver API
 * (/root/reference/proj/include/stokesbie/*.hpp).  The reference exposes
 * Eigen value types and exceptions and has no C ABI or FFI of its own (its
 * python/ binding is an empty stub, proj/python/CMakeLists.txt:1); each entry
 * point below names the reference call it replaces.  Plain pointers and sizes
 * only — no torch or CUDA types in the signatures (streams are `void*`
 * aliases of cudaStream_t, NULL = the library stream).
 *
 * Conventions (mirroring proj/include/stokesbie/common.hpp:11-15,
 * geometry.hpp:60-62):
 *   - unknowns are interleaved per node: scalar index = 2*node + component;
 *   - multi-RHS blocks are n x nrhs, column-major with leading dimension ld;
 *   - handles are immutable after build, so concurrent solves on distinct
 *     streams are legal;
 *   - every function returns a status code (SBX_OK ...) and, on failure, a
 *     thread-local message is available from sbx_last_error() (the
 *     reference's exception text, including SingularMatrixError::where).
 */
#ifndef SBX_H_
#define SBX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (exception classes of common.hpp:20-52, CLI exit codes of
 * tools/bench_main.cpp:42-55). */
enum {
  SBX_OK = 0,
  SBX_INVALID_ARGUMENT = 1,   /* std::invalid_argument from require()        */
  SBX_NONCONVERGENCE = 2,     /* ConvergenceError (GMRES)                     */
  SBX_GEOMETRY_ERROR = 3,     /* GeometryError                                */
  SBX_SINGULAR_MATRIX = 4,    /* SingularMatrixError{where}                   */
  SBX_PROXY_VIOLATION = 5,    /* ProxyViolationError                          */
  SBX_CUDA_ERROR = 6,         /* CUDA / NCCL failure (no CPU fallback)        */
  SBX_RUNTIME_ERROR = 7       /* any other std::runtime_error (e.g. HBS1 I/O) */
};

/* Curve kinds (geometry.hpp:10 CurveKind) and formulations (kernels.hpp:35).
 * SBX_CHANNEL extends the reference's radial kinds with the closed wavy
 * channel of BASELINE configs[3] (in units of h = scale, shifted by center):
 * walls Y = -/+(1 + a sin(k X)), X in [0, Lam] (a = amplitude, Lam = aspect,
 * k = 2 pi n_prongs / Lam), closed by two degree-9 polynomial caps whose
 * coefficients are cos_coef[0..9] (X) and [10..19] (Y) of the right cap,
 * [20..29] / [30..39] of the left cap (chosen so the caps join the walls
 * with matching derivatives up to the fourth).  t in [0, 2 pi) runs bottom
 * wall, right cap, top wall, left cap over the fractions sin_coef[0],
 * sin_coef[1], sin_coef[0], 1 - 2 sin_coef[0] - sin_coef[1] (multiples of
 * 1/n_panels put the joins on panel ends). */
enum { SBX_CIRCLE = 0, SBX_ELLIPSE = 1, SBX_STAR = 2, SBX_FOURIER = 3, SBX_CHANNEL = 4 };
enum { SBX_INTERIOR_DIRICHLET = 0, SBX_EXTERIOR_COMBINED = 1, SBX_MIXED = 2 };

/* Sweep flags. */
enum {
  SBX_TRANSPOSE = 1,     /* hbs_solve_t / hbs_apply_t                        */
  SBX_DEVICE_PTRS = 2,   /* b / x are device pointers (else host, pinned or
                            pageable; copies are issued on the stream)     */
  SBX_ROW_MAJOR = 4      /* with SBX_DEVICE_PTRS, sbx_hbs_solve / _apply only:
                            b / x are n x nrhs ROW-major (ld = row stride
                            >= nrhs), the sweep workspace's own layout, so
                            they move by strided copies instead of
                            transposes (a C-contiguous torch tensor)       */
};

typedef struct sbx_geom_s* sbx_geom;     /* Discretization           */
typedef struct sbx_plan_s* sbx_plan;     /* RefinementPlan           */
typedef struct sbx_hbs_s* sbx_hbs;       /* HbsOperator (device)     */
typedef struct sbx_update_s* sbx_update; /* LowRankUpdate (device)   */
typedef struct sbx_els_s* sbx_els;       /* ElsSolver (device)       */
typedef struct sbx_app_s* sbx_app;       /* A_pp inverse (device)    */
typedef struct sbx_update_cache_s* sbx_update_cache; /* snapshot update cache */
typedef struct sbx_comm_s* sbx_comm;     /* communicator set (multi-GPU) */
typedef struct sbx_els_shard_s* sbx_els_shard; /* ElsSolver on a subtree partition */

/* CurveParams (geometry.hpp:14-26). */
typedef struct {
  int32_t kind;
  double center_x, center_y, scale;
  int32_t flip_normal, n_prongs;
  double amplitude, aspect;
  int32_t n_cos, n_sin;          /* fourier coefficient counts (<= 64 each) */
  double cos_coef[64], sin_coef[64];
} sbx_curve;

/* HbsOptions (hbs.hpp:39-46). n_proxy is accepted and, as in the reference
 * (hbs.cpp:276-279), ignored: compression always starts at 64 samples. */
typedef struct {
  double eps;          /* 1e-10 */
  int64_t leaf_nodes;  /* 64    */
  int32_t n_proxy;     /* 64    */
  double bas_factor;   /* 1.5   */
  double div_factor;   /* 3.0   */
} sbx_hbs_options;

const char* sbx_last_error(void);
int sbx_init(int device);                  /* selects the CUDA device */
int sbx_sync(void);                        /* waits for the library stream */
void* sbx_stream(void);                    /* the library stream (cudaStream_t) */

/* ---------------------------------------------------------- geometry
 * panelize (geometry.hpp:103), build_discretization + add_holes
 * (geometry.hpp:104-106,134-135), refine (:120-121), coarsen (:124),
 * panels_near_point (:139-140).  Node generation is O(N) host work. */
int sbx_geom_create(const sbx_curve* curve, int n_panels, int q, sbx_geom* out);
int sbx_geom_add_holes(sbx_geom wall, int n_holes, const sbx_curve* holes,
                       const int32_t* n_panels, const int32_t* q, sbx_geom* out,
                       sbx_plan* plan);
int sbx_geom_destroy(sbx_geom g);
int sbx_geom_info(sbx_geom g, int64_t* n_nodes, int64_t* n_panels, int64_t* n_components);
/* 9*n doubles: x, y, nx, ny, tx, ty, w, curvature, param; panel_of n int64 */
int sbx_geom_nodes(sbx_geom g, double* out9, int64_t* panel_of);
int sbx_panels_near_point(sbx_geom g, double px, double py, double radius,
                          int64_t* out, int64_t cap, int64_t* count);
int sbx_refine(sbx_geom g, const int64_t* panel_ids, int64_t n, int m, sbx_geom* out,
               sbx_plan* plan);
int sbx_coarsen(sbx_geom g, sbx_plan plan, sbx_geom* out);
int sbx_plan_destroy(sbx_plan p);
int sbx_plan_sizes(sbx_plan p, int64_t* n_k, int64_t* n_c, int64_t* n_p);
int sbx_plan_maps(sbx_plan p, int64_t* kept_old, int64_t* kept_new, int64_t* cut_old,
                  int64_t* added_new);

/* ---------------------------------------------------------- entries / data
 * BieAssembler::submatrix (nystrom.hpp:30) evaluated on the device;
 * boundary_data (nystrom.hpp:116-117). Host in/out buffers. */
int sbx_submatrix(sbx_geom g, int formulation, double mu, const int64_t* rows, int64_t nr,
                  const int64_t* cols, int64_t nc, double* out);
/* evaluate_solution (nystrom.hpp:137-139, nystrom.cpp:408-448): velocity at
 * n_targets points (x, y interleaved) from nrhs densities (2N x nrhs,
 * column-major, ld ldt); velocity: 2 x n_targets per density (stacked);
 * pressure (optional, with_pressure): n_targets per density; near_boundary
 * (optional): 1 where the closest node lies within its panel's length. */
int sbx_evaluate_solution(sbx_geom g, int formulation, double mu, const double* tau, int64_t ldt,
                          int64_t nrhs, const double* targets, int64_t n_targets, int with_pressure,
                          double* velocity, double* pressure, uint8_t* near_boundary);
int sbx_boundary_data(sbx_geom g, int64_t n_src, const double* src_xyf, double mu,
                      double* out);

/* ---------------------------------------------------------- HBS
 * hbs_compress (hbs.hpp:80, on the device), hbs_invert (:85),
 * hbs_solve/_t, hbs_apply/_t (:87-94), hbs_save/hbs_load "HBS1" (:97-98). */
int sbx_hbs_compress(sbx_geom g, int formulation, double mu, const sbx_hbs_options* opts,
                     sbx_hbs* out);
int sbx_hbs_compress_subset(sbx_geom g, int formulation, double mu, const int64_t* nodes,
                            int64_t n_nodes, const sbx_hbs_options* opts, sbx_hbs* out);
/* hbs_compress over a caller-supplied entry oracle: the reference's plugin
 * point HbsSource::entries (hbs.hpp:19-31), swapped in by its tests
 * (test_hbs.cpp:186-245).  The geometry g still supplies the points (tree,
 * proxy circles) and the source normals / weights / kernel roles of the
 * proxy functionals; `entries` supplies every block the compression draws
 * (leaf diagonal blocks, near rows of the IDs, sibling couplings): it fills
 * the column-major nr x nc block of scalar indices (rows, cols), on the
 * calling thread, and must not call back into the library.
 * with_completion = 0 drops the rank-one completion functionals
 * (HbsSource::row_null / col_null empty). */
typedef void (*sbx_entries_fn)(void* ctx, const int64_t* rows, int64_t nr, const int64_t* cols, int64_t nc,
                               double* out);
int sbx_hbs_compress_custom(sbx_geom g, int formulation, double mu, sbx_entries_fn entries, void* ctx,
                            int with_completion, const sbx_hbs_options* opts, sbx_hbs* out);
int sbx_hbs_invert(sbx_hbs h);
int sbx_hbs_destroy(sbx_hbs h);
int sbx_hbs_solve(sbx_hbs h, const double* b, int64_t ldb, int64_t nrhs, double* x,
                  int64_t ldx, int flags, void* stream);
int sbx_hbs_apply(sbx_hbs h, const double* v, int64_t ldv, int64_t nrhs, double* y,
                  int64_t ldy, int flags, void* stream);
/* Subtree-partitioned solve across G = 2^g ranks (one
 * process per GPU, the caller owns the collective).  Rank p owns the
 * subtree rooted at the p-th BFS node of depth g: old-mesh scalar rows
 * [row0, row1).  kmax = largest subtree-root skeleton rank (rows of one
 * exchanged hat block).  Sequence per solve:
 *   sbx_hbs_solve_shard_up(b_local -> hat_out)          local up-sweep
 *   all-gather of the G hat blocks (kmax x nrhs, row-major) in rank order
 *   sbx_hbs_solve_shard_down(hats -> x_local)           top g levels
 *                                                       (redundant) + local
 *                                                       down-sweep
 * Replaces hbs_solve (hbs.cpp:589-625) split at depth g; the reference is
 * single-process, so there is no reference signature to mirror. */
int sbx_hbs_shard_info(sbx_hbs h, int G, int p, int64_t* row0, int64_t* row1, int64_t* kmax);
int sbx_hbs_solve_shard_up(sbx_hbs h, int G, int p, const double* b_local, int64_t ldb,
                           int64_t nrhs, double* hat_out, int flags, void* stream);
int sbx_hbs_solve_shard_down(sbx_hbs h, int G, int p, const double* hats, int64_t nrhs,
                             double* x_local, int64_t ldx, int flags, void* stream);
int sbx_hbs_save_hbs1(sbx_hbs h, const char* path);
int sbx_hbs_load_hbs1(const char* path, sbx_hbs* out);
/* info[0..13]: n, nodes, total_skeleton, max_block_drawn, has_inverse,
 * solve_factor_doubles, max_depth, max_k, apply_factor_doubles, leaf_nodes,
 * top_depth, top_size (the solve's collapsed top: depth and K of the dense
 * map, 0 when every level runs; set once a solve plan exists),
 * arena_doubles (the factors this handle stores on the device), sharded
 * (1: a subtree-sharded operator, sbx_hbs_compress_sharded) */
int sbx_hbs_info(sbx_hbs h, int64_t* info);
int sbx_hbs_node_ranks(sbx_hbs h, int64_t* k, int64_t cap);

/* ---------------------------------------------------------- low-rank update
 * compress_update(blocks, proxy, eps, TwoStepId, {seed}) (lowrank.hpp:59-62),
 * with BlockSource(old, new, plan) and make_proxy_geometry(new, plan) built
 * internally (nystrom.hpp:75-76, proxy.hpp:48-49). */
int sbx_update_compress(sbx_geom old_g, sbx_geom new_g, sbx_plan plan, int formulation,
                        double mu, double eps, uint64_t seed, sbx_update* out);
int sbx_update_destroy(sbx_update u);
/* info: k, k1, kc.k, kp.k, pk.k, n_ext, nk2, nc2, np2 */
int sbx_update_info(sbx_update u, int64_t* info);
/* which: 0 L (n_ext x k), 1 R (k x n_ext); column-major host copies */
int sbx_update_factor(sbx_update u, int which, double* out);
/* Tier-1 injection of externally computed factors (dump_matrix exchange,
 * nystrom.hpp:141-143). */
int sbx_update_from_factors(sbx_plan plan, const double* L, const double* R, int64_t n_ext,
                            int64_t k, sbx_update* out);

/* ---------------------------------------------------------- ELS / Woodbury
 * els_build (els.hpp:42-44), els_solve / els_solve_raw (els.hpp:57,65),
 * density_on_refined (els.hpp:69). */
int sbx_els_build(sbx_hbs a_oo, sbx_geom old_g, sbx_geom new_g, sbx_plan plan,
                  sbx_update upd, int formulation, double mu, sbx_els* out);
int sbx_els_destroy(sbx_els e);
/* The added-unknown diagonal block's inverse alone (els.cpp:111-118: dense
 * LU for 2 N_p <= 2048 scalars, else its own HBS), for callers that split the
 * extended system across ranks (parallel.ShardedWoodbury: the block lives on
 * one rank).  new_g must outlive the handle.  info: n_p (scalars), is_hbs.
 * sbx_app_solve: out = A_pp^{-1} v (flags & SBX_TRANSPOSE: A_pp^{-T} v),
 * n_p x nrhs column-major; flags & SBX_DEVICE_PTRS for device buffers. */
int sbx_app_build(sbx_geom new_g, sbx_plan plan, int formulation, double mu, double eps, sbx_app* out);
int sbx_app_destroy(sbx_app a);
int sbx_app_info(sbx_app a, int64_t* info);
int sbx_app_solve(sbx_app a, const double* v, int64_t ldv, int64_t nrhs, double* out, int64_t ldo, int flags,
                  void* stream);
/* info[0..5]: n_k, n_c, n_p (scalars), k, app_is_hbs, app_solve_doubles (factor
 * doubles one A_pp solve streams: its HBS factors, or n_p^2 for the dense inverse) */
int sbx_els_info(sbx_els e, int64_t* info);
/* g_n: (n_k + n_p) x nrhs (kept, added); tau_n same shape. */
int sbx_els_solve(sbx_els e, const double* g_n, int64_t ldg, int64_t nrhs, double* tau_n,
                  int64_t ldt, int flags, void* stream);
/* g_ext: n_ext x nrhs (kept, cut, added).  flags & SBX_TRANSPOSE:
 * els_solve_raw_t (els.cpp:154-163), y = ELS^{-T} g_ext. */
int sbx_els_solve_raw(sbx_els e, const double* g_ext, int64_t ldg, int64_t nrhs, double* y,
                      int64_t ldy, int flags, void* stream);
/* els_apply_forward (els.cpp:181-186): out = (Atilde + L R) v on the extended
 * system (host buffers, n_ext x nrhs, column-major). */
int sbx_els_apply_forward(sbx_els e, const double* v, int64_t ldv, int64_t nrhs, double* out,
                          int64_t ldo);
/* els_apply_forward_t (els.cpp:188-193): out = (Atilde + L R)^T v. */
int sbx_els_apply_forward_t(sbx_els e, const double* v, int64_t ldv, int64_t nrhs, double* out,
                            int64_t ldo);
/* GMRES / PGMRES-Local (gmres.cpp:14-126 driven as scenario.cpp:694-727):
 * solves the refined system on the (kept, added) unknowns with operator
 * els_apply_forward (els.cpp:181-186) and, when precond != 0, the left
 * preconditioner els_solve.  Host g_n in (n_k + n_p), tau_n out; n_iter and
 * up to history_cap relative residuals (starting at 1).  Returns
 * SBX_NONCONVERGENCE (tau_n = last iterate) on stagnation or budget. */
int sbx_els_gmres(sbx_els e, const double* g_n, double* tau_n, int precond, double tol,
                  int64_t max_iter, int64_t restart, int64_t* n_iter, double* history,
                  int64_t history_cap);
int sbx_els_density_on_refined(sbx_els e, const double* tau_n, double* out);
/* conditioning_report (els.cpp:225-270), estimator route: out[7] = kappa_w,
 * kappa_l, kappa_r, kappa_ext, kappa_tilde, bound, bound_holds (0/1).
 * kappa_w / kappa_l / kappa_r are exact (singular values of W and of the R
 * factors of L and R^T); kappa_ext / kappa_tilde by `iters` rounds of seeded
 * power iteration on the device operators and their solves (linop.cpp:17-43;
 * the reference uses 80). */
int sbx_els_conditioning(sbx_els e, int iters, double* out);
/* conditioning_report(s, dense_oracles_allowed) (els.cpp:225-270) with the
 * route chosen: dense != 0 takes kappa_tilde / kappa_ext from the singular
 * values of the assembled Atilde and Atilde + L R (device Jacobi SVD,
 * n_ext <= 12000; the meshes the ELS was built on must still be alive);
 * dense == 0 is sbx_els_conditioning.  Same 7 outputs. */
int sbx_els_conditioning_report(sbx_els e, int dense, int iters, double* out);
/* Woodbury factors for inspection: X (n_ext x k), W (k x k). */
int sbx_els_xw(sbx_els e, double* X, double* W);

/* compress_update with the CompressionMode (lowrank.hpp:17, lowrank.cpp:366-373):
 * SBX_TWO_STEP_ID is sbx_update_compress; SBX_SVD_OPTIMAL is svd_optimal
 * (lowrank.cpp:329-362): dense truncated SVDs of the kc / kp / pk blocks
 * re-truncated through the stacked factor (device Jacobi SVD; a diagnostic
 * mode for small refinements, like the reference's). */
enum { SBX_TWO_STEP_ID = 0, SBX_SVD_OPTIMAL = 1 };
int sbx_update_compress_mode(sbx_geom old_g, sbx_geom new_g, sbx_plan plan, int formulation, double mu,
                             double eps, uint64_t seed, int mode, sbx_update* out);

/* ---------------------------------------------------------- snapshot update cache
 * run_snapshot_batch's cache (scenario.cpp:836-899): updates are determined
 * by the refinement plan alone, so identical (panel ids, m) -- at the same
 * eps, formulation, mu and seed -- share one compression.  On a miss the
 * update is compressed exactly as sbx_update_compress does and stored; on a
 * hit the stored update is returned (*hit = 1).  Returned handles are
 * independent (destroy each); the cache keeps its own reference. */
int sbx_update_cache_create(sbx_update_cache* out);
int sbx_update_cache_destroy(sbx_update_cache c);
int sbx_update_cache_compress(sbx_update_cache c, sbx_geom old_g, sbx_geom new_g, sbx_plan plan,
                              const int64_t* panel_ids, int64_t n_panels, int m, int formulation, double mu,
                              double eps, uint64_t seed, sbx_update* out, int* hit);
int sbx_update_cache_stats(sbx_update_cache c, int64_t* entries, int64_t* hits, int64_t* misses);

/* ---------------------------------------------------------- multi-GPU
 * One process per GPU.  A communicator set is created once per rank from a
 * 128-byte NCCL unique id made by rank 0 and distributed by the caller (any
 * side channel); call it with the rank's device current (sbx_init).  NCCL is
 * loaded at run time (an NCCL already in the process, e.g. torch's, is
 * reused).  The loopback variant makes `world` members of one in-process
 * group (member r driven by its own host thread, exchanges by device copies):
 * the same protocol on one GPU, for tests and emulation.
 *
 * Subtree partition: for world = G = 2^g, rank p owns the subtree rooted at
 * the p-th BFS node of depth g, i.e. old-mesh rows [row0, row1) of
 * sbx_hbs_shard_info.  sbx_hbs_solve_sharded: local up-sweep, all-gather of
 * the G subtree-root hats (the only exchange), top levels redundantly, local
 * down-sweep; b_local / x_local are this rank's rows (column-major). */
int sbx_comm_unique_id(uint8_t* id128);
/* hbs_compress over the subtree partition: every rank of
 * the communicator set calls it; rank p compresses the nodes of its subtree
 * and, redundantly, the top levels, exchanging each level's skeleton lists
 * (and the subtree roots' couplings) through the communicator, and keeps
 * only those factors.  sbx_hbs_invert then inverts the subtree and the top
 * (the subtree roots' dhat blocks exchanged); the operator solves through
 * sbx_hbs_solve_sharded on the same communicator, which must outlive it. */
int sbx_hbs_compress_sharded(sbx_geom g, int formulation, double mu, const sbx_hbs_options* opts, sbx_comm c,
                             sbx_hbs* out);
int sbx_comm_create(const uint8_t* id128, int world, int rank, sbx_comm* out);
int sbx_comm_create_loopback(int world, sbx_comm* members);
int sbx_comm_destroy(sbx_comm c);
int sbx_comm_info(sbx_comm c, int* world, int* rank);
int sbx_hbs_solve_sharded(sbx_hbs h, sbx_comm c, const double* b_local, int64_t ldb, int64_t nrhs, double* x_local,
                          int64_t ldx, int flags, void* stream);
/* Woodbury on the same ownership (els.cpp:80-179): X = Atilde^{-1} L and the
 * columns of R follow the row ownership, A_pp lives on rank 0, R X and R y
 * are all-reduced, W^{-1} is formed on every rank (same rcond gate and
 * message as sbx_els_build).  info: row0, row1, n_p on this rank (0 except
 * rank 0), k, n_ext, world, rank.  rows: the ext row of each owned row, in
 * old-mesh order (rows = row1 - row0).  solve: g_local / y_local are the
 * owned rows in that order, g_p / y_p the added rows (rank 0 only; null
 * elsewhere). */
int sbx_els_shard_build(sbx_hbs a_oo, sbx_comm c, sbx_geom old_g, sbx_geom new_g, sbx_plan plan, sbx_update upd,
                        int formulation, double mu, void* stream, sbx_els_shard* out);
int sbx_els_shard_info(sbx_els_shard e, int64_t* info);
int sbx_els_shard_rows(sbx_els_shard e, int64_t* ext_rows);
int sbx_els_shard_solve(sbx_els_shard e, const double* g_local, int64_t ldg, const double* g_p, int64_t ldgp,
                        int64_t nrhs, double* y_local, int64_t ldy, double* y_p, int64_t ldyp, int flags,
                        void* stream);
int sbx_els_shard_destroy(sbx_els_shard e);

/* ---------------------------------------------------------- dense interchange
 * dump_matrix / load_matrix (nystrom.cpp:450-477; nystrom.hpp:142-143):
 * u32 rows, u32 cols, then the entries row by row as doubles.  Host buffers
 * are column-major with leading dimension ld (>= rows). */
int sbx_dump_matrix(const char* path, const double* m, int64_t rows, int64_t cols, int64_t ld);
int sbx_load_matrix_dims(const char* path, int64_t* rows, int64_t* cols);
int sbx_load_matrix(const char* path, double* out, int64_t ld);
/* The update factors L (n_ext x k) and R (k x n_ext) as two dump_matrix
 * files, and back: tier-1 hand-over of externally computed factors (e.g. the
 * reference's) into sbx_els_build, like sbx_update_from_factors. */
int sbx_update_dump(sbx_update u, const char* path_L, const char* path_R);
int sbx_update_load(sbx_plan plan, const char* path_L, const char* path_R, sbx_update* out);

/* ---------------------------------------------------------- diagnostics
 * Number of sbx kernels launched since the last reset (bench evidence). */
int64_t sbx_kernel_launches(int reset);
/* CUDA-event timing of the named hot kernels on the stream they run on
 * ("sweep_flow_dmma", "sweep_flow_gemv"): enable, then read the total
 * milliseconds and launch count since the last reset. */
int sbx_kernel_timing(int enable);
int sbx_kernel_time(const char* name, int reset, double* total_ms, int64_t* count);
/* Algorithmic flops attributed to a timed kernel family while timing is on
 * ("id_factor": every CPQR launch of the interpolative decompositions, 4
 * flops per trailing-block entry of each pivoted Householder step taken). */
int sbx_kernel_flops(const char* name, int reset, double* flops);

/* Device row ID of a host matrix W (m x n, column-major) — idlib.cpp:73-99
 * (row_id; forced >= 0 selects row_id_rank).  engine: 0 auto, 1 one CTA per
 * problem, 2 cooperative multi-CTA (slabs in L2), 3 cooperative on chip
 * (slabs in shared memory), 4 one thread-block cluster per problem (slabs in
 * shared memory), 5 one cluster per problem with the slab in registers.
 * J: m entries, P: m*min(m,n) doubles. */
int sbx_row_id(const double* w, int64_t m, int64_t n, double eps, int64_t forced, int engine,
               int64_t* k, int64_t* J, double* P);

/* Explicit inverse and Eigen-style reciprocal condition estimate of a dense
 * host matrix a (n x n, column-major, n <= 2048) through the device path the
 * Woodbury operator W and the dense A_pp use — els.cpp:111-127
 * (PartialPivLU + rcond()).  inv: n*n doubles. */
int sbx_dense_inverse(const double* a, int64_t n, double* inv, double* rcond);

/* C = A B for host column-major operands (A m x k, B k x n) through the
 * device GEMM dispatcher the ELS uses (W = I + R X, els.cpp:124; R y and
 * X z of the Woodbury solve, els.cpp:150) — DMMA tiles, split-K with a
 * fixed-order reduction, the thin-product kernel for small outputs over a
 * long inner dimension. */
int sbx_matmul(const double* a, int64_t m, int64_t k, const double* b, int64_t n, double* c);

#ifdef __cplusplus
}
#endif
#endif /* SBX_H_ */
