// Batched small dense linear algebra on sm_100a, one CTA per problem:
// the building blocks of the device compression / inversion / Woodbury
// build (reference Eigen calls: ColPivHouseholderQR, PartialPivLU,
// HouseholderQR, triangular solves and GEMMs).
#pragma once

#include <vector>

#include "common.hpp"

namespace sbx {

// ---------------------------------------------------------------- QR / CPQR
// A (M x n, column-major, lda) factored in place.  pivot=1 follows Eigen's
// ColPivHouseholderQR (first-max pivot on updated norms, xGEQPF downdating
// with direct recomputation under sqrt(eps)); pivot=0 is a plain Householder
// QR (the TSQR row reduction).  With stop_eps > 0 the pivoted loop ends after
// the first step whose |r_jj| <= stop_eps*|r_00| (truncated CPQR: the rows
// of R above that step are final, so the ID is unchanged).
struct QrJob {
  double* a;
  int M, n, lda;
  int pivot;
  int max_steps;
  double stop_eps;
  int* perm;      // n entries (pivoted only): perm[i] = original column at position i
  double* diag;   // min(M, n) entries: |r_jj| (0 after the stop)
  int* steps;     // number of completed steps
};
void qr_batched(const std::vector<QrJob>& jobs, cudaStream_t s);
// Shared memory qr_batched needs to keep one problem on chip (bytes), and
// whether the blocked (LAPACK dlaqps-style) CPQR loop is in use.
size_t qr_smem_need(int M, int n, bool blocked = true);
int cpqr_blocked_enabled();

// Cooperative CPQR for problems too large for one CTA: the CTAs of a group
// own disjoint column slabs of A (kept in global memory / L2), recompute the
// pivot's Householder vector redundantly and meet at one group barrier per
// step.  Columns are not moved: perm[l] is the physical (= original) column
// at logical position l and R(i, l) = A(i, perm[l]).  Pivot choice, the
// Householder convention and the norm downdating are those of qr_kernel.
void cpqr_coop_batched(const std::vector<QrJob>& jobs, cudaStream_t s);

// On-chip cooperative CPQR: like cpqr_coop_batched, but each CTA holds its
// column slab in shared memory for the whole factorisation and publishes
// its pivot candidate before the group barrier (one barrier per step, no
// trailing-matrix traffic).  Problems are packed into co-resident waves.
// cpqr_smem_ctas gives the CTAs a problem needs (0: does not fit on chip).
int cpqr_smem_ctas(int M, int n);
void cpqr_smem_batched(const std::vector<QrJob>& jobs, cudaStream_t s);

// Cluster CPQR: the same on-chip algorithm with one problem per thread-block
// cluster of C <= 16 CTAs (partials and pivot column through DSMEM, hardware
// cluster barrier): no cooperative launch, so it runs beside other streams.
// cpqr_cluster_size gives C (a power of two) or 0 when one cluster is too small.
int cpqr_cluster_size(int M, int n);
void cpqr_cluster_batched(const std::vector<QrJob>& jobs, cudaStream_t s);
// Register-resident cluster CPQR (one problem per cluster of G <= 16 CTAs,
// M <= 1088): returns the layout index (G set) or -1 when it does not apply.
int cpqr_reg_config(int M, int n, int* G);
void cpqr_reg_batched(const std::vector<QrJob>& jobs, cudaStream_t s);
// Row-split cluster CPQR (engine 7, cpqr_rows.cu): one tall problem (M >= 2n)
// per cluster of G <= 8 CTAs, each holding a row slab in shared memory; the
// column norms are replicated, so a step needs two O(n) DSMEM exchanges.
// cpqr_rows_cluster gives the smallest G that fits (0: not applicable).
int cpqr_rows_cluster(int M, int n);
void cpqr_rows_batched(const std::vector<QrJob>& jobs, cudaStream_t s);
// One-exchange row-split cluster CPQR (engine 8, cpqr_push.cu): the same
// slab split, but one pushed exchange per step (unscaled pivot-column dots
// and row j, st.async into every CTA's slot, mbarrier transaction counts).
int cpqr_push_cluster(int M, int n);
void cpqr_push_batched(const std::vector<QrJob>& jobs, cudaStream_t s);
// Register-resident row-split cluster CPQR (engine 9, cpqr_push.cu): the
// slab in registers (<= 32 rows per thread), one pushed exchange and two CTA
// barriers per step, next pivot chosen before the update.
int cpqr_regrows_cluster(int M, int n);
void cpqr_regrows_batched(const std::vector<QrJob>& jobs, cudaStream_t s);
// Blocked QR (engine 10): tall W^T (M <= 1280, n <= 128), one CTA per
// problem; 16-column Householder panels in shared memory, the trailing
// matrix updated in global memory on DMMA, then the CPQR of R0 on chip.
bool bqr_ok(int M, int n);
void bqr_batched(const std::vector<QrJob>& jobs, cudaStream_t s);
// Streaming one-CTA CPQR (M <= 1088): columns beyond the shared-memory slab
// are updated in place in global memory (L2).
bool cpqr_stream_ok(int M, int n);
void cpqr_stream_batched(const std::vector<QrJob>& jobs, cudaStream_t s);

// ---------------------------------------------------------------- ID interpolation
// Given a pivoted factor (R in the upper triangle of a, ld lda, n columns)
// and a rank k: P (n x k, column-major, ldp) with P(J_i, i) = 1 (i < k) and
// P(J_{k+j}, :) = (R11^{-1} R12)(:, j)^T  (idlib.cpp:55-62).  T scratch
// must hold k*(n-k) doubles.
struct InterpJob {
  const double* a;
  int lda, n, k;
  const int* perm;
  const int* colmap;  // R column l stored at physical column colmap[l] (null: l)
  double* P;
  int ldp;
  double* T;
};
void interp_batched(const std::vector<InterpJob>& jobs, cudaStream_t s);

// ---------------------------------------------------------------- GEMM
// C = alpha * op(A) * op(B) + beta * C, column-major; op via trans flags.
struct GemmJob {
  const double* A;
  const double* B;
  double* C;
  int m, n, k;
  int lda, ldb, ldc;
  int ta, tb;
  double alpha, beta;
  // set by gemm_batched: deterministic split-K for long, thin products
  // (partials reduced in a fixed order by a second kernel)
  int splitk = 1;
  int kchunk = 0;
  double* part = nullptr;
};
void gemm_batched(const std::vector<GemmJob>& jobs, cudaStream_t s);

// ---------------------------------------------------------------- LU
// Partial-pivot LU of each square A (in place, column-major), optional
// explicit inverse into inv (ld n), and the Hager/Higham reciprocal
// condition estimate of Eigen's PartialPivLU::rcond() into rcond.
struct LuJob {
  double* a;
  int n, lda;
  int* piv;        // n entries (row i of PA = row piv[i] of A)
  double* inv;     // optional n x n output (ld n)
  double* rcond;   // optional
  double* work;    // 4n doubles scratch (required when rcond requested)
};
void lu_batched(const std::vector<LuJob>& jobs, cudaStream_t s);

// Solve with a factored LU (one problem): X = A^{-1} B in place, B n x nrhs.
void lu_solve(const double* lu, int n, int lda, const int* piv, double* B, int ldb, int nrhs,
              double* scratch, cudaStream_t s);

// Batched block copies dst = src or src^T (column-major).
struct CopyJob {
  const double* src;
  double* dst;
  int rows, cols;  // of the destination block
  int lds, ldd;
  int trans;       // dst(i, j) = src(j, i)
  int pad;
};
void copy_batched(const std::vector<CopyJob>& jobs, cudaStream_t s);

// Row scatter / gather: scatter  dst(map[r], col_off + c) = alpha src(r, c)
//                       gather   dst(r, col_off + c)      = alpha src(map[r], c)
// map == null means identity.
struct ScatterJob {
  const double* src;
  double* dst;
  const i64* map;
  int rows, cols;
  int lds, ldd;
  int col_off;
  int gather;
  double alpha;
};
void scatter_batched(const std::vector<ScatterJob>& jobs, cudaStream_t s);

// Scatter / gather helpers.
void launch_copy2d(const double* src, i64 lds, double* dst, i64 ldd, i64 rows, i64 cols,
                   cudaStream_t s);
void launch_add_identity(double* a, i64 lda, i64 n, cudaStream_t s);

}  // namespace sbx
