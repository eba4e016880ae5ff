// Device entry oracle: the 2x2 kernel blocks of the completed Stokes BIE
// (reference BieAssembler::fill_block, nystrom.cpp:80-172) and the proxy
// interaction blocks used by the compressions (hbs.cpp:131-189,
// proxy.cpp:136-162), evaluated by sm_100a kernels.
#pragma once

#include "common.hpp"
#include "geometry.hpp"

namespace sbx {

// POD view handed to kernels.
struct EntryView {
  const double *x, *y, *nx, *ny, *w, *kappa, *tx, *ty;
  const int* comp;
  const i64* map;  // node subset map (make_hbs_source_subset) or null
  double jump;
  double mu;
  int form;        // SBX_INTERIOR_DIRICHLET / EXTERIOR / MIXED
  // single-layer tables (SlTables, geometry.hpp); null without single-layer components
  const int* sl_i;
  const double *sl_d, *sl_lam, *sl_tab;
  i64 sl_n;
  int sl_qmax;
};

// A caller-supplied entry oracle (the reference's HbsSource::entries plugin,
// hbs.hpp:19-31): fn fills the column-major nr x nc block of the scalar
// indices (rows, cols) on the host.  with_completion = false drops the
// rank-one completion functionals of the compression (HbsSource::row_null /
// col_null left empty).
struct HostEntries {
  void (*fn)(void* ctx, const i64* rows, i64 nr, const i64* cols, i64 nc, double* out) = nullptr;
  void* ctx = nullptr;
  bool with_completion = true;
  // column-major nr x nc block (host)
  std::vector<double> block(const i64* rows, i64 nr, const i64* cols, i64 nc) const;
};

class EntryOracle {
 public:
  EntryOracle(const Geom& g, int formulation, double mu, cudaStream_t s,
              const i64* d_map = nullptr);
  const EntryView& view() const { return v_; }
  bool has_nullspace() const { return form_ != SBX_EXTERIOR_COMBINED; }
  // Column-major out (nr x nc) on the device; rows/cols device arrays of
  // scalar indices (local to the subset when a map is installed).
  void submatrix(const i64* d_rows, i64 nr, const i64* d_cols, i64 nc, double* d_out, i64 ld,
                 cudaStream_t s) const;
  void submatrix_host(const i64* rows, i64 nr, const i64* cols, i64 nc, double* out,
                      cudaStream_t s) const;

 private:
  EntryView v_{};
  int form_;
};

// evaluate_solution (nystrom.cpp:408-448) on the device: velocity (2 x T per
// density, densities stacked), optional pressure (T per density) and the
// near-boundary flag, host buffers.
void evaluate_solution_host(const Geom& g, int formulation, double mu, const double* tau, i64 ldt, i64 nrhs,
                            const double* targets, i64 n_targets, bool with_pressure, double* velocity,
                            double* pressure, unsigned char* near, cudaStream_t s);
void boundary_data_host(const Geom& g, i64 n_src, const double* src_xyf, double mu, double* out,
                        cudaStream_t s);

// Batched dense blocks D_b = A(rows_b, cols_b) written column-major at
// out + off_b (ld = nr_b).  Index lists are concatenated device arrays.
struct BlockJob {
  i64 row_off, col_off;  // into the concatenated index arrays
  int nr, nc;
  i64 out_off;
  int ld, pad;
  i64 dst_col_off = -1;  // >= 0: output column c goes to column dst_cols[dst_col_off + c]
};
void launch_block_jobs(const EntryView& v, const BlockJob* d_jobs, int n_jobs, i64 max_entries,
                       const i64* d_rows, const i64* d_cols, double* out, cudaStream_t s,
                       const i64* d_dst_cols = nullptr);

// Proxy-surface blocks of the HBS compression, written TRANSPOSED as the
// first rows of W^T (the ID engine factors W^T): for candidate scalar list
// cand (n = |cand|) and ns circle samples around (cx, cy) with radius rad,
//   kind 0 (row / outgoing, hbs.cpp:131-154): rows 4s..4s+3 = S(x_c, p_s)
//          (comp a, cols 0/1), D(x_c, p_s; radial)(a, 0/1); row 4ns = row_null
//   kind 1 (col / incoming, hbs.cpp:159-189): w_j-weighted D (+S) values and
//          radial gradients at p_s, row 4ns = col_null
//   kind 2 (proxy_interaction, proxy.cpp:136-162): as kind 0 with mu = 1
//          and the completion column from the node normal (mask applied by
//          the caller through `null_mask_comp`)
struct ProxyJob {
  i64 cand_off;     // into the candidate scalar array
  int n;            // candidates (columns of W^T)
  int ns;           // samples per circle
  double cx, cy, rad;
  i64 out_off;      // W^T base (column-major, leading dimension ld)
  int ld;
  int kind;
  int with_null;    // 1 = append the completion row
  int pad;
};
void launch_proxy_jobs(const EntryView& v, const ProxyJob* d_jobs, int n_jobs, int max_rows,
                       int max_n, const i64* d_cand, double* out, cudaStream_t s);

// Near-field rows of W^T: out(r, c) = A(cand_c, near_r) (row ID) or
// A(near_r, cand_c) (column ID) — i.e. W^T = [proxy^T ; rnear^T].
struct NearJob {
  i64 cand_off, near_off;
  int n, n_near;
  i64 out_off;  // first near row of W^T
  int ld;
  int transpose;  // 0: A(cand, near)^T (row ID), 1: A(near, cand) (col ID)
};
void launch_near_jobs(const EntryView& v, const NearJob* d_jobs, int n_jobs, i64 max_entries,
                      const i64* d_cand, const i64* d_near, double* out, cudaStream_t s);

// The same jobs through a caller-supplied entry oracle: blocks evaluated on
// the host, copied into place (host index arrays of the jobs).
void host_block_jobs(const HostEntries& h, const std::vector<BlockJob>& jobs, const std::vector<i64>& rows,
                     const std::vector<i64>& cols, double* out, cudaStream_t s);
void host_near_jobs(const HostEntries& h, const std::vector<NearJob>& jobs, const std::vector<i64>& cand,
                    const std::vector<i64>& near, double* out, cudaStream_t s);

}  // namespace sbx
