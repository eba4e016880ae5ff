// Multi-GPU partitioned path: one process (or host thread)
// per GPU, the HBS tree split by leaf subtrees, NCCL over NVLink for the only
// exchanges.
//
//   solve     rank p of G = 2^g owns the subtree rooted at the p-th BFS node
//             of depth g (hbs.cpp:379-383 halving makes it a contiguous range
//             of old-mesh rows): local up-sweep -> all-gather of the G
//             subtree-root hats (G x kmax x nrhs doubles) -> the top g levels
//             redundantly -> local down-sweep.
//   Woodbury  X = Atilde^{-1} L and the columns of R follow the same row
//             ownership, A_pp (and its rows of X and y) lives on rank 0, the
//             u x u product R X and the u x nrhs product R y are all-reduced,
//             W^{-1} is formed redundantly (els.cpp:80-179).
//
// Collective is the exchange interface: NCCL (libnccl loaded at run time,
// reusing an NCCL the process already has, e.g. torch's) or a loopback group
// of G ranks inside one process (one host thread per rank, exchanges by
// device copies) that tests the same protocol on a single GPU.
#pragma once

#include <memory>
#include <vector>

#include "els.hpp"
#include "hbs.hpp"

namespace sbx {

class Collective {
 public:
  virtual ~Collective() = default;
  virtual int world() const = 0;
  virtual int rank() const = 0;
  // In place: buf holds world() blocks of `count` doubles; this rank's block
  // (at rank() * count) is sent, the others are received.  Stream ordered.
  virtual void all_gather(double* buf, size_t count, cudaStream_t s) = 0;
  // In place sum over ranks (every rank gets the same bits).  Stream ordered.
  virtual void all_reduce_sum(double* buf, size_t count, cudaStream_t s) = 0;
};

// All-gather of one variable-length host vector per rank (sizes, then the
// payload padded to the longest), through the collective on stream s;
// integers travel exactly as doubles (< 2^53).
std::vector<std::vector<double>> gather_host(Collective& c, const std::vector<double>& mine, cudaStream_t s);

// 128-byte NCCL unique id (rank 0 creates it, the caller distributes it).
void nccl_unique_id(unsigned char out[128]);
std::unique_ptr<Collective> make_nccl_collective(const unsigned char id[128], int world, int rank);
// `world` members of one in-process group (member r must be driven by its own host thread).
std::vector<std::unique_ptr<Collective>> make_loopback_group(int world);

// x_local = A_oo^{-1} b restricted to this rank's rows [row0, row1) of the
// subtree partition (device column-major blocks).
void hbs_solve_sharded(HbsOp& op, Collective& c, const double* b_local, i64 ldb, i64 nrhs, double* x_local,
                       i64 ldx, cudaStream_t s);

// The Woodbury factors of the extended system on the subtree ownership.
struct ElsShard {
  HbsOp* a_oo = nullptr;
  Collective* comm = nullptr;
  std::shared_ptr<AppSolver> app;   // rank 0 (n_p > 0)
  int G = 1, p = 0;
  i64 row0 = 0, row1 = 0;           // owned old-mesh scalar rows
  i64 n_k = 0, n_c = 0, n_p = 0, k = 0;
  std::vector<i64> ext_of_local;    // ext row of each owned row (old-mesh order)
  DevBuf<i64> d_ext_of_local;
  DevBuf<double> X;                 // rows x k: owned rows of Atilde^{-1} L
  DevBuf<double> Rt;                // rows x k: owned columns of R, transposed
  DevBuf<double> Xp, Rpt;           // rank 0: n_p x k rows of X / columns of R (transposed)
  DevBuf<double> Winv;              // k x k
  DevBuf<double> Wmat;              // k x k (I + R X), for inspection
  i64 rows() const { return row1 - row0; }
  i64 local_p() const { return p == 0 ? n_p : 0; }
};

std::unique_ptr<ElsShard> els_shard_build(HbsOp& a_oo, Collective& c, const Geom& old_g, const Geom& new_g,
                                          const Plan& plan, const Update& upd, int formulation, double mu,
                                          cudaStream_t s);
// y = ELS^{-1} g on the shard layout: g_local / y_local are the owned rows
// (old-mesh order, rows() x nrhs), g_p / y_p the added rows on rank 0
// (local_p() x nrhs; ignored elsewhere).  Device column-major blocks.
void els_shard_solve(ElsShard& e, const double* g_local, i64 ldg, const double* g_p, i64 ldgp, i64 nrhs,
                     double* y_local, i64 ldy, double* y_p, i64 ldyp, cudaStream_t s);

}  // namespace sbx
