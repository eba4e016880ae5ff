// Device HBS compression and telescoping inversion (north-star
// subsystem 4, reference hbs.cpp:349-487), timed separately from the
// per-step path.
#pragma once

#include "entries.hpp"
#include "geometry.hpp"
#include "hbs.hpp"
#include "sbx.h"

namespace sbx {

struct HbsBuildOptions {
  double eps = 1e-10;
  i64 leaf_nodes = 64;
  double bas_factor = 1.5;
  double div_factor = 3.0;
  // caller-supplied entry oracle (HbsSource::entries plugin); null: the
  // formulation's kernel entries on the device
  const HostEntries* entries = nullptr;
  // subtree-sharded build (multi-GPU): this rank's subtree and the top
  // levels only, skeletons exchanged level by level through `comm`
  class Collective* comm = nullptr;
  static HbsBuildOptions from(const sbx_hbs_options& o) {
    HbsBuildOptions b;
    b.eps = o.eps;
    b.leaf_nodes = o.leaf_nodes;
    b.bas_factor = o.bas_factor;
    b.div_factor = o.div_factor;
    return b;
  }
};

// Compress the operator of (g, formulation, mu) restricted to `nodes`
// (global node ids, make_hbs_source_subset) or the whole discretization.
std::unique_ptr<HbsOp> hbs_compress_device(const Geom& g, int formulation, double mu,
                                           const i64* nodes, i64 n_nodes,
                                           const HbsBuildOptions& o, cudaStream_t s);

void hbs_invert_device(HbsOp& op, cudaStream_t s);

// Compression and inverse in one pass: the telescoping inverse of depth d
// runs on a second stream while depth d - 1 is compressed (same kernels and
// results as hbs_compress_device + hbs_invert_device).
std::unique_ptr<HbsOp> hbs_compress_invert_device(const Geom& g, int formulation, double mu, const i64* nodes,
                                                  i64 n_nodes, const HbsBuildOptions& o, cudaStream_t s);

}  // namespace sbx
