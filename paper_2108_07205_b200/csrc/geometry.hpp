// Wall discretization and refinement plans (reference geometry.hpp:58-146).
//
// Node generation and the refine/coarsen index bookkeeping are O(N) host
// work; the per-node arrays are kept structure-of-arrays
// and mirrored to the device once per discretization for the kernels.
#pragma once

#include <vector>

#include "common.hpp"
#include "sbx.h"

namespace sbx {

struct GaussTable {
  std::vector<double> x, w;
};
const GaussTable& gauss_table(int q);

struct CurveDef {
  sbx_curve p;
  void eval(double t, double& px, double& py, double& dx, double& dy, double& ddx,
            double& ddy) const;
  void channel_eval(double t, double& px, double& py, double& dx, double& dy, double& ddx,
                    double& ddy) const;
};

struct PanelDef {
  double a = 0, b = 0;
  int level = 0;
};

struct Component {
  CurveDef curve;
  std::vector<PanelDef> panels;
  int q = 16;
  i64 node_offset = 0, panel_offset = 0;
  bool is_hole = false;
};

struct PanelRow {
  i64 component = 0, local = 0;
  double a = 0, b = 0;
  int level = 0;
  i64 node_begin = 0;
  int q = 16;
};

// Device mirror of the node arrays (SoA, doubles).
struct GeomDev {
  DevBuf<double> buf;  // x | y | nx | ny | w | kappa | tx | ty
  DevBuf<int> comp;    // component of node
  i64 n = 0;
  const double* x() const { return buf.get(); }
  const double* y() const { return buf.get() + n; }
  const double* nx() const { return buf.get() + 2 * n; }
  const double* ny() const { return buf.get() + 3 * n; }
  const double* w() const { return buf.get() + 4 * n; }
  const double* kappa() const { return buf.get() + 5 * n; }
  const double* tx() const { return buf.get() + 6 * n; }
  const double* ty() const { return buf.get() + 7 * n; }
};

// Per-node tables of the log-corrected single layer (nystrom.cpp:40-63 and
// the self tables of logquad.cpp), device resident.  ints: loc | q | panel
// local index | component panel count | self-table offset; doubles: Gauss
// abscissa | jacobian | u_prev | u_next; lam: lambda_prev | lambda_next
// (n x qmax each).
struct SlTables {
  std::vector<char> mask;  // single-layer flag per component it was built for
  i64 n = 0;
  int qmax = 0;
  DevBuf<int> ints;
  DevBuf<double> dbl, lam, tab;
};

struct Geom {
  std::vector<Component> comps;
  std::vector<PanelRow> panels;
  std::vector<double> x, y, nx, ny, tx, ty, w, kappa, t;
  std::vector<i64> panel_of;
  i64 n_nodes() const { return i64(x.size()); }
  i64 component_of(i64 i) const { return panels[size_t(panel_of[size_t(i)])].component; }
  double panel_arclength(i64 p) const;
  GeomDev dev;
  void upload(cudaStream_t s);
  mutable std::shared_ptr<SlTables> sl;  // built on first single-layer use
};

struct Plan {
  std::vector<i64> panel_ids;
  int m = 1;
  std::vector<i64> kept_old, kept_new, cut_old, added_new;
  std::vector<std::vector<PanelDef>> old_panels;
  std::vector<int> old_q;
};

std::unique_ptr<Geom> geom_panelize(const sbx_curve& c, int n_panels, int q);
std::unique_ptr<Geom> geom_build(const std::vector<sbx_curve>& curves,
                                 const std::vector<std::vector<PanelDef>>& meshes,
                                 const std::vector<int>& qs, const std::vector<bool>& holes);
std::pair<std::unique_ptr<Geom>, std::unique_ptr<Plan>> geom_refine(const Geom& g,
                                                                    std::vector<i64> ids, int m);
std::unique_ptr<Geom> geom_coarsen(const Geom& g, const Plan& p);
std::pair<std::unique_ptr<Geom>, std::unique_ptr<Plan>> geom_add_holes(
    const Geom& wall, const std::vector<sbx_curve>& holes, const std::vector<int>& n_panels,
    const std::vector<int>& qs);
std::vector<i64> panels_near_point(const Geom& g, double px, double py, double radius);

}  // namespace sbx
