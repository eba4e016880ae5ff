// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference refined-wall Stokes solver
// (/root/reference/proj, "stokesbie") used as the parity checker for the
// B200 product path.  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load this code; the product
// library (paper_2108_07205_b200/) never links or calls it.
//
// The reference itself cannot be compiled here (it needs Eigen3, doctest,
// CLI11 — none present), so this is a restatement that
// follows the reference algorithm line by line (tree split, rank rules,
// sample doubling, rank equalisation, thresholds, seeded sketch) with its
// own small dense linear algebra in place of Eigen (ColPivHouseholderQR,
// PartialPivLU + Hager/Higham rcond, HouseholderQR, triangular solves).
// Parity is "not bitwise" (Eigen's vectorised summation order is not
// reproduced); it is pinned against the reference's own test assertions,
// which tests/test_oracle_*.py re-state.
#pragma once

#include <cmath>
#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

using Index = std::int64_t;
constexpr double kPi = 3.141592653589793238462643383279502884;

// ---------------------------------------------------------------- errors
// Mirrors proj/include/stokesbie/common.hpp:20-52.
struct GeometryError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct SingularMatrixError : std::runtime_error {
  SingularMatrixError(const std::string& msg, std::string w)
      : std::runtime_error(msg + " at " + w), where(std::move(w)) {}
  std::string where;
};
struct ProxyViolationError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
inline void require(bool c, const std::string& m) {
  if (!c) throw std::invalid_argument(m);
}

// ---------------------------------------------------------------- dense LA
// Column-major dense matrix (Eigen MatrixXd storage order).
struct Mat {
  Index r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(Index rows, Index cols) : r(rows), c(cols), a(size_t(rows * cols), 0.0) {}
  double& operator()(Index i, Index j) { return a[size_t(i + j * r)]; }
  double operator()(Index i, Index j) const { return a[size_t(i + j * r)]; }
  double* col(Index j) { return a.data() + j * r; }
  const double* col(Index j) const { return a.data() + j * r; }
  Index size() const { return r * c; }
  static Mat identity(Index n) {
    Mat m(n, n);
    for (Index i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
  Mat transpose() const;
  Mat rows_of(const std::vector<Index>& rows) const;
  Mat block(Index i0, Index j0, Index nr, Index nc) const;
  void set_block(Index i0, Index j0, const Mat& b);
  double norm() const;  // Frobenius
};

Mat matmul(const Mat& a, const Mat& b);                  // a*b
Mat matmul_tn(const Mat& a, const Mat& b);               // a^T*b
Mat hcat(const Mat& a, const Mat& b);
Mat vcat(const Mat& a, const Mat& b);
Mat sub(const Mat& a, const Mat& b);

// Eigen::ColPivHouseholderQR restated (Eigen/src/QR/ColPivHouseholderQR.h):
// pivot = first index of the largest updated column norm, LAPACK xGEQPF
// style norm downdating with direct recomputation when the downdate loses
// accuracy (threshold sqrt(eps)), Householder vectors as in
// makeHouseholderInPlace (beta = -sign(c0) * norm).
struct CPQR {
  Mat qr;                  // R in the upper triangle
  std::vector<Index> perm; // perm[i] = original column at position i
};
CPQR cpqr(const Mat& a);

// Eigen::HouseholderQR + householderQ() * Identity(rows, ncols).
Mat householder_q_thin(const Mat& a, Index ncols);

// Eigen::PartialPivLU restated: first-max pivot, rcond() = Hager/Higham
// 1-norm estimator (Eigen/src/Core/ConditionEstimator.h).
struct LU {
  Mat lu;
  std::vector<Index> piv;  // row permutation: row i of PA = row piv[i] of A
  double l1norm = 0.0;
  explicit LU(const Mat& a);
  Mat solve(const Mat& b) const;
  Mat solve_t(const Mat& b) const;  // (A^T)^{-1} b
  Mat inverse() const;
  double rcond() const;
  Index n() const { return lu.r; }
};

// Upper-triangular solve U x = B (U = top-left k x k of `u`).
Mat upper_solve(const Mat& u, Index k, const Mat& b);

// ---------------------------------------------------------------- quadrature
struct GaussRule {
  std::vector<double> nodes, weights;
};
const GaussRule& gauss_rule(int n);                     // gauss.cpp:24-59
void legendre_values(int n, double x, double* out);     // gauss.cpp:61-68
std::vector<double> log_rule_weights(int q, double u);  // logquad.cpp:84-98
const Mat& log_rule_self_table(int q);                  // logquad.cpp:100-112

// ---------------------------------------------------------------- geometry
struct V2 {
  double x = 0, y = 0;
};
inline V2 operator+(V2 a, V2 b) { return {a.x + b.x, a.y + b.y}; }
inline V2 operator-(V2 a, V2 b) { return {a.x - b.x, a.y - b.y}; }
inline V2 operator*(double s, V2 a) { return {s * a.x, s * a.y}; }
inline double dot(V2 a, V2 b) { return a.x * b.x + a.y * b.y; }
inline double norm(V2 a) { return std::sqrt(a.x * a.x + a.y * a.y); }

// Channel (4): the closed wavy channel of BASELINE configs[3] (sbx.h SBX_CHANNEL;
// the reference has no such kind).
enum class CurveKind { Circle = 0, Ellipse = 1, Star = 2, Fourier = 3, Channel = 4 };

struct CurveParams {  // geometry.hpp:14-26
  CurveKind kind = CurveKind::Circle;
  V2 center;
  double scale = 1.0;
  bool flip_normal = false;
  int n_prongs = 0;
  double amplitude = 0.0;
  double aspect = 1.0;
  std::vector<double> cos_coef, sin_coef;
};

struct Curve {  // geometry.cpp:11-110
  CurveParams p;
  explicit Curve(CurveParams params);
  void radial(double t, double& r, double& dr, double& ddr) const;
  void channel(double t, double& px, double& py, double& dx, double& dy, double& ddx, double& ddy) const;
  V2 position(double t) const;
  V2 derivative(double t) const;
  V2 second_derivative(double t) const;
  double speed(double t) const { return norm(derivative(t)); }
  V2 unit_tangent(double t) const;
  V2 normal(double t) const;
  double curvature(double t) const;
};

struct Panel {
  double a = 0, b = 0;
  int level = 0;
};
struct PanelMesh {
  std::vector<Panel> panels;
  int q = 16;
};
PanelMesh uniform_mesh(int n_panels, int q);

struct Discretization {  // geometry.hpp:60-101
  struct Component {
    Curve curve;
    PanelMesh mesh;
    Index node_offset = 0, panel_offset = 0;
    bool is_hole = false;
  };
  struct PanelRef {
    Index component = 0, local = 0;
    double a = 0, b = 0;
    int level = 0;
    Index node_begin = 0;
    int q = 16;
  };
  std::vector<Component> components;
  std::vector<PanelRef> panels;
  std::vector<V2> x, normal, tangent;
  std::vector<double> w, curvature, param;
  std::vector<Index> panel_of;
  Index n_nodes() const { return Index(x.size()); }
  Index n_unknowns() const { return 2 * n_nodes(); }
  Index n_panels() const { return Index(panels.size()); }
  Index component_of_node(Index i) const { return panels[size_t(panel_of[size_t(i)])].component; }
  double panel_arclength(Index p) const;
};

Discretization panelize(const Curve& c, int n_panels, int q);
Discretization build_discretization(const std::vector<CurveParams>& curves,
                                    const std::vector<PanelMesh>& meshes,
                                    const std::vector<bool>& holes);

struct RefinementPlan {  // geometry.hpp:105-116
  std::vector<Index> panel_ids;
  int m = 1;
  std::vector<Index> kept_old, kept_new, cut_old, added_new;
  std::vector<PanelMesh> old_meshes;
  Index n_k() const { return Index(kept_old.size()); }
  Index n_c() const { return Index(cut_old.size()); }
  Index n_p() const { return Index(added_new.size()); }
};

std::pair<Discretization, RefinementPlan> refine(const Discretization& d,
                                                 std::vector<Index> panel_ids, int m);
Discretization coarsen(const Discretization& d, const RefinementPlan& plan);
struct HoleSpec {
  CurveParams curve;
  int n_panels = 10, q = 16;
};
std::pair<Discretization, RefinementPlan> add_holes(const Discretization& d,
                                                    const std::vector<HoleSpec>& holes);
std::vector<Index> panels_near_point(const Discretization& d, V2 p, double radius);
bool point_inside(const Curve& c, V2 p, int samples = 512);

// ---------------------------------------------------------------- kernels
struct M2 {
  double a00 = 0, a01 = 0, a10 = 0, a11 = 0;
  double operator()(int i, int j) const {
    return i == 0 ? (j == 0 ? a00 : a01) : (j == 0 ? a10 : a11);
  }
};
M2 stokeslet(V2 x, V2 y, double mu);                         // kernels.cpp:13-23
M2 double_layer(V2 x, V2 y, V2 ny);                          // kernels.cpp:25-31
M2 stokeslet_gradient(V2 x, V2 y, double mu, V2 d);          // kernels.cpp:50-60
M2 double_layer_gradient(V2 x, V2 y, V2 ny, V2 d);           // kernels.cpp:62-72

enum class FormulationKind { InteriorDirichlet = 0, ExteriorCombined = 1, Mixed = 2 };
struct Formulation {
  FormulationKind kind = FormulationKind::InteriorDirichlet;
  double mu = 1.0;
};
struct ComponentRole {
  double jump = -0.5;
  bool single_layer = false, in_nullspace = false;
};
ComponentRole component_role(const Formulation& f, const Discretization& d, Index comp);

// ---------------------------------------------------------------- Nystrom
class Assembler {  // nystrom.cpp:16-217
 public:
  Assembler(std::shared_ptr<const Discretization> d, Formulation f);
  const Discretization& disc() const { return *d_; }
  std::shared_ptr<const Discretization> disc_ptr() const { return d_; }
  const Formulation& formulation() const { return f_; }
  void fill_block(Index i, Index j, double out[4]) const;
  Mat submatrix(const std::vector<Index>& rows, const std::vector<Index>& cols) const;
  Mat full_matrix() const;
  bool has_nullspace() const { return any_nullspace_; }
  bool has_single_layer() const { return any_single_layer_; }
  const ComponentRole& role(Index c) const { return roles_[size_t(c)]; }

 private:
  std::shared_ptr<const Discretization> d_;
  Formulation f_;
  std::vector<ComponentRole> roles_;
  bool any_single_layer_ = false, any_nullspace_ = false;
  std::vector<Index> comp_of_;
  std::vector<int> local_in_panel_;
  std::vector<double> gl_xi_, jac_;
  std::vector<std::vector<double>> lam_prev_, lam_next_;
  std::vector<double> u_prev_, u_next_;
};

enum class BlockName { kk, kc, ck, cc, kp, pk, pp };

class BlockSource {  // nystrom.cpp:271-358
 public:
  BlockSource(std::shared_ptr<const Assembler> o, std::shared_ptr<const Assembler> n,
              RefinementPlan plan);
  Mat eval(BlockName b, const std::vector<Index>& rows, const std::vector<Index>& cols) const;
  Mat eval_full(BlockName b) const;
  Index rows_of(BlockName b) const { return Index(row_map(b).size()); }
  Index cols_of(BlockName b) const { return Index(col_map(b).size()); }
  const RefinementPlan& plan() const { return plan_; }
  const Assembler& old_oracle() const { return *old_; }
  const Assembler& new_oracle() const { return *new_; }
  std::shared_ptr<const Assembler> old_ptr() const { return old_; }
  std::shared_ptr<const Assembler> new_ptr() const { return new_; }
  const std::vector<Index>& kept_old_s() const { return kept_old_s_; }
  const std::vector<Index>& kept_new_s() const { return kept_new_s_; }
  const std::vector<Index>& cut_s() const { return cut_s_; }
  const std::vector<Index>& added_s() const { return added_s_; }

 private:
  const Assembler& oracle_of(BlockName b) const;
  const std::vector<Index>& row_map(BlockName b) const;
  const std::vector<Index>& col_map(BlockName b) const;
  std::shared_ptr<const Assembler> old_, new_;
  RefinementPlan plan_;
  std::vector<Index> kept_old_s_, kept_new_s_, cut_s_, added_s_;
};

struct StokesletSource {
  V2 location, strength{1, 0};
};
std::vector<StokesletSource> ring_sources(int n, V2 center, double radius);
std::vector<double> boundary_data(const Discretization& d,
                                  const std::vector<StokesletSource>& s, double mu);
V2 field_velocity(const std::vector<StokesletSource>& s, double mu, V2 p);
void dump_matrix(const std::string& path, const Mat& m);  // nystrom.cpp:450-461
Mat load_matrix(const std::string& path);                  // nystrom.cpp:463-477
std::vector<V2> evaluate_velocity(const Discretization& d, const Formulation& f,
                                  const std::vector<double>& tau,
                                  const std::vector<V2>& targets);

// ---------------------------------------------------------------- ID
struct IdResult {  // idlib.hpp:15-27
  std::vector<Index> J;
  Mat P;
  Index k = 0;
  double eps = 0;
};
IdResult row_id(const Mat& w, double eps);                              // idlib.cpp:73-86
IdResult row_id_rank(const Mat& w, Index k);                            // idlib.cpp:88-99
IdResult randomized_row_id(const Mat& w, double eps, std::uint64_t seed,
                           int oversample = 10, int power_iters = 1);   // idlib.cpp:101-132
// The host Gaussian sketch of idlib.cpp:108-113 (mt19937_64 + libstdc++
// normal_distribution, filled column by column).
Mat gaussian_sketch(Index n, Index l, std::uint64_t seed);

// ---------------------------------------------------------------- proxy
enum class ProxySurface { Basis, Division };
struct ProxyCircle {
  V2 center;
  double r0 = 0;
};
struct ProxyGeometry {  // proxy.hpp:31-46
  std::vector<ProxyCircle> circles;
  double bas_factor = 1.5, div_factor = 3.0;
  int n_proxy = 64;
  struct Sample {
    V2 p, radial;
  };
  double radius(ProxySurface s, size_t c) const;
  std::vector<Sample> surface_samples(ProxySurface s, int n) const;
  bool inside_any(ProxySurface s, V2 p) const;
  double band_distance(V2 p) const;
};
ProxyGeometry make_proxy_geometry(const Discretization& d, const RefinementPlan& plan);
std::pair<std::vector<Index>, std::vector<Index>> split_far_near(const std::vector<V2>& pts,
                                                                 const ProxyGeometry& g);
struct PartitionTree {
  enum class Kind { DyadicByDistance, BinaryByIndex };
  Kind kind = Kind::DyadicByDistance;
  std::vector<std::vector<Index>> leaves;
  int depth = 0;
};
PartitionTree build_partition_tree(PartitionTree::Kind kind, const std::vector<V2>& pts,
                                   const ProxyGeometry& g, Index leaf_cap = 128);
IdResult compress_block_far(const std::vector<V2>& pts, const std::vector<V2>* nrm,
                            const ProxyGeometry& g, ProxySurface s,
                            const PartitionTree& tree, double eps);

// ---------------------------------------------------------------- HBS
struct HbsSource {  // hbs.hpp:19-31
  std::function<Mat(const std::vector<Index>&, const std::vector<Index>&)> entries;
  std::vector<V2> points, source_normal;
  std::vector<double> source_weight;
  std::vector<char> source_single_layer;
  std::vector<V2> row_null, col_null;
  double mu = 1.0;
  Index n_nodes() const { return Index(points.size()); }
};
HbsSource make_hbs_source(std::shared_ptr<const Assembler> a);
HbsSource make_hbs_source_subset(std::shared_ptr<const Assembler> a, std::vector<Index> nodes);

struct HbsOptions {
  double eps = 1e-10;
  Index leaf_nodes = 64;
  int n_proxy = 64;
  double bas_factor = 1.5, div_factor = 3.0;
};
struct HbsNode {  // hbs.hpp:48-62
  Index begin = 0, end = 0, parent = -1, left = -1, right = -1;
  int depth = 0;
  Index k = 0;
  std::vector<Index> row_skel, col_skel;
  Mat u, v, d, b_sib, dhat, e, f, g;
  bool is_leaf() const { return left < 0; }
};
struct HbsOperator {  // hbs.hpp:64-74
  Index n = 0, leaf_nodes = 64;
  double eps = 0;
  std::vector<HbsNode> nodes;
  Mat root_g;
  bool has_inverse = false;
  std::vector<std::string> notes;
  Index max_block_drawn = 0;
  Index total_skeleton() const;
};
HbsOperator hbs_compress(const HbsSource& src, const HbsOptions& o = {});
void hbs_invert(HbsOperator& op);
Mat hbs_apply(const HbsOperator& op, const Mat& v);
Mat hbs_apply_t(const HbsOperator& op, const Mat& v);
Mat hbs_solve(const HbsOperator& op, const Mat& b);
Mat hbs_solve_t(const HbsOperator& op, const Mat& b);
void hbs_save(const HbsOperator& op, const std::string& path);
HbsOperator hbs_load(const std::string& path);

// ---------------------------------------------------------------- low rank
struct BlockFactor {
  Mat L, R;
  Index k = 0;
};
struct LowRankUpdate {  // lowrank.hpp:28-47
  Mat L, R;
  Index k = 0;
  BlockFactor kc, kp, pk;
  Mat L1, R1;
  Index k1 = 0;
  std::vector<Index> skeleton;
  std::vector<std::string> notes;
  Index nk2 = 0, nc2 = 0, np2 = 0;
  Index n_ext() const { return nk2 + nc2 + np2; }
};
struct CompressOptions {
  PartitionTree::Kind tree_kind = PartitionTree::Kind::DyadicByDistance;
  Index leaf_cap = 128;
  bool reid_concat = false;
  std::uint64_t seed = 0;
  Index near_dense_limit = Index{1} << 22;
};
LowRankUpdate compress_update(const BlockSource& src, const ProxyGeometry& proxy, double eps,
                              const CompressOptions& o = {});

// ---------------------------------------------------------------- ELS
constexpr Index kDenseAddedLimit = 2048;  // els.hpp:40 (scalars)
struct ElsSolver {  // els.hpp:17-37
  std::shared_ptr<const HbsOperator> a_oo;
  Mat app_dense;
  std::unique_ptr<LU> app_lu;
  std::shared_ptr<const HbsOperator> app_h;
  LowRankUpdate update;
  Mat x, w;
  std::unique_ptr<LU> w_lu;
  RefinementPlan plan;
  std::shared_ptr<const Assembler> old_a, new_a;
  std::vector<Index> kept_old_s, kept_new_s, cut_s, added_s;
  Index n_k = 0, n_c = 0, n_p = 0;
  Index n_ext() const { return n_k + n_c + n_p; }
};
std::unique_ptr<ElsSolver> els_build(std::shared_ptr<const HbsOperator> a_oo,
                                     const BlockSource& blocks, const RefinementPlan& plan,
                                     LowRankUpdate update);
Mat els_solve_raw(const ElsSolver& s, const Mat& g_ext);
Mat els_solve_raw_t(const ElsSolver& s, const Mat& g_ext);
Mat els_solve(const ElsSolver& s, const Mat& g_n);  // multi-column els_solve
Mat els_apply_forward(const ElsSolver& s, const Mat& v);
std::vector<double> density_on_refined(const ElsSolver& s, const std::vector<double>& tau_n);

}  // namespace orc
