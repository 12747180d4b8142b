// TEST INFRASTRUCTURE ONLY -- NOT PART OF THE PRODUCT.
//
// CPU oracle: a plain C++/OpenMP restatement of the reference ComBo solver
// (/root/reference/proj/src/*.cpp) used by tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline leg as the parity checker. The reference itself
// cannot be built here (no Eigen3, no FFTW3, vendor/ missing), so
// every routine below restates the reference algorithm with the file:line it
// follows. Eigen's dense kernels are replaced by explicit loops in the same
// arithmetic order; FFTW is replaced by an own mixed-radix FFT with the same
// r2c/c2r conventions (FFT summation order is therefore "parity unpinned" at
// the bit level). Compiled with -ffp-contract=off so that the
// bit-exact paths (generators, coarsen, normals) match the GPU kernels built
// with --fmad=false.
#pragma once

#include <array>
#include <cmath>
#include <complex>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace oracle {

// ---------------------------------------------------------------- tensors
// tensor.hpp:18-25 -- row-major 3x3, 9-vector image (11,12,13,21,...).
struct Mat3 {
  double a[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  double& operator()(int i, int j) { return a[3 * i + j]; }
  double operator()(int i, int j) const { return a[3 * i + j]; }
  static Mat3 identity() {
    Mat3 m;
    m.a[0] = m.a[4] = m.a[8] = 1.0;
    return m;
  }
};
struct Vec3 {
  double v[3] = {0, 0, 0};
  double& operator[](int i) { return v[i]; }
  double operator[](int i) const { return v[i]; }
};
struct Mat6 {
  double a[36] = {0};
  double& operator()(int i, int j) { return a[6 * i + j]; }
  double operator()(int i, int j) const { return a[6 * i + j]; }
};
struct Mat9 {
  double a[81] = {0};
  double& operator()(int i, int j) { return a[9 * i + j]; }
  double operator()(int i, int j) const { return a[9 * i + j]; }
  static Mat9 identity() {
    Mat9 m;
    for (int i = 0; i < 9; ++i) m.a[10 * i] = 1.0;
    return m;
  }
};

constexpr double kSqrt2 = 1.4142135623730951;  // tensor.hpp:27

struct SingularMatrix : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InadmissibleMacroState : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ConfigInvalid : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NonDividingFactor : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct BadShapeSpec : std::runtime_error {
  using std::runtime_error::runtime_error;
};

Mat3 add(const Mat3& x, const Mat3& y);
Mat3 sub(const Mat3& x, const Mat3& y);
Mat3 scale(double s, const Mat3& x);
Mat3 matmul(const Mat3& x, const Mat3& y);
Mat3 transpose(const Mat3& x);
Vec3 matvec(const Mat3& x, const Vec3& v);
double norm(const Mat3& x);
double norm(const Vec3& v);
double dot(const Vec3& x, const Vec3& y);
double det3(const Mat3& t);   // Eigen 3x3 cofactor order
Mat3 inv3(const Mat3& t);     // tensor.cpp:49-63
Vec3 mat3_col(const Mat3& m, int c);
double norm9(const Mat9& a);
Mat6 full_to_mandel(const std::array<double, 81>& f);   // tensor.cpp:118-125
std::array<double, 81> mandel_to_full(const Mat6& c);   // tensor.cpp:101-116
Mat9 mandel_to_mat9(const Mat6& c);                     // tensor.cpp:127-136

/// Symmetric eigen-solver (cyclic Jacobi, sqrt-only arithmetic). Replaces
/// Eigen::SelfAdjointEigenSolver at tensor.cpp:70-91 and materials.cpp:117.
/// Eigenvalues ascending; eigenvectors are the columns of vec (row-major n*n).
void sym_eig(int n, const double* m, double* lam, double* vec);
/// 3x3 variant used by the normals (tensor.cpp:70-91). Arithmetic is kept in
/// a fixed order so the GPU normals kernel can reproduce it bit for bit.
void sym_eig3_jacobi(const double m[9], double lam[3], double vec[9]);

// -------------------------------------------------------------- materials
// materials.hpp:14-21, 67-107
enum LawKind { kNeoHookean = 0, kLinear = 1 };
struct Law {
  int kind = kNeoHookean;
  double lambda = 0.0, mu = 0.0;
  Mat6 c6;   // Mandel stiffness (linear law)
  Mat9 a9;   // mandel_to_mat9(c6) (linear law)
  static Law neo_hookean(double lambda, double mu);
  static Law neo_hookean_enu(double e, double nu);  // materials.cpp:11-20
  static Law linear(const Mat6& c6);
  static Mat6 iso_mandel(double lambda, double mu);  // materials.cpp:22-30
};
bool law_eval(const Law& law, const Mat3& f, Mat3& p);
bool law_eval_tangent(const Law& law, const Mat3& f, Mat3& p, Mat9& a);
void law_spectrum_bounds(const Law& law, const Mat3& f, double& lo,
                         double& hi);

// --------------------------------------------------------------- laminate
// laminate.hpp:13-19, 69-141
struct ComboMeta {
  Vec3 normal;
  double c_plus = 0.5, c_minus = 0.5;
  static ComboMeta make(const Vec3& n, double c_plus);  // laminate.cpp:28-34
};
struct AdmissibleBounds {
  Vec3 m_beta;
  double beta_plus = 0.0, beta_minus = 0.0;
  bool admissible(const Vec3& a) const {
    const double b = dot(a, m_beta);
    return beta_plus < b && b < beta_minus;
  }
};
AdmissibleBounds admissibility_bounds(const Mat3& f_box, const ComboMeta& m);
Vec3 back_project(const Vec3& a1, const Vec3& a0, const AdmissibleBounds& b);
Mat9 effective_tangent(const Mat9& ap, const Mat9& am, const ComboMeta& m);

struct LaminateOptions {
  double tol_abs = 0.0;
  double tol_rel = 1e-10;
  double stress_floor = 0.0;
  int max_iter = 50;
  bool back_projection = true;
  double c_min = 0.0;
};
struct JumpVectorState {
  Vec3 a;
  bool converged = false;
  int iterations = 0;
  double residual = 0.0, residual_rel = 0.0;
  int back_projections = 0;
  int first_inadmissible_iter = -1;
};
struct LaminateResult {
  Mat3 f_plus = Mat3::identity(), f_minus = Mat3::identity();
  Mat3 p_plus, p_minus, p_box, s_box;
  Mat9 a_box;
  Vec3 traction;
  bool tangent_valid = false;
};
struct LaminateSolution {
  LaminateResult result;
  JumpVectorState state;
};
LaminateSolution finite_strain_solve(const Mat3& f_box, const Law& plus,
                                     const Law& minus, const ComboMeta& meta,
                                     const Vec3& a0, const LaminateOptions& opt,
                                     bool want_tangent);

// ------------------------------------------------------------ grid/fields
struct SimGrid {  // field.hpp:16-28
  std::array<std::int64_t, 3> dims{1, 1, 1};
  std::array<double, 3> lengths{1.0, 1.0, 1.0};
  std::int64_t cells() const { return dims[0] * dims[1] * dims[2]; }
  double spacing(int a) const { return lengths[a] / double(dims[a]); }
  std::size_t index(std::int64_t i, std::int64_t j, std::int64_t k) const {
    return std::size_t((i * dims[1] + j) * dims[2] + k);
  }
};
struct Field9 {  // field.hpp:32-70, component major, c = 3i+J
  SimGrid grid;
  std::vector<double> data;
  Field9() = default;
  explicit Field9(const SimGrid& g) : grid(g), data(std::size_t(9 * g.cells()), 0.0) {}
  std::int64_t cells() const { return grid.cells(); }
  double* comp(int c) { return data.data() + std::ptrdiff_t(c) * cells(); }
  const double* comp(int c) const { return data.data() + std::ptrdiff_t(c) * cells(); }
  Mat3 cell(std::size_t idx) const;
  void set_cell(std::size_t idx, const Mat3& m);
  void fill(const Mat3& m);
  Mat3 mean() const;                  // field.cpp:18-26
  void pin_mean(const Mat3& target);  // field.cpp:28-38
};
double deterministic_sum(const double* x, std::size_t n);   // parallel.hpp:40-66
double deterministic_dot(const double* x, const double* y, std::size_t n);
double deterministic_sumsq(const double* x, std::size_t n);

// ------------------------------------------------------------------- FFT
/// Batched 3D r2c / c2r with FFTW conventions (fft.hpp:17-52, fft.cpp:23-60):
/// complex layout [c][i][j][k3], k3 < n3/2+1; inverse scales by 1/n.
class Fft3 {
 public:
  Fft3(const std::array<std::int64_t, 3>& dims, int ncomp);
  std::int64_t n_real() const { return n_; }
  std::int64_t n_complex() const { return nc_; }
  double* real(int c) { return real_.data() + std::ptrdiff_t(c) * n_; }
  std::complex<double>* cplx(int c) { return cplx_.data() + std::ptrdiff_t(c) * nc_; }
  void forward();
  void inverse();

 private:
  std::array<std::int64_t, 3> dims_;
  int ncomp_;
  std::int64_t n_, nc_;
  std::vector<double> real_;
  std::vector<std::complex<double>> cplx_;
};

// ----------------------------------------------------------------- green
enum GreenKind { kContinuous = 0, kRotated = 1, kStaggered = 2 };
class GreenOperator {  // green.hpp:30-59, green.cpp:16-151
 public:
  GreenOperator(int kind, const SimGrid& grid);
  void apply_fourier(Fft3& fft) const;
  void project(const Field9& in, Field9& out, Fft3& fft) const;
  const std::vector<std::complex<double>>& forward_symbols(int a) const { return fwd_[a]; }

 private:
  int kind_;
  SimGrid grid_;
  std::array<std::vector<std::complex<double>>, 3> fwd_, avg_;
  std::array<std::vector<double>, 3> xi_;
};

// ----------------------------------------------------- image / preprocess
struct PhaseImage {  // image.hpp:17-44
  std::array<std::int64_t, 3> dims{0, 0, 0};
  std::array<double, 3> lengths{1.0, 1.0, 1.0};
  std::vector<std::uint8_t> data;
  std::int64_t size() const { return dims[0] * dims[1] * dims[2]; }
  std::size_t index(std::int64_t i, std::int64_t j, std::int64_t k) const {
    return std::size_t((i * dims[1] + j) * dims[2] + k);
  }
  std::uint8_t at(std::int64_t i, std::int64_t j, std::int64_t k) const { return data[index(i, j, k)]; }
  double spacing(int a) const { return lengths[a] / double(dims[a]); }
  Vec3 voxel_center(std::int64_t i, std::int64_t j, std::int64_t k) const {
    Vec3 x;
    x[0] = (double(i) + 0.5) * spacing(0);
    x[1] = (double(j) + 0.5) * spacing(1);
    x[2] = (double(k) + 0.5) * spacing(2);
    return x;
  }
  std::int64_t inclusion_count() const;
};

struct Splitmix64 {  // image.cpp:18-32
  std::uint64_t state;
  explicit Splitmix64(std::uint64_t s) : state(s) {}
  std::uint64_t next() {
    state += 0x9e3779b97f4a7c15ULL;
    std::uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  double unit() { return double(next() >> 11) * 0x1.0p-53; }
  double symmetric() { return 2.0 * unit() - 1.0; }
};

PhaseImage generate_from_predicate(const std::array<std::int64_t, 3>& dims,
                                   const std::array<double, 3>& lengths,
                                   const std::function<bool(const Vec3&)>& inside);
PhaseImage generate_sphere(const std::array<std::int64_t, 3>& dims,
                           const std::array<double, 3>& lengths, double r);
PhaseImage generate_octahedron(const std::array<std::int64_t, 3>& dims,
                               const std::array<double, 3>& lengths, double r);
PhaseImage generate_fiber(const std::array<std::int64_t, 3>& dims,
                          const std::array<double, 3>& lengths, int axis,
                          double radius, double length);
PhaseImage generate_cross_ply(const std::array<std::int64_t, 3>& dims,
                              const std::array<double, 3>& lengths,
                              double radius, double pitch, int layers);
PhaseImage generate_fiber_pack(const std::array<std::int64_t, 3>& dims,
                               const std::array<double, 3>& lengths,
                               std::uint64_t seed, int count, double radius,
                               double length, double spread);
PhaseImage generate_slab(const std::array<std::int64_t, 3>& dims,
                         const std::array<double, 3>& lengths, int axis,
                         double fraction);
PhaseImage mirrored(const PhaseImage& img, int axis);
/// seeded config microstructures (shape 10 rsa spheres, 11 rsa z-fibres,
/// 12 Boolean ellipsoids); see preprocess.cpp
PhaseImage generate_config(int shape, const std::array<std::int64_t, 3>& dims,
                           const std::array<double, 3>& lengths, const double* params);

enum BoxelKind : std::uint8_t { kPureMatrix = 0, kPureInclusion = 1, kComposite = 2 };
enum NormalFlag : std::uint8_t {
  kNormalNone = 0, kNormalBarycenterOk = 1, kNormalSecondMomentOk = 2,
  kNormalDegenerate = 3, kNormalTooFew = 4,
};
struct ComboGrid {  // combo_grid.hpp:29-59
  std::array<std::int64_t, 3> dims{0, 0, 0};
  std::array<std::int64_t, 3> factors{1, 1, 1};
  std::array<double, 3> lengths{1.0, 1.0, 1.0};
  std::vector<std::uint8_t> kind;
  std::vector<double> c_plus;
  std::vector<std::int64_t> count_plus;
  std::vector<Vec3> normal;
  std::vector<std::uint8_t> normal_flag;
  std::int64_t boxel_count() const { return dims[0] * dims[1] * dims[2]; }
  std::int64_t fine_per_boxel() const { return factors[0] * factors[1] * factors[2]; }
  std::size_t index(std::int64_t a, std::int64_t b, std::int64_t c) const {
    return std::size_t((a * dims[1] + b) * dims[2] + c);
  }
  double boxel_length(int a) const { return lengths[a] / double(dims[a]); }
  std::int64_t composite_count() const;
  std::int64_t global_count_plus() const;
  double global_c_plus() const;
};
ComboGrid coarsen(const PhaseImage& img, const std::array<std::int64_t, 3>& factors);

enum NormalMethod { kBarycenter = 0, kSecondMoment = 1 };
enum Centering { kWeightedCentroid = 0, kBoxelCenter = 1 };
struct NormalStats {
  std::int64_t composite = 0, degenerate_fallbacks = 0, too_few_fallbacks = 0;
};
std::vector<double> laplace_weights(const PhaseImage& img);  // normals.cpp:25-52
NormalStats compute_normals(const PhaseImage& img, ComboGrid& grid, int method,
                            int centering, int min_interface_voxels);

// --------------------------------------------------------- cell binding
class CellMaterials {  // cell_material.hpp:19-74, cell_material.cpp:12-84
 public:
  CellMaterials(const ComboGrid& grid, const Law& matrix, const Law& inclusion,
                bool combo, LaminateOptions lam = {});
  const SimGrid& grid() const { return grid_; }
  std::int64_t cells() const { return grid_.cells(); }
  const Law& matrix() const { return matrix_; }
  const Law& inclusion() const { return inclusion_; }
  std::uint8_t cell_phase(std::size_t c) const { return phase_[c]; }
  std::int32_t combo_id(std::size_t c) const { return combo_id_[c]; }
  const ComboMeta& meta(std::int32_t id) const { return metas_[std::size_t(id)]; }
  std::int64_t composite_cells() const { return std::int64_t(metas_.size()); }
  std::vector<Vec3>& warm_all() { return warm_a_; }
  const LaminateOptions& laminate_options() const { return lam_; }
  double represented_c_plus() const;
  void spectrum_bounds(const Mat3& fbar, double& lo, double& hi) const;

 private:
  SimGrid grid_;
  Law matrix_, inclusion_;
  std::vector<std::uint8_t> phase_;
  std::vector<std::int32_t> combo_id_;
  std::vector<ComboMeta> metas_;
  std::vector<Vec3> warm_a_;
  std::vector<double> c_plus_;
  LaminateOptions lam_;
  bool combo_ = true;
};

struct SweepStats {  // cell_material.hpp:76-84
  std::int64_t inadmissible_cells = 0, laminate_failures = 0, back_projections = 0;
  int laminate_iter_max = 0;
};
SweepStats stress_sweep(CellMaterials& cm, const Field9& f, Field9& p,
                        std::vector<double>* tangents45, bool lean = false);
void tangent_matvec_lean(const CellMaterials& cm, const std::vector<double>& t45c, const Field9& f,
                         const Field9& x, Field9& y);
void tangent_matvec(const std::vector<double>& t45, const Field9& x, Field9& y);
void pack45(const Mat9& a, double* dst);
Mat9 unpack45(const double* src);

struct DfmgState {  // dfmg.hpp:13-19
  std::vector<Vec3> warm_a;
  void resize(std::int64_t cells) { warm_a.assign(std::size_t(8 * cells), Vec3()); }
};
SweepStats dfmg_stress(CellMaterials& cm, DfmgState& st, const Field9& f, Field9& p);
SweepStats dfmg_tangent_pass(CellMaterials& cm, DfmgState& st, const Field9& f,
                             std::vector<double>& t45);
void dfmg_tangent_matvec(const std::vector<double>& t45, const Field9& x, Field9& y);

// ---------------------------------------------------------------- solver
enum Scheme { kBasic = 0, kNewtonCg = 1 };
enum MaterialEval { kPerCell = 0, kDfmg = 1 };
struct SolverConfig {  // solver.hpp:18-32
  int scheme = kNewtonCg;
  int green = kRotated;
  int eval = kPerCell;
  double tol_equilibrium = 1e-8;
  int max_outer = 200;
  double cg_tol = 1e-2;
  int cg_max = 2000;
  int load_steps = 1;
  int max_bisections = 5;
  int threads = 0;
  bool verbose = false;
  /// Test/bench hook (not in the reference): stop after this many LS
  /// iterations (Green-operator applications); 0 = unlimited. Used only for
  /// the bounded CPU-baseline sample.
  std::int64_t max_ls_iterations = 0;
};
struct StepReport {  // solver.hpp:34-46
  double t_start = 0.0, t_end = 0.0;
  Mat3 fbar;
  bool converged = false;
  int outer_iters = 0;
  std::vector<double> residuals;
  std::vector<int> cg_iters;
  int cg_breakdowns = 0;
  int line_search_cuts = 0;
  SweepStats sweep;
  double seconds = 0.0;
  std::vector<Mat3> pbar_history;  // added: P-bar per residual evaluation
  std::int64_t ls_basic = 0, ls_residual = 0, ls_cg = 0, ls_trial = 0;
};
struct ConvergenceReport {
  std::vector<StepReport> steps;
  bool success = false;
  std::string error;
  int bisections = 0;
  double alpha = 0.0;
  double seconds_total = 0.0;
  std::int64_t ls_total = 0;  // Green-operator applications (LS iterations)
  std::vector<double> ls_clock;  // seconds since solve() began, at the end of each LS iteration
};
struct SolveResult {
  Field9 f, p;
  Mat3 pbar;
  ConvergenceReport report;
};
SolveResult solve(CellMaterials& cm, const Mat3& fbar, const SolverConfig& cfg);

}  // namespace oracle
