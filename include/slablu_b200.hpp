// slablu_b200.hpp — C++ mirror of the reference solver API on top of the C ABI
// (include/slablu_gpu.h, libslablu_gpu.so).  Header-only.
//
// Names, argument meaning and error behaviour follow the reference library
// (/root/reference/proj/include/slablu/):
//   Error, ConfigError, SingularMatrixError        common.hpp:32-60
//   ProblemSpec, assemble_fd5, SparseSystem        problem.hpp:40-132
//   kappa_from_ppw, canned problems                problem.hpp:153-157, 210-261
//   SolverConfig, CompressionChoice, choose_b      driver.hpp:37-66
//   GridStrip, SlabPartition, partition            partition.hpp:27-91
//   Factorization, factorize, solve                driver.hpp:72-179
//   ErrorReport, error_report, sample_field        problem.hpp:160-206
//   SolveReport, csv_row, json_row, run_problem,
//   benchmark                                      driver.hpp:182-322
//   Shard (multi-GPU split, engine extension)      include/slablu_gpu.h slablu_gpu_shard_*
//
// Matrices are column major std::vector<double> (the reference uses
// Eigen::MatrixXd, also column major; INTEGRATION.md shows the Eigen shim).
#ifndef SLABLU_B200_HPP
#define SLABLU_B200_HPP

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <functional>
#include <ostream>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "slablu_gpu.h"

namespace slablu_b200 {

// ---- errors (common.hpp:32-60) --------------------------------------------
class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};
class ConfigError : public Error {
 public:
  explicit ConfigError(const std::string& what) : Error(what) {}
};
class SingularMatrixError : public Error {
 public:
  SingularMatrixError(const std::string& what, std::ptrdiff_t index)
      : Error(what + " (index " + std::to_string(index) + ")"), index(index) {}
  std::ptrdiff_t index;
};

class CompressionError : public Error {
 public:
  CompressionError(const std::string& what, double residual_estimate)
      : Error(what), residual_estimate(residual_estimate) {}
  double residual_estimate;
};

namespace detail {
inline void check(const slablu_gpu_status& s) {
  if (s.code == SLABLU_OK) return;
  const std::string msg(s.msg);
  if (s.code == SLABLU_ERR_CONFIG) throw ConfigError(msg);
  if (s.code == SLABLU_ERR_COMPRESSION) throw CompressionError(msg, s.residual);
  if (s.code == SLABLU_ERR_SINGULAR) throw SingularMatrixError(msg, static_cast<std::ptrdiff_t>(s.index));
  throw Error(msg);
}
}  // namespace detail

// ---- problems (problem.hpp) --------------------------------------------------
using ScalarField = std::function<double(double, double)>;

struct ProblemSpec {
  int64_t n1 = 0;
  int64_t n2 = 0;
  double h = 0.0;
  double kappa = 0.0;
  ScalarField coefficient_field = [](double, double) { return 1.0; };
  ScalarField dirichlet_data = [](double, double) { return 0.0; };
  ScalarField body_load = [](double, double) { return 0.0; };
};

struct SparseSystem {
  std::vector<int32_t> row_ptr, col_idx;  // Eigen RowMajor compressed form
  std::vector<double> values;
  std::vector<double> rhs;
  int64_t n1 = 0, n2 = 0;
  double h = 0.0;
  int64_t dim() const { return n1 * n2; }
  int64_t node_index(int64_t i, int64_t j) const { return i * n2 + j; }
};

inline SparseSystem assemble_fd5(const ProblemSpec& spec) {
  SparseSystem s;
  s.n1 = spec.n1;
  s.n2 = spec.n2;
  s.h = spec.h;
  const int64_t n = spec.n1 * spec.n2;
  if (n <= 0 || spec.n2 < 2 || spec.n1 < spec.n2) throw ConfigError("assemble_fd5: grid must satisfy n1 >= n2 >= 2");
  s.row_ptr.assign(n + 1, 0);
  s.col_idx.assign(5 * n, 0);
  s.values.assign(5 * n, 0.0);
  s.rhs.assign(n, 0.0);
  struct Fields {
    const ProblemSpec* p;
  } f{&spec};
  auto coef = [](double x, double y, void* u) { return static_cast<Fields*>(u)->p->coefficient_field(x, y); };
  auto dir = [](double x, double y, void* u) { return static_cast<Fields*>(u)->p->dirichlet_data(x, y); };
  auto load = [](double x, double y, void* u) { return static_cast<Fields*>(u)->p->body_load(x, y); };
  int64_t nnz = 0;
  detail::check(slablu_gpu_assemble_fd5(spec.n1, spec.n2, spec.h, spec.kappa, coef, dir, load, &f, s.row_ptr.data(),
                                        s.col_idx.data(), s.values.data(), s.rhs.data(), &nnz));
  s.col_idx.resize(nnz);
  s.values.resize(nnz);
  return s;
}

inline double kappa_from_ppw(double ppw, int64_t n2) {
  if (!(ppw > 0.0)) throw ConfigError("kappa_from_ppw: ppw must be positive");
  if (n2 < 2) throw ConfigError("kappa_from_ppw: n2 must be at least 2");
  return slablu_gpu_kappa_from_ppw(ppw, n2);
}
inline double bessel_j0(double t) { return slablu_gpu_bessel_j0(t); }

inline ProblemSpec poisson_log_problem(int64_t n1, int64_t n2) {
  ProblemSpec s;
  s.n1 = n1;
  s.n2 = n2;
  s.h = 1.0 / double(n2 + 1);
  s.dirichlet_data = [](double x, double y) { return std::log(std::hypot(x + 0.1, y - 0.5)); };
  return s;
}
inline ProblemSpec helmholtz_problem(int64_t n1, int64_t n2, double kappa) {
  ProblemSpec s;
  s.n1 = n1;
  s.n2 = n2;
  s.h = 1.0 / double(n2 + 1);
  s.kappa = kappa;
  s.dirichlet_data = [kappa](double x, double y) { return bessel_j0(kappa * std::hypot(x + 0.1, y - 0.5)); };
  return s;
}
inline ProblemSpec helmholtz_bump_problem(int64_t n1, int64_t n2, double kappa) {
  ProblemSpec s = helmholtz_problem(n1, n2, kappa);
  s.coefficient_field = [n1, n2](double x, double y) {
    const double h = 1.0 / double(n2 + 1);
    const double cx = 0.5 * double(n1 + 1) * h, cy = 0.5;
    const double d2 = (x - cx) * (x - cx) + (y - cy) * (y - cy);
    return 1.0 - 0.9 * std::exp(-64.0 * d2);
  };
  return s;
}

// ---- configuration and geometry (driver.hpp:37-66, partition.hpp) ------------
enum class CompressionChoice { automatic = 0, dense = 1, hbs = 2 };

struct SolverConfig {
  int64_t b = 0;
  double c = 0.6;
  CompressionChoice compression = CompressionChoice::automatic;
  double hbs_tol = 1e-11;
  double hbs_trunc_rel = 1e-13;
  int64_t hbs_leaf_size = 64;
  uint64_t seed = 0;
  int threads = 1;
  // engine extensions
  int device = 0;
  bool keep_T = false;
  int refine = 1;
  slablu_gpu_config c_config() const {
    slablu_gpu_config g{};
    g.b = b;
    g.c = c;
    g.compression = static_cast<int>(compression);
    g.seed = seed;
    g.threads = threads;
    g.device = device;
    g.keep_T = keep_T ? 1 : 0;
    g.refine = refine;
    g.hbs_tol = hbs_tol;
    g.hbs_trunc_rel = hbs_trunc_rel;
    g.hbs_leaf_size = hbs_leaf_size;
    return g;
  }
};

inline int64_t choose_b(int64_t n1, int64_t n2, const SolverConfig& config) {
  int64_t out = 0;
  detail::check(slablu_gpu_choose_b(n1, n2, config.b, config.c, &out));
  return out;
}

struct GridStrip {
  int64_t first_col = 0;
  int64_t width = 0;
};
struct SlabPartition {
  int64_t n1 = 0, n2 = 0, b = 0;
  std::vector<GridStrip> interfaces, interiors;
  int64_t interface_count() const { return static_cast<int64_t>(interfaces.size()); }
  int64_t interior_count() const { return static_cast<int64_t>(interiors.size()); }
  int64_t dim() const { return n1 * n2; }
  int64_t interface_offset(int64_t j) const { return interfaces[j].first_col * n2; }
  int64_t interior_offset(int64_t i) const { return interiors[i].first_col * n2; }
  int64_t interior_size(int64_t i) const { return interiors[i].width * n2; }
  int64_t left_interior(int64_t j) const { return j; }
  int64_t right_interior(int64_t j) const { return j + 1 < interior_count() ? j + 1 : -1; }
};

inline SlabPartition partition(int64_t n1, int64_t n2, int64_t b) {
  const int64_t cap = n1 + 2 > 4 ? n1 + 2 : 4;
  std::vector<int64_t> ints(2 * cap), ifcs(2 * cap);
  int64_t ni = 0, nf = 0;
  detail::check(slablu_gpu_partition(n1, n2, b, &ni, ints.data(), &nf, ifcs.data(), cap));
  SlabPartition p;
  p.n1 = n1;
  p.n2 = n2;
  p.b = b;
  for (int64_t k = 0; k < ni; k++) p.interiors.push_back({ints[2 * k], ints[2 * k + 1]});
  for (int64_t k = 0; k < nf; k++) p.interfaces.push_back({ifcs[2 * k], ifcs[2 * k + 1]});
  return p;
}

// ---- randomized HBS compression of a dense operator (hbs_compress.hpp:21-311) ---
struct CompressOptions {
  double tol = 1e-10;
  double trunc_rel = 1e-12;
  uint64_t seed = 0;
};
struct CompressStats {
  int64_t products_normal = 0, products_adjoint = 0;
  int rounds = 0;
  int64_t final_rank = 0;
  double residual_estimate = 0.0;
};
namespace detail {
inline std::vector<double> hbs_run(const std::vector<double>& m, int64_t n, int64_t leaf, int64_t r_start,
                                   int64_t r_max, int adaptive, const CompressOptions& o, CompressStats* st) {
  if ((int64_t)m.size() != n * n) throw Error("hbs_compress: dimension mismatch");
  std::vector<double> out((size_t)(n * n));
  slablu_gpu_hbs_stats s{};
  check(slablu_gpu_hbs_compress(n, m.data(), leaf, r_start, r_max, adaptive, o.tol, o.trunc_rel, o.seed, 0,
                                out.data(), &s));
  if (st) *st = CompressStats{s.products_normal, s.products_adjoint, s.rounds, s.final_rank, s.residual_estimate};
  return out;
}
}  // namespace detail
// hbs_compress with the dense sampler (test_hbs.cpp:64-68) on a column-major n x n operator;
// returns the dense materialization of the compressed operator (HbsMatrix::to_dense).
inline std::vector<double> hbs_compress(const std::vector<double>& m, int64_t n, int64_t leaf_size,
                                        int64_t rank_bound, const CompressOptions& o = {},
                                        CompressStats* stats = nullptr) {
  return detail::hbs_run(m, n, leaf_size, 0, rank_bound, 0, o, stats);
}
inline std::vector<double> hbs_compress_adaptive(const std::vector<double>& m, int64_t n, int64_t leaf_size,
                                                 int64_t r_start, int64_t r_max, const CompressOptions& o = {},
                                                 CompressStats* stats = nullptr) {
  return detail::hbs_run(m, n, leaf_size, r_start, r_max, 1, o, stats);
}

// ---- factorize / solve (driver.hpp:72-179) -----------------------------------
class Factorization {
 public:
  int64_t n1 = 0, n2 = 0, b = 0;
  SolverConfig config{};
  double t_stage1 = 0.0, t_stage2 = 0.0;  // seconds (device time)
  std::size_t storage_stage1 = 0, storage_stage2 = 0;
  int64_t hbs_max_rank = 0;

  bool single_slab() const { return stats_.single_slab != 0; }
  std::size_t storage_scalars() const { return storage_stage1 + storage_stage2; }
  const slablu_gpu_stats_t& stats() const { return stats_; }
  const slablu_gpu_fact* handle() const { return h_.get(); }

 private:
  struct Deleter {
    void operator()(slablu_gpu_fact* f) const { slablu_gpu_destroy(f); }
  };
  std::shared_ptr<slablu_gpu_fact> h_;
  slablu_gpu_stats_t stats_{};
  friend Factorization factorize(const SparseSystem&, SolverConfig);
};

inline Factorization factorize(const SparseSystem& system, SolverConfig config) {
  if (system.dim() == 0) throw ConfigError("factorize: empty system");
  const slablu_gpu_config c = config.c_config();
  slablu_gpu_fact* raw = nullptr;
  detail::check(slablu_gpu_factorize(system.n1, system.n2, system.row_ptr.data(), system.col_idx.data(),
                                     system.values.data(), &c, &raw));
  Factorization f;
  f.h_ = std::shared_ptr<slablu_gpu_fact>(raw, Factorization::Deleter{});
  detail::check(slablu_gpu_stats(raw, &f.stats_));
  f.n1 = system.n1;
  f.n2 = system.n2;
  f.b = f.stats_.b;
  config.b = f.b;
  config.compression = f.stats_.compression == 2 ? CompressionChoice::hbs : CompressionChoice::dense;
  f.config = config;
  f.hbs_max_rank = f.stats_.hbs_max_rank;
  f.t_stage1 = f.stats_.t_stage1;
  f.t_stage2 = f.stats_.t_stage2;
  f.storage_stage1 = static_cast<std::size_t>(f.stats_.storage_stage1);
  f.storage_stage2 = static_cast<std::size_t>(f.stats_.storage_stage2);
  return f;
}

// u (N x nrhs, column major) = A^{-1} f (N x nrhs, column major)
inline std::vector<double> solve(const Factorization& fact, const std::vector<double>& f, int64_t nrhs = 1) {
  const int64_t n = fact.n1 * fact.n2;
  if (nrhs < 0 || static_cast<int64_t>(f.size()) != n * nrhs)
    throw Error("solve: rhs length must equal the grid size");
  std::vector<double> u(f.size());
  detail::check(slablu_gpu_solve(fact.handle(), f.data(), n, nrhs, u.data(), n));
  return u;
}

// ---- validation and reports (problem.hpp:160-206, driver.hpp:182-322) ---------------
struct ErrorReport {
  double relerr_res = 0.0, relerr_true = 0.0;
  int64_t n_rhs = 0;
  bool residual_norm_is_absolute = false, solution_norm_is_absolute = false;
};
// error_report on the GPU (slablu_gpu_error_report): Frobenius norms over the nrhs columns.
inline ErrorReport error_report(const SparseSystem& system, const std::vector<double>& u_calc,
                                const std::vector<double>& u_true, const std::vector<double>& f, int64_t nrhs = 1,
                                int device = 0) {
  const int64_t n = system.dim();
  if (nrhs < 1 || static_cast<int64_t>(u_calc.size()) != n * nrhs ||
      static_cast<int64_t>(u_true.size()) != n * nrhs || static_cast<int64_t>(f.size()) != n * nrhs)
    throw Error("error_report: vector length must equal system dimension");
  double out[4] = {0, 0, 0, 0};
  detail::check(slablu_gpu_error_report(n, system.row_ptr.data(), system.col_idx.data(), system.values.data(),
                                        f.data(), u_calc.data(), u_true.data(), nrhs, device, out));
  ErrorReport r;
  r.relerr_res = out[0];
  r.relerr_true = out[1];
  r.n_rhs = nrhs;
  r.residual_norm_is_absolute = out[2] != 0.0;
  r.solution_norm_is_absolute = out[3] != 0.0;
  return r;
}
inline ErrorReport error_report(const SparseSystem& system, const std::vector<double>& u_calc,
                                const std::vector<double>& u_true) {
  return error_report(system, u_calc, u_true, system.rhs, 1);
}
// sample_field (problem.hpp:199-206): node (i, j) at ((i+1) h, (j+1) h), index i * n2 + j
inline std::vector<double> sample_field(const SparseSystem& system, const ScalarField& field) {
  std::vector<double> v(system.dim());
  for (int64_t i = 0; i < system.n1; i++)
    for (int64_t j = 0; j < system.n2; j++) v[i * system.n2 + j] = field(double(i + 1) * system.h, double(j + 1) * system.h);
  return v;
}

struct SolveReport {
  int64_t n = 0, n1 = 0, n2 = 0, b = 0;
  double kappa = 0.0;
  double t_factor_stage1 = 0.0, t_factor_stage2 = 0.0, t_solve = 0.0;
  std::size_t m_factor_scalars = 0;
  ErrorReport errors{};
  int64_t hbs_max_rank = 0;
  uint64_t seed = 0;
};

inline const char* kCsvHeader =
    "N,n1,n2,b,kappa,T_factor_stage1_s,T_factor_stage2_s,T_solve_s,"
    "M_factor_scalars,relerr_res,relerr_true,hbs_max_rank,seed";

namespace detail {
inline std::string format_double(double v) {
  char buf[40];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}
inline std::string format_time(double v) {
  char buf[40];
  std::snprintf(buf, sizeof(buf), "%.6e", v);
  return buf;
}
}  // namespace detail

// driver.hpp:218-236 column order; `status` appends the benchmark status column
inline std::string csv_row(const SolveReport& r, const char* status = nullptr) {
  std::string row = std::to_string(r.n) + "," + std::to_string(r.n1) + "," + std::to_string(r.n2) + "," +
                    std::to_string(r.b) + "," + detail::format_double(r.kappa) + "," +
                    detail::format_time(r.t_factor_stage1) + "," + detail::format_time(r.t_factor_stage2) + "," +
                    detail::format_time(r.t_solve) + "," + std::to_string(r.m_factor_scalars) + "," +
                    detail::format_double(r.errors.relerr_res) + "," + detail::format_double(r.errors.relerr_true) +
                    "," + std::to_string(r.hbs_max_rank) + "," + std::to_string(r.seed);
  if (status) row += std::string(",") + status;
  return row;
}
// driver.hpp:239-262: the CSV fields under identical names
inline std::string json_row(const SolveReport& r, const char* status = nullptr) {
  std::string out = "{";
  out += "\"N\": " + std::to_string(r.n) + ", ";
  out += "\"n1\": " + std::to_string(r.n1) + ", ";
  out += "\"n2\": " + std::to_string(r.n2) + ", ";
  out += "\"b\": " + std::to_string(r.b) + ", ";
  out += "\"kappa\": " + detail::format_double(r.kappa) + ", ";
  out += "\"T_factor_stage1_s\": " + detail::format_time(r.t_factor_stage1) + ", ";
  out += "\"T_factor_stage2_s\": " + detail::format_time(r.t_factor_stage2) + ", ";
  out += "\"T_solve_s\": " + detail::format_time(r.t_solve) + ", ";
  out += "\"M_factor_scalars\": " + std::to_string(r.m_factor_scalars) + ", ";
  out += "\"relerr_res\": " + detail::format_double(r.errors.relerr_res) + ", ";
  out += "\"relerr_true\": " + detail::format_double(r.errors.relerr_true) + ", ";
  out += "\"hbs_max_rank\": " + std::to_string(r.hbs_max_rank) + ", ";
  out += "\"seed\": " + std::to_string(r.seed);
  if (status) out += std::string(", \"status\": \"") + status + "\"";
  out += "}";
  return out;
}

// run_problem (driver.hpp:268-292): assemble, factorize (device-timed stages), solve (wall clock
// around the call, as the reference), error report against the Dirichlet field
inline SolveReport run_problem(const ProblemSpec& spec, const SolverConfig& config) {
  const SparseSystem system = assemble_fd5(spec);
  SolveReport report;
  report.n = system.dim();
  report.n1 = system.n1;
  report.n2 = system.n2;
  report.kappa = spec.kappa;
  report.seed = config.seed;
  const Factorization fact = factorize(system, config);
  report.b = fact.b;
  report.hbs_max_rank = fact.hbs_max_rank;
  report.t_factor_stage1 = fact.t_stage1;
  report.t_factor_stage2 = fact.t_stage2;
  report.m_factor_scalars = fact.storage_scalars();
  const auto t0 = std::chrono::steady_clock::now();
  const std::vector<double> u = solve(fact, system.rhs);
  report.t_solve = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  const std::vector<double> u_true = sample_field(system, spec.dirichlet_data);
  report.errors = error_report(system, u, u_true);
  return report;
}

// benchmark (driver.hpp:298-322): one report per problem, rows appended as they complete; a
// failed run keeps its row with the error in the status column and the sweep continues
inline std::vector<SolveReport> benchmark(const std::vector<ProblemSpec>& sweep, const SolverConfig& config,
                                          std::ostream* csv = nullptr) {
  std::vector<SolveReport> reports;
  if (csv) *csv << kCsvHeader << ",status\n" << std::flush;
  for (const ProblemSpec& spec : sweep) {
    SolveReport report;
    std::string status = "ok";
    try {
      report = run_problem(spec, config);
    } catch (const Error& e) {
      report.n1 = spec.n1;
      report.n2 = spec.n2;
      report.n = spec.n1 * spec.n2;
      report.kappa = spec.kappa;
      report.seed = config.seed;
      status = std::string("error: ") + e.what();
      for (char& ch : status)
        if (ch == ',' || ch == '\n') ch = ';';
    }
    reports.push_back(report);
    if (csv) *csv << csv_row(report, status.c_str()) << "\n" << std::flush;
  }
  return reports;
}

// ---- multi-GPU shards (no reference counterpart) -------------------
// One process per GPU.  All pointers are device memory of the shard's device; the caller moves
// the n2 x n2 (sweep) and n2 x nrhs (solve) messages between neighbouring ranks, e.g. with
// ncclSend/ncclRecv.  Factorize: eliminate() (no communication), then sweep() in rank order
// (r-1 -> r).  Solve: solve_local() (no communication), solve_forward() in rank order (r-1 -> r),
// solve_backward() in reverse order (r+1 -> r).
class Shard {
 public:
  Shard(int64_t n1, int64_t n2, int64_t nnz, const int32_t* d_row_ptr, const int32_t* d_col_idx,
        const double* d_val, const SolverConfig& config, int rank, int nranks) {
    const slablu_gpu_config c = config.c_config();
    slablu_gpu_fact* raw = nullptr;
    detail::check(slablu_gpu_shard_factorize_device(n1, n2, nnz, d_row_ptr, d_col_idx, d_val, &c, rank, nranks, &raw));
    h_.reset(raw, [](slablu_gpu_fact* f) { slablu_gpu_destroy(f); });
    slablu_gpu_stats_t st{};
    detail::check(slablu_gpu_stats(raw, &st));
    detail::check(slablu_gpu_shard_plan(n1, n2, st.b, rank, nranks, &plan_));
  }
  const slablu_gpu_shard_t& plan() const { return plan_; }
  void eliminate() { detail::check(slablu_gpu_shard_eliminate(h_.get())); }
  void sweep(const double* d_in, double* d_out) { detail::check(slablu_gpu_shard_sweep(h_.get(), d_in, d_out)); }
  void solve_local(const double* d_f, int64_t ldf, int64_t nrhs) {
    detail::check(slablu_gpu_shard_solve_local(h_.get(), d_f, ldf, nrhs));
  }
  void solve_forward(const double* d_in, double* d_out) {
    detail::check(slablu_gpu_shard_solve_forward(h_.get(), d_in, d_out));
  }
  void solve_backward(const double* d_in, double* d_out, double* d_u, int64_t ldu) {
    detail::check(slablu_gpu_shard_solve_backward(h_.get(), d_in, d_out, d_u, ldu));
  }

 private:
  std::shared_ptr<slablu_gpu_fact> h_;
  slablu_gpu_shard_t plan_{};
};

}  // namespace slablu_b200

#endif  // SLABLU_B200_HPP
