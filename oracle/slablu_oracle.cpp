// ============================================================================
//  TEST INFRASTRUCTURE ONLY — CPU oracle for the SlabLU dense-mode path.
//
//  This file is a plain C++17 restatement (no Eigen) of the reference
//  library's factorize/solve path, linked against the LAPACK (OpenBLAS
//  0.3.15, LAPACKE) bundled in this image.  Only tests/, __graft_entry__.smoke()
//  and bench.py's cpu_baseline / --impl reference legs may load it; the
//  product (paper_2211_07572_b200/) never does.
//
//  Every function cites the reference file:line it follows
//  (inc/ = /root/reference/proj/include/slablu/).  The reference itself cannot
//  be compiled here (no Eigen, no lapacke.h).  The
//  restatement is pinned against the reference's own known-answer tests
//  (tests/golden/reference_known_answers.json, tests/test_oracle_*.py).
//
//  Deviations that are not bitwise (documented in DESIGN.md):
//   * Eigen's internal GEMM in SweepFactorization (inc/stage_two.hpp:138-140)
//     and in the sweep solve (:178-185) is replaced by dgemm.
//   * build_reduced's independent blocks and factor_interiors' independent
//     slabs may run on several std::threads (each with single-threaded BLAS);
//     every block is computed by the same sequence of calls, so the result
//     does not depend on the thread count.
// ============================================================================
#include <algorithm>
#include <atomic>
#include <mutex>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

extern "C" {
// LAPACKE / BLAS prototypes (OpenBLAS LP64; lapack_int == int).
int LAPACKE_dgbtrf(int layout, int m, int n, int kl, int ku, double* ab,
                   int ldab, int* ipiv);
int LAPACKE_dgbtrs(int layout, char trans, int n, int kl, int ku, int nrhs,
                   const double* ab, int ldab, const int* ipiv, double* b,
                   int ldb);
int LAPACKE_dgetrf(int layout, int m, int n, double* a, int lda, int* ipiv);
int LAPACKE_dgetrs(int layout, char trans, int n, int nrhs, const double* a,
                   int lda, const int* ipiv, double* b, int ldb);
void dgemm_(const char* ta, const char* tb, const int* m, const int* n,
            const int* k, const double* alpha, const double* a,
            const int* lda, const double* b, const int* ldb,
            const double* beta, double* c, const int* ldc);
void openblas_set_num_threads(int);
int openblas_get_num_threads(void);
}

namespace orc {

constexpr int kColMajor = 102;  // LAPACK_COL_MAJOR

// inc/common.hpp:32-60 — error hierarchy, mapped to status codes.
enum Code { OK = 0, ERR_GENERIC = 1, ERR_CONFIG = 2, ERR_SINGULAR = 3 };
struct Failure {
  int code;
  long index;
  std::string msg;
};
[[noreturn]] inline void fail(int code, const std::string& m, long index = -1) {
  throw Failure{code, index, m};
}

// ---------------------------------------------------------------------------
// inc/bessel.hpp:28-50 — J0 by power series (|t|<=8, long double) or the
// midpoint rule on the integral representation.
double bessel_j0(double t) {
  if (!std::isfinite(t)) fail(ERR_GENERIC, "bessel_j0: argument must be finite");
  t = std::fabs(t);
  if (t <= 8.0) {
    const long double q = static_cast<long double>(t) / 2.0L;
    long double sum = 1.0L, term = 1.0L;
    for (int m = 1; m <= 64; m++) {
      term *= -(q * q) / (static_cast<long double>(m) * m);
      sum += term;
      if (std::fabs(static_cast<double>(term)) < 1e-20) break;
    }
    return static_cast<double>(sum);
  }
  const int n = static_cast<int>(std::ceil(0.75 * t)) + 30;
  const long double lt = static_cast<long double>(t);
  const long double pi = 3.14159265358979323846264338327950288L;
  long double sum = 0.0L;
  for (int k = 0; k < n; k++) {
    const long double theta = pi * (static_cast<long double>(k) + 0.5L) / n;
    sum += std::cos(lt * std::sin(theta));
  }
  return static_cast<double>(sum / n);
}

// inc/problem.hpp:136-149 — manufactured solutions.
double true_solution_poisson(double x, double y) {
  const double r = std::hypot(x + 0.1, y - 0.5);
  if (r == 0.0) fail(ERR_GENERIC, "true_solution_poisson: evaluated at the source point");
  return std::log(r);
}
double true_solution_helmholtz(double x, double y, double kappa) {
  if (kappa < 0.0) fail(ERR_GENERIC, "true_solution_helmholtz: kappa must be nonnegative");
  return bessel_j0(kappa * std::hypot(x + 0.1, y - 0.5));
}

// inc/problem.hpp:153-157
double kappa_from_ppw(double ppw, long n2) {
  if (!(ppw > 0.0)) fail(ERR_CONFIG, "kappa_from_ppw: ppw must be positive");
  if (n2 < 2) fail(ERR_CONFIG, "kappa_from_ppw: n2 must be at least 2");
  return 2.0 * 3.14159265358979323846 * double(n2 + 1) / ppw;
}

// Field selectors standing in for ProblemSpec's std::function members
// (inc/problem.hpp:40-48).  The canned problems of :210-261 and the
// hand-built specs of tests/test_problem.cpp use exactly these fields.
enum Coef { COEF_ONE = 0, COEF_BUMP = 1, COEF_LINEAR_X2Y = 2, COEF_NEG_ONE = 3 };
enum Dir { DIR_ZERO = 0, DIR_POISSON_LOG = 1, DIR_HELMHOLTZ_J0 = 2, DIR_X_PLUS_Y = 3 };

struct Spec {
  long n1, n2;
  double h, kappa;
  int coef, dir;
  double load;   // constant body load
  long bump_n1;  // helmholtz_bump_problem captures n1, n2 (problem.hpp:245-250)
  long bump_n2;
};

double eval_coef(const Spec& s, double x, double y) {
  switch (s.coef) {
    case COEF_ONE: return 1.0;
    case COEF_BUMP: {  // inc/problem.hpp:245-251
      const double h = 1.0 / double(s.bump_n2 + 1);
      const double cx = 0.5 * double(s.bump_n1 + 1) * h, cy = 0.5;
      const double d2 = (x - cx) * (x - cx) + (y - cy) * (y - cy);
      return 1.0 - 0.9 * std::exp(-64.0 * d2);
    }
    case COEF_LINEAR_X2Y: return x + 2.0 * y;
    case COEF_NEG_ONE: return -1.0;
  }
  return 1.0;
}
double eval_dir(const Spec& s, double x, double y) {
  switch (s.dir) {
    case DIR_ZERO: return 0.0;
    case DIR_POISSON_LOG: return true_solution_poisson(x, y);
    case DIR_HELMHOLTZ_J0: return true_solution_helmholtz(x, y, s.kappa);
    case DIR_X_PLUS_Y: return x + y;
  }
  return 0.0;
}

// Row-major CSR with sorted column indices (Eigen RowMajor compressed form).
struct Csr {
  long n = 0;
  std::vector<int32_t> rp, ci;
  std::vector<double> v;
};

struct System {
  Csr a;
  std::vector<double> rhs;
  long n1 = 0, n2 = 0;
  double h = 0;
};

// inc/problem.hpp:78-132 — five-point assembly; Dirichlet data folded in
// neighbour order W, E, S, N; duplicates impossible, so the triplet sort of
// setFromTriplets reduces to column sorting inside each row.
System assemble_fd5(const Spec& spec) {
  if (spec.n2 < 2 || spec.n1 < spec.n2)
    fail(ERR_CONFIG, "assemble_fd5: grid must satisfy n1 >= n2 >= 2");
  if (!(spec.h > 0.0)) fail(ERR_CONFIG, "assemble_fd5: h must be positive");
  if (spec.kappa < 0.0) fail(ERR_CONFIG, "assemble_fd5: kappa must be nonnegative");
  const long n1 = spec.n1, n2 = spec.n2;
  const double h = spec.h;
  const double inv_h2 = 1.0 / (h * h);
  const long n = n1 * n2;
  System sys;
  sys.n1 = n1;
  sys.n2 = n2;
  sys.h = h;
  sys.rhs.assign(n, 0.0);
  sys.a.n = n;
  sys.a.rp.assign(n + 1, 0);
  sys.a.ci.reserve(5 * n);
  sys.a.v.reserve(5 * n);
  for (long i = 0; i < n1; i++) {
    for (long j = 0; j < n2; j++) {
      const long row = i * n2 + j;
      const double x = double(i + 1) * h;
      const double y = double(j + 1) * h;
      const double b = eval_coef(spec, x, y);
      if (b < 0.0) fail(ERR_GENERIC, "assemble_fd5: coefficient field is negative at a node");
      const double diag = 4.0 * inv_h2 - spec.kappa * spec.kappa * b;
      double r = spec.load;
      const long di[4] = {-1, 1, 0, 0};
      const long dj[4] = {0, 0, -1, 1};
      long cols[5];
      double vals[5];
      int cnt = 0;
      cols[cnt] = row;
      vals[cnt++] = diag;
      for (int s = 0; s < 4; s++) {
        const long ii = i + di[s], jj = j + dj[s];
        if (ii >= 0 && ii < n1 && jj >= 0 && jj < n2) {
          cols[cnt] = ii * n2 + jj;
          vals[cnt++] = -inv_h2;
        } else {
          r += eval_dir(spec, double(ii + 1) * h, double(jj + 1) * h) * inv_h2;
        }
      }
      sys.rhs[row] = r;
      // sort by column (insertion sort over <= 5 entries)
      for (int a = 1; a < cnt; a++)
        for (int c = a; c > 0 && cols[c - 1] > cols[c]; c--) {
          std::swap(cols[c - 1], cols[c]);
          std::swap(vals[c - 1], vals[c]);
        }
      for (int a = 0; a < cnt; a++) {
        sys.a.ci.push_back(static_cast<int32_t>(cols[a]));
        sys.a.v.push_back(vals[a]);
      }
      sys.a.rp[row + 1] = static_cast<int32_t>(sys.a.ci.size());
    }
  }
  return sys;
}

// ---------------------------------------------------------------------------
// inc/partition.hpp:27-91
struct Strip {
  long first_col, width;
};
struct Partition {
  long n1 = 0, n2 = 0, b = 0;
  std::vector<Strip> interfaces, interiors;
  long nifc() const { return (long)interfaces.size(); }
  long nint() const { return (long)interiors.size(); }
  long dim() const { return n1 * n2; }
  long ifc_off(long j) const { return interfaces[j].first_col * n2; }
  long int_off(long i) const { return interiors[i].first_col * n2; }
  long int_size(long i) const { return interiors[i].width * n2; }
};

Partition partition(long n1, long n2, long b) {
  if (n2 < 1) fail(ERR_CONFIG, "partition: n2 must be positive");
  if (b < 1 || b > n1 - 2)
    fail(ERR_CONFIG, "partition: slab width must satisfy 1 <= b <= n1 - 2");
  Partition p;
  p.n1 = n1;
  p.n2 = n2;
  p.b = b;
  long col = 0;
  for (long t = 1; col < n1; t++) {
    const long ifc = t * (b + 1) - 1;
    const long stop = std::min(ifc, n1);
    if (stop > col) p.interiors.push_back({col, stop - col});
    col = stop;
    if (col == ifc && col < n1) {
      p.interfaces.push_back({col, 1});
      col++;
    }
  }
  return p;
}

// inc/driver.hpp:55-66
long choose_b(long n1, long n2, long b, double c) {
  if (b > 0) return b;
  if (n2 < 8) fail(ERR_CONFIG, "choose_b: n2 must be at least 8");
  if (!(c > 0.0) || c > 2.0) fail(ERR_CONFIG, "choose_b: coefficient c must lie in (0, 2]");
  const double raw = c * std::pow(double(n2), 2.0 / 3.0);
  const long rounded = 10 * static_cast<long>(std::llround(raw / 10.0));
  const long hi = std::max<long>(1, n1 / 2);
  return std::clamp(rounded, std::min<long>(10, hi), hi);
}

// ---------------------------------------------------------------------------
// inc/banded.hpp:33-128 — LAPACK band storage + dgbtrf/dgbtrs.
struct BandedLU {
  long n = 0, kl = 0, ku = 0, ldab = 0;
  std::vector<double> band;
  std::vector<int> ipiv;
  double& at(long i, long j) {
    if (i < 0 || j < 0 || i >= n || j >= n || i - j > kl || j - i > ku)
      fail(ERR_GENERIC, "BandedMatrix::at: index outside band");
    return band[(size_t)j * ldab + kl + ku + i - j];
  }
  void init(long n_, long kl_, long ku_) {
    if (n_ < 1 || kl_ < 0 || ku_ < 0 || kl_ >= n_ || ku_ >= n_)
      fail(ERR_GENERIC, "BandedMatrix: inconsistent bandwidths");
    n = n_;
    kl = kl_;
    ku = ku_;
    ldab = 2 * kl + ku + 1;
    band.assign((size_t)ldab * n, 0.0);
  }
  void factor() {  // inc/banded.hpp:99-111
    ipiv.assign(n, 0);
    int info = LAPACKE_dgbtrf(kColMajor, (int)n, (int)n, (int)kl, (int)ku,
                              band.data(), (int)ldab, ipiv.data());
    if (info > 0) fail(ERR_SINGULAR, "BandedLU: exactly singular pivot", info - 1);
    if (info < 0) fail(ERR_GENERIC, "BandedLU: illegal argument to dgbtrf");
  }
  // inc/banded.hpp:116-128 (in place on b, ldb = n)
  void solve(double* b, long nrhs, bool adjoint = false) const {
    if (nrhs == 0) return;
    int info = LAPACKE_dgbtrs(kColMajor, adjoint ? 'T' : 'N', (int)n, (int)kl,
                              (int)ku, (int)nrhs, band.data(), (int)ldab,
                              ipiv.data(), b, (int)n);
    if (info != 0) fail(ERR_GENERIC, "BandedLU: dgbtrs failed");
  }
};

// inc/dense.hpp:29-61
struct DenseLU {
  long n = 0;
  std::vector<double> lu;
  std::vector<int> ipiv;
  void factor() {
    ipiv.assign(n, 0);
    if (n == 0) return;
    int info = LAPACKE_dgetrf(kColMajor, (int)n, (int)n, lu.data(), (int)n, ipiv.data());
    if (info > 0) fail(ERR_SINGULAR, "DenseLU: exactly singular pivot", info - 1);
    if (info < 0) fail(ERR_GENERIC, "DenseLU: illegal argument to dgetrf");
  }
  void solve(double* b, long nrhs, long ldb, bool adjoint = false) const {
    if (n == 0 || nrhs == 0) return;
    int info = LAPACKE_dgetrs(kColMajor, adjoint ? 'T' : 'N', (int)n, (int)nrhs,
                              lu.data(), (int)n, ipiv.data(), b, (int)ldb);
    if (info != 0) fail(ERR_GENERIC, "DenseLU: dgetrs failed");
  }
};

// C(m x n) += alpha * A(m x k) * B(k x n), all column major.
void gemm(long m, long n, long k, double alpha, const double* a, long lda,
          const double* b, long ldb, double beta, double* c, long ldc) {
  if (m == 0 || n == 0) return;
  int im = (int)m, in = (int)n, ik = (int)k, ila = (int)lda, ilb = (int)ldb, ilc = (int)ldc;
  dgemm_("N", "N", &im, &in, &ik, &alpha, a, &ila, b, &ilb, &beta, c, &ilc);
}

// Sparse coupling block as triplets (row, col, value) — the reference keeps
// them as Eigen column-major sparse matrices (inc/stage_one.hpp:100-101).
struct Trip {
  long r, c;
  double v;
};
struct Sparse {
  long rows = 0, cols = 0;
  std::vector<Trip> t;
};

// ---------------------------------------------------------------------------
// inc/stage_one.hpp:96-159 — SlabFactor with permuted (iy*w+ix) interior.
struct SlabFactor {
  long strip, first_col, width, n2, left_ifc, right_ifc;
  BandedLU lu;
  Sparse from_left, from_right, to_left, to_right;
  long rows() const { return width * n2; }
  // permute_in (:108-114): natural (ix*n2+iy) -> banded (iy*w+ix)
  void permute_in(const double* f, long ldf, long nrhs, double* out) const {
    const long m = rows();
    for (long c = 0; c < nrhs; c++)
      for (long ix = 0; ix < width; ix++)
        for (long iy = 0; iy < n2; iy++)
          out[c * m + iy * width + ix] = f[c * ldf + ix * n2 + iy];
  }
  void permute_out(const double* u, long nrhs, double* out, long ldo) const {
    const long m = rows();
    for (long c = 0; c < nrhs; c++)
      for (long ix = 0; ix < width; ix++)
        for (long iy = 0; iy < n2; iy++)
          out[c * ldo + ix * n2 + iy] = u[c * m + iy * width + ix];
  }
};

// inc/stage_one.hpp:163-238
SlabFactor factor_one_interior(const System& sys, const Partition& part, long strip) {
  const long n2 = part.n2;
  const Strip& st = part.interiors[strip];
  const long w = st.width, col0 = st.first_col;
  const long begin = col0 * n2, end = (col0 + w) * n2;
  const long left = strip > 0 ? strip - 1 : -1;
  const long right = strip < part.nifc() ? strip : -1;
  const long left_off = left >= 0 ? part.ifc_off(left) : -1;
  const long right_off = right >= 0 ? part.ifc_off(right) : -1;
  SlabFactor f;
  f.strip = strip;
  f.first_col = col0;
  f.width = w;
  f.n2 = n2;
  f.left_ifc = left;
  f.right_ifc = right;
  f.lu.init(w * n2, w, w);
  f.from_left = {w * n2, left >= 0 ? n2 : 0, {}};
  f.from_right = {w * n2, right >= 0 ? n2 : 0, {}};
  f.to_left = {left >= 0 ? n2 : 0, w * n2, {}};
  f.to_right = {right >= 0 ? n2 : 0, w * n2, {}};
  const Csr& a = sys.a;
  for (long ix = 0; ix < w; ix++)
    for (long iy = 0; iy < n2; iy++) {
      const long g = (col0 + ix) * n2 + iy;
      const long r = iy * w + ix;
      for (long p = a.rp[g]; p < a.rp[g + 1]; p++) {
        const long c = a.ci[p];
        if (c >= begin && c < end) {
          const long cx = c / n2 - col0, cy = c % n2;
          f.lu.at(r, cy * w + cx) = a.v[p];
        } else if (left >= 0 && c >= left_off && c < left_off + n2) {
          f.from_left.t.push_back({r, c - left_off, a.v[p]});
        } else if (right >= 0 && c >= right_off && c < right_off + n2) {
          f.from_right.t.push_back({r, c - right_off, a.v[p]});
        } else {
          fail(ERR_GENERIC, "factor_one_interior: interior couples past its adjacent interfaces");
        }
      }
    }
  auto gather = [&](long off, Sparse& out) {
    for (long q = 0; q < n2; q++)
      for (long p = a.rp[off + q]; p < a.rp[off + q + 1]; p++) {
        const long c = a.ci[p];
        if (c >= begin && c < end) {
          const long cx = c / n2 - col0, cy = c % n2;
          out.t.push_back({q, cy * w + cx, a.v[p]});
        }
      }
  };
  if (left >= 0) gather(left_off, f.to_left);
  if (right >= 0) gather(right_off, f.to_right);
  try {
    f.lu.factor();
  } catch (const Failure& e) {
    if (e.code == ERR_SINGULAR)
      fail(ERR_SINGULAR, "factor_one_interior: singular slab interior", strip);
    throw;
  }
  return f;
}

// Run fn(i) for i in [0, count) on up to `threads` std::threads.
template <class F>
void parallel_for(long count, int threads, F fn) {
  if (threads <= 1 || count <= 1) {
    for (long i = 0; i < count; i++) fn(i);
    return;
  }
  std::atomic<long> next{0};
  std::vector<Failure> errs;
  std::vector<long> err_idx;
  std::mutex* mu = new std::mutex;
  std::vector<std::thread> pool;
  for (int t = 0; t < std::min<long>(threads, count); t++)
    pool.emplace_back([&]() {
      for (;;) {
        const long i = next.fetch_add(1);
        if (i >= count) return;
        try {
          fn(i);
        } catch (const Failure& e) {
          std::lock_guard<std::mutex> g(*mu);
          errs.push_back(e);
          err_idx.push_back(i);
        }
      }
    });
  for (auto& th : pool) th.join();
  delete mu;
  if (!errs.empty()) {  // deterministic: report the lowest index
    size_t best = 0;
    for (size_t e = 1; e < errs.size(); e++)
      if (err_idx[e] < err_idx[best]) best = e;
    throw errs[best];
  }
}

// inc/stage_one.hpp:242-251
std::vector<SlabFactor> factor_interiors(const System& sys, const Partition& part, int threads) {
  if (sys.n1 != part.n1 || sys.n2 != part.n2)
    fail(ERR_GENERIC, "factor_interiors: system and partition dimensions differ");
  std::vector<SlabFactor> f(part.nint());
  parallel_for(part.nint(), threads, [&](long i) { f[i] = factor_one_interior(sys, part, i); });
  return f;
}

// y(rows x ncol) = S * x or S^T * x (x dense, column major with ld = its rows)
void sparse_apply(const Sparse& s, bool transpose, const double* x, long ncol, double* y) {
  const long out_rows = transpose ? s.cols : s.rows;
  const long in_rows = transpose ? s.rows : s.cols;
  std::fill(y, y + out_rows * ncol, 0.0);
  for (long c = 0; c < ncol; c++)
    for (const Trip& t : s.t) {
      if (!transpose)
        y[c * out_rows + t.r] += t.v * x[c * in_rows + t.c];
      else
        y[c * out_rows + t.c] += t.v * x[c * in_rows + t.r];
    }
}

// Dense copy of the CSR block rows [r0, r0+nr) x cols [c0, c0+nc) (stage_one.hpp:40-55)
std::vector<double> dense_block(const Csr& a, long r0, long nr, long c0, long nc) {
  std::vector<double> d(nr * nc, 0.0);
  for (long r = 0; r < nr; r++)
    for (long p = a.rp[r0 + r]; p < a.rp[r0 + r + 1]; p++) {
      const long c = a.ci[p];
      if (c >= c0 && c < c0 + nc) d[(c - c0) * nr + r] = a.v[p];
    }
  return d;
}

// inc/stage_one.hpp:258-299 — y = T_jk x (or T_jk^T x); x is n2 x ncol.
// RHS columns may be split into chunks of `chunk` columns: dgbtrs is column
// independent, so the result is unchanged.
std::vector<double> apply_T_block(long j, long k, const double* x, long ncol, bool adjoint,
                                  const std::vector<SlabFactor>& fac, const System& sys,
                                  const Partition& part, long chunk = 0) {
  const long n2 = part.n2, nifc = part.nifc();
  if (j < 0 || j >= nifc || k < 0 || k >= nifc)
    fail(ERR_GENERIC, "apply_T_block: interface index out of range");
  if (j != k && j != k + 1 && k != j + 1)
    fail(ERR_GENERIC, "apply_T_block: interfaces are not adjacent");
  std::vector<double> direct = dense_block(sys.a, part.ifc_off(j), n2, part.ifc_off(k), n2);
  std::vector<double> y(n2 * ncol, 0.0);
  // direct term (:270-273): Eigen sparse*dense; the 5-point direct block is
  // tridiagonal, so dense evaluation sums the same products in the same order.
  for (long c = 0; c < ncol; c++)
    for (long q = 0; q < n2; q++) {
      double s = 0.0;
      for (long r = 0; r < n2; r++) {
        const double d = adjoint ? direct[q * n2 + r] : direct[r * n2 + q];
        if (d != 0.0) s += d * x[c * n2 + r];
      }
      y[c * n2 + q] = s;
    }
  if (chunk <= 0) chunk = ncol;
  auto schur_term = [&](const SlabFactor& f, bool via_right_of_j, bool via_right_of_k) {
    const Sparse& out_blk = via_right_of_j ? f.to_right : f.to_left;
    const Sparse& in_blk = via_right_of_k ? f.from_right : f.from_left;
    const long m = f.rows();
    std::vector<double> tmp(m * std::min(chunk, ncol));
    std::vector<double> part_out(n2 * std::min(chunk, ncol));
    for (long c0 = 0; c0 < ncol; c0 += chunk) {
      const long nc = std::min(chunk, ncol - c0);
      if (!adjoint) {
        sparse_apply(in_blk, false, x + c0 * n2, nc, tmp.data());
        f.lu.solve(tmp.data(), nc, false);
        sparse_apply(out_blk, false, tmp.data(), nc, part_out.data());
      } else {
        sparse_apply(out_blk, true, x + c0 * n2, nc, tmp.data());
        f.lu.solve(tmp.data(), nc, true);
        sparse_apply(in_blk, true, tmp.data(), nc, part_out.data());
      }
      for (long i = 0; i < n2 * nc; i++) y[c0 * n2 + i] -= part_out[i];
    }
  };
  if (j == k) {
    schur_term(fac[j], true, true);
    if (j + 1 < part.nint()) schur_term(fac[j + 1], false, false);
  } else if (k == j + 1) {
    schur_term(fac[j + 1], false, true);
  } else {
    schur_term(fac[j], true, false);
  }
  return y;
}

// inc/stage_two.hpp:31-56
struct BlockTri {
  long k = 0, m = 0;
  std::vector<std::vector<double>> diag, sub, super;
  void validate() const {
    if (k == 0) fail(ERR_CONFIG, "BlockTridiagonal: no blocks");
    if ((long)sub.size() != k - 1 || (long)super.size() != k - 1)
      fail(ERR_CONFIG, "BlockTridiagonal: off-diagonal count must be k - 1");
    auto check = [&](const std::vector<double>& b) {
      if ((long)b.size() != m * m) fail(ERR_CONFIG, "BlockTridiagonal: inconsistent block dimensions");
      for (double v : b)
        if (!std::isfinite(v)) fail(ERR_GENERIC, "BlockTridiagonal: non-finite block entry");
    };
    for (auto& b : diag) check(b);
    for (auto& b : sub) check(b);
    for (auto& b : super) check(b);
  }
};

// inc/stage_one.hpp:357-411 (dense branch): diag blocks first, then
// super/sub pairs; each block = apply_T_block(j, k, Identity(n2)).
BlockTri build_reduced(const System& sys, const Partition& part,
                       const std::vector<SlabFactor>& fac, int threads, long chunk) {
  const long n2 = part.n2, nifc = part.nifc();
  if ((long)fac.size() != part.nint())
    fail(ERR_GENERIC, "build_reduced: factor list does not match the partition");
  BlockTri t;
  t.k = nifc;
  t.m = n2;
  t.diag.resize(nifc);
  t.super.resize(std::max<long>(0, nifc - 1));
  t.sub.resize(std::max<long>(0, nifc - 1));
  std::vector<double> eye(n2 * n2, 0.0);
  for (long i = 0; i < n2; i++) eye[i * n2 + i] = 1.0;
  const long nblocks = 3 * nifc - 2;
  parallel_for(nblocks, threads, [&](long b) {
    if (b < nifc) {
      t.diag[b] = apply_T_block(b, b, eye.data(), n2, false, fac, sys, part, chunk);
    } else {
      const long j = (b - nifc) / 2;
      if ((b - nifc) % 2 == 0)
        t.super[j] = apply_T_block(j, j + 1, eye.data(), n2, false, fac, sys, part, chunk);
      else
        t.sub[j] = apply_T_block(j + 1, j, eye.data(), n2, false, fac, sys, part, chunk);
    }
  });
  return t;
}

// inc/stage_two.hpp:127-150 — sweeping block LU.
struct Sweep {
  long k = 0, m = 0;
  std::vector<DenseLU> S;
  std::vector<std::vector<double>> sub, super;
};

Sweep sweep_build(BlockTri t) {
  t.validate();
  Sweep sw;
  sw.k = t.k;
  sw.m = t.m;
  const long m = t.m;
  sw.S.resize(t.k);
  for (long j = 0; j < t.k; j++) {
    DenseLU& f = sw.S[j];
    f.n = m;
    f.lu = std::move(t.diag[j]);
    if (j > 0) {
      std::vector<double> x = t.super[j - 1];
      sw.S[j - 1].solve(x.data(), m, m);
      gemm(m, m, m, -1.0, t.sub[j - 1].data(), m, x.data(), m, 1.0, f.lu.data(), m);
    }
    try {
      f.factor();
    } catch (const Failure& e) {
      if (e.code == ERR_SINGULAR)
        fail(ERR_SINGULAR, "sweep_build: singular Schur complement block", j);
      throw;
    }
  }
  sw.sub = std::move(t.sub);
  sw.super = std::move(t.super);
  return sw;
}

// inc/stage_two.hpp:170-188 — f is (k*m) x nrhs, ld = k*m.
std::vector<double> sweep_solve(const Sweep& sw, const double* f, long nrhs) {
  const long k = sw.k, m = sw.m, ld = k * m;
  std::vector<double> u(ld * nrhs);
  std::vector<double> rhs(m * nrhs);
  for (long j = 0; j < k; j++) {
    for (long c = 0; c < nrhs; c++)
      std::memcpy(&rhs[c * m], f + c * ld + j * m, m * sizeof(double));
    if (j > 0) gemm(m, nrhs, m, -1.0, sw.sub[j - 1].data(), m, u.data() + (j - 1) * m, ld, 1.0, rhs.data(), m);
    sw.S[j].solve(rhs.data(), nrhs, m);
    for (long c = 0; c < nrhs; c++)
      std::memcpy(u.data() + c * ld + j * m, &rhs[c * m], m * sizeof(double));
  }
  for (long j = k - 2; j >= 0; j--) {
    gemm(m, nrhs, m, 1.0, sw.super[j].data(), m, u.data() + (j + 1) * m, ld, 0.0, rhs.data(), m);
    sw.S[j].solve(rhs.data(), nrhs, m);
    for (long c = 0; c < nrhs; c++)
      for (long i = 0; i < m; i++) u[c * ld + j * m + i] -= rhs[c * m + i];
  }
  return u;
}

// inc/stage_one.hpp:415-433
std::vector<double> reduce_rhs(const double* f, long nrhs, const std::vector<SlabFactor>& fac,
                               const Partition& part) {
  const long n2 = part.n2, N = part.dim(), K = part.nifc() * n2;
  std::vector<double> out(K * nrhs);
  for (long j = 0; j < part.nifc(); j++)
    for (long c = 0; c < nrhs; c++)
      std::memcpy(&out[c * K + j * n2], f + c * N + part.ifc_off(j), n2 * sizeof(double));
  for (const SlabFactor& fc : fac) {
    const long m = fc.rows();
    std::vector<double> g(m * nrhs);
    fc.permute_in(f + part.int_off(fc.strip), N, nrhs, g.data());
    fc.lu.solve(g.data(), nrhs, false);
    std::vector<double> tmp(n2 * nrhs);
    if (fc.left_ifc >= 0) {
      sparse_apply(fc.to_left, false, g.data(), nrhs, tmp.data());
      for (long c = 0; c < nrhs; c++)
        for (long i = 0; i < n2; i++) out[c * K + fc.left_ifc * n2 + i] -= tmp[c * n2 + i];
    }
    if (fc.right_ifc >= 0) {
      sparse_apply(fc.to_right, false, g.data(), nrhs, tmp.data());
      for (long c = 0; c < nrhs; c++)
        for (long i = 0; i < n2; i++) out[c * K + fc.right_ifc * n2 + i] -= tmp[c * n2 + i];
    }
  }
  return out;
}

// inc/stage_one.hpp:438-462
std::vector<double> recover_interiors(const double* u_ifc, const double* f, long nrhs,
                                      const std::vector<SlabFactor>& fac, const Partition& part) {
  const long n2 = part.n2, N = part.dim(), K = part.nifc() * n2;
  std::vector<double> u(N * nrhs);
  for (long j = 0; j < part.nifc(); j++)
    for (long c = 0; c < nrhs; c++)
      std::memcpy(&u[c * N + part.ifc_off(j)], u_ifc + c * K + j * n2, n2 * sizeof(double));
  for (const SlabFactor& fc : fac) {
    const long m = fc.rows();
    std::vector<double> rhs(m * nrhs), tmp(m * nrhs), ui(n2 * nrhs);
    fc.permute_in(f + part.int_off(fc.strip), N, nrhs, rhs.data());
    auto sub_coupling = [&](const Sparse& s, long ifc) {
      for (long c = 0; c < nrhs; c++)
        std::memcpy(&ui[c * n2], u_ifc + c * K + ifc * n2, n2 * sizeof(double));
      sparse_apply(s, false, ui.data(), nrhs, tmp.data());
      for (long i = 0; i < m * nrhs; i++) rhs[i] -= tmp[i];
    };
    if (fc.left_ifc >= 0) sub_coupling(fc.from_left, fc.left_ifc);
    if (fc.right_ifc >= 0) sub_coupling(fc.from_right, fc.right_ifc);
    fc.lu.solve(rhs.data(), nrhs, false);
    fc.permute_out(rhs.data(), nrhs, u.data() + part.int_off(fc.strip), N);
  }
  return u;
}

// inc/driver.hpp:72-87, 100-167 — dense-mode factorization.
struct Factorization {
  long n1 = 0, n2 = 0, b = 0;
  Partition part;
  std::vector<SlabFactor> slabs;
  Sweep sweep;
  bool has_sweep = false;
  BandedLU whole;
  bool single_slab = false;
  double t_stage1 = 0, t_stage2 = 0;
  size_t storage_stage1 = 0, storage_stage2 = 0;
  BlockTri reduced_copy;  // staged-parity snapshot of T (optional)
};

double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

Factorization* factorize(const System& sys, long b_cfg, double c, int threads, long chunk,
                         bool keep_T) {
  if (sys.a.n == 0) fail(ERR_CONFIG, "factorize: empty system");
  auto* fact = new Factorization;
  try {
    fact->n1 = sys.n1;
    fact->n2 = sys.n2;
    fact->b = b_cfg > 0 ? b_cfg : choose_b(sys.n1, sys.n2, 0, c);
    const auto t0 = std::chrono::steady_clock::now();
    if (fact->b > sys.n1 - 2 || sys.n1 < 3) {  // driver.hpp:134-139, 100-109
      const long n = sys.a.n, n2 = sys.n2;
      fact->whole.init(n, n2, n2);
      for (long r = 0; r < n; r++)
        for (long p = sys.a.rp[r]; p < sys.a.rp[r + 1]; p++) fact->whole.at(r, sys.a.ci[p]) = sys.a.v[p];
      fact->whole.factor();
      fact->single_slab = true;
      fact->storage_stage1 = fact->whole.band.size();
      fact->t_stage1 = seconds_since(t0);
      return fact;
    }
    fact->part = partition(sys.n1, sys.n2, fact->b);
    fact->slabs = factor_interiors(sys, fact->part, threads);
    BlockTri red = build_reduced(sys, fact->part, fact->slabs, threads, chunk);
    for (const SlabFactor& f : fact->slabs)
      fact->storage_stage1 += f.lu.band.size() + f.from_left.t.size() + f.from_right.t.size() +
                              f.to_left.t.size() + f.to_right.t.size();
    fact->t_stage1 = seconds_since(t0);
    if (keep_T) fact->reduced_copy = red;
    const auto t1 = std::chrono::steady_clock::now();
    fact->sweep = sweep_build(std::move(red));
    fact->has_sweep = true;
    const long m = fact->sweep.m;
    fact->storage_stage2 = (size_t)(fact->sweep.k + 2 * (fact->sweep.k - 1)) * m * m;
    fact->t_stage2 = seconds_since(t1);
  } catch (...) {
    delete fact;
    throw;
  }
  return fact;
}

// inc/driver.hpp:171-179
std::vector<double> solve(const Factorization& fact, const double* f, long nrhs) {
  const long N = fact.n1 * fact.n2;
  if (fact.single_slab) {
    std::vector<double> u(f, f + N * nrhs);
    fact.whole.solve(u.data(), nrhs, false);
    return u;
  }
  std::vector<double> red = reduce_rhs(f, nrhs, fact.slabs, fact.part);
  std::vector<double> u_ifc = sweep_solve(fact.sweep, red.data(), nrhs);
  return recover_interiors(u_ifc.data(), f, nrhs, fact.slabs, fact.part);
}

}  // namespace orc

// ===========================================================================
//  C ABI for ctypes (tests / bench cpu_baseline only).
// ===========================================================================
using namespace orc;

namespace {
thread_local std::string g_err;
thread_local long g_err_index = -1;
int set_err(const Failure& e) {
  g_err = e.msg;
  g_err_index = e.index;
  return e.code;
}
#define ORC_TRY(...)                         \
  try {                                      \
    __VA_ARGS__;                             \
    return 0;                                \
  } catch (const Failure& e) {               \
    return set_err(e);                       \
  } catch (const std::exception& e) {        \
    g_err = e.what();                        \
    g_err_index = -1;                        \
    return ERR_GENERIC;                      \
  }

Spec make_spec(long n1, long n2, double h, double kappa, int coef, int dir, double load) {
  Spec s{n1, n2, h, kappa, coef, dir, load, n1, n2};
  return s;
}
}  // namespace

struct orc_system {
  System sys;
};

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
long orc_last_error_index(void) { return g_err_index; }
void orc_set_blas_threads(int t) { openblas_set_num_threads(t); }
int orc_get_blas_threads(void) { return openblas_get_num_threads(); }

double orc_bessel_j0(double t) {
  try {
    return bessel_j0(t);
  } catch (...) {
    return NAN;
  }
}
double orc_true_solution_poisson(double x, double y) {
  try {
    return true_solution_poisson(x, y);
  } catch (...) {
    return NAN;
  }
}
double orc_true_solution_helmholtz(double x, double y, double k) {
  try {
    return true_solution_helmholtz(x, y, k);
  } catch (...) {
    return NAN;
  }
}
int orc_kappa_from_ppw(double ppw, long n2, double* out) { ORC_TRY(*out = kappa_from_ppw(ppw, n2)) }
int orc_choose_b(long n1, long n2, long b, double c, long* out) { ORC_TRY(*out = choose_b(n1, n2, b, c)) }

// partition: fills up to `cap` (first_col, width) pairs for interiors and interfaces.
int orc_partition(long n1, long n2, long b, long* n_int, long* int_cols, long* n_ifc,
                  long* ifc_cols, long cap) {
  ORC_TRY({
    Partition p = partition(n1, n2, b);
    *n_int = p.nint();
    *n_ifc = p.nifc();
    for (long i = 0; i < p.nint() && i < cap; i++) {
      int_cols[2 * i] = p.interiors[i].first_col;
      int_cols[2 * i + 1] = p.interiors[i].width;
    }
    for (long i = 0; i < p.nifc() && i < cap; i++) {
      ifc_cols[2 * i] = p.interfaces[i].first_col;
      ifc_cols[2 * i + 1] = p.interfaces[i].width;
    }
  })
}

// Assemble a spec (field selectors as in make_spec); returns an opaque system.
int orc_assemble(long n1, long n2, double h, double kappa, int coef, int dir, double load,
                 orc_system** out) {
  ORC_TRY({
    auto* s = new orc_system;
    try {
      s->sys = assemble_fd5(make_spec(n1, n2, h, kappa, coef, dir, load));
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  })
}
// Canned problems (inc/problem.hpp:210-261): 0 poisson_log, 1 helmholtz, 2 helmholtz_bump.
int orc_assemble_canned(int kind, long n1, long n2, double kappa, orc_system** out) {
  const double h = 1.0 / double(n2 + 1);
  if (kind == 0) return orc_assemble(n1, n2, h, 0.0, COEF_ONE, DIR_POISSON_LOG, 0.0, out);
  if (kind == 1) return orc_assemble(n1, n2, h, kappa, COEF_ONE, DIR_HELMHOLTZ_J0, 0.0, out);
  if (kind == 2) return orc_assemble(n1, n2, h, kappa, COEF_BUMP, DIR_HELMHOLTZ_J0, 0.0, out);
  g_err = "unknown problem kind";
  return ERR_CONFIG;
}
// Wrap a caller CSR (copied).
int orc_system_from_csr(long n1, long n2, double h, const int32_t* rp, const int32_t* ci,
                        const double* v, const double* rhs, orc_system** out) {
  ORC_TRY({
    auto* s = new orc_system;
    const long n = n1 * n2;
    s->sys.n1 = n1;
    s->sys.n2 = n2;
    s->sys.h = h;
    s->sys.a.n = n;
    s->sys.a.rp.assign(rp, rp + n + 1);
    s->sys.a.ci.assign(ci, ci + rp[n]);
    s->sys.a.v.assign(v, v + rp[n]);
    s->sys.rhs.assign(rhs, rhs + n);
    *out = s;
  })
}
void orc_system_free(orc_system* s) { delete s; }
long orc_system_dim(const orc_system* s) { return s->sys.a.n; }
long orc_system_nnz(const orc_system* s) { return (long)s->sys.a.ci.size(); }
void orc_system_csr(const orc_system* s, int32_t* rp, int32_t* ci, double* v, double* rhs) {
  const auto& a = s->sys.a;
  if (rp) std::memcpy(rp, a.rp.data(), a.rp.size() * sizeof(int32_t));
  if (ci) std::memcpy(ci, a.ci.data(), a.ci.size() * sizeof(int32_t));
  if (v) std::memcpy(v, a.v.data(), a.v.size() * sizeof(double));
  if (rhs) std::memcpy(rhs, s->sys.rhs.data(), s->sys.rhs.size() * sizeof(double));
}
// Sample a canned problem's Dirichlet field on the grid (inc/problem.hpp:199-206).
int orc_sample_dirichlet(int kind, long n1, long n2, double kappa, double* out) {
  ORC_TRY({
    const double h = 1.0 / double(n2 + 1);
    for (long i = 0; i < n1; i++)
      for (long j = 0; j < n2; j++) {
        const double x = double(i + 1) * h, y = double(j + 1) * h;
        out[i * n2 + j] = kind == 0 ? true_solution_poisson(x, y) : true_solution_helmholtz(x, y, kappa);
      }
  })
}
// y = A x for nrhs columns (ld = N).
void orc_spmv(const orc_system* s, const double* x, long nrhs, double* y) {
  const auto& a = s->sys.a;
  for (long c = 0; c < nrhs; c++)
    for (long r = 0; r < a.n; r++) {
      double acc = 0.0;
      for (long p = a.rp[r]; p < a.rp[r + 1]; p++) acc += a.v[p] * x[c * a.n + a.ci[p]];
      y[c * a.n + r] = acc;
    }
}

struct orc_fact {
  Factorization* f;
  const orc_system* sys;
};

int orc_factorize(const orc_system* s, long b, double c, int threads, long chunk, int keep_T,
                  orc_fact** out) {
  ORC_TRY({
    auto* h = new orc_fact{nullptr, s};
    try {
      h->f = factorize(s->sys, b, c, threads, chunk, keep_T != 0);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  })
}
void orc_fact_free(orc_fact* h) {
  if (h) delete h->f;
  delete h;
}
// stats: [b, k(ifc), strips, single_slab, storage1, storage2]; times: [t1, t2]
void orc_fact_stats(const orc_fact* h, long* stats, double* times) {
  const Factorization& f = *h->f;
  stats[0] = f.b;
  stats[1] = f.single_slab ? 0 : f.part.nifc();
  stats[2] = f.single_slab ? 1 : f.part.nint();
  stats[3] = f.single_slab ? 1 : 0;
  stats[4] = (long)f.storage_stage1;
  stats[5] = (long)f.storage_stage2;
  times[0] = f.t_stage1;
  times[1] = f.t_stage2;
}
// Copy a reduced block (before sweep factorization; requires keep_T).
// which: 0 diag[j], 1 super[j], 2 sub[j]
int orc_fact_T_block(const orc_fact* h, int which, long j, double* out) {
  ORC_TRY({
    const BlockTri& t = h->f->reduced_copy;
    const std::vector<std::vector<double>>& v = which == 0 ? t.diag : which == 1 ? t.super : t.sub;
    if (j < 0 || j >= (long)v.size()) fail(ERR_GENERIC, "T block index out of range");
    std::memcpy(out, v[j].data(), v[j].size() * sizeof(double));
  })
}
int orc_solve(const orc_fact* h, const double* f, long nrhs, double* u) {
  ORC_TRY({
    std::vector<double> r = solve(*h->f, f, nrhs);
    std::memcpy(u, r.data(), r.size() * sizeof(double));
  })
}
// Staged: reduced rhs (k*n2 x nrhs).
int orc_reduce_rhs(const orc_fact* h, const double* f, long nrhs, double* out) {
  ORC_TRY({
    std::vector<double> r = reduce_rhs(f, nrhs, h->f->slabs, h->f->part);
    std::memcpy(out, r.data(), r.size() * sizeof(double));
  })
}

// ---------------------------------------------------------------------------
// Bounded CPU-baseline samples (bench.py cpu_baseline / --impl reference).
// Times, for one strip of the given width, the reference's stage-one work:
// band fill + dgbtrf, and one dgbtrs with `nrhs_sample` identity columns
// (the dense-mode call of inc/stage_one.hpp:280 with n2 RHS, sampled).
int orc_time_slab_sample(const orc_system* s, long b, long strip, long nrhs_sample,
                         double* t_trf, double* t_trs) {
  ORC_TRY({
    Partition p = partition(s->sys.n1, s->sys.n2, b);
    auto t0 = std::chrono::steady_clock::now();
    SlabFactor f = factor_one_interior(s->sys, p, strip);
    *t_trf = seconds_since(t0);
    const long m = f.rows(), n2 = p.n2;
    std::vector<double> x(n2 * nrhs_sample, 0.0), tmp(m * nrhs_sample);
    for (long c = 0; c < nrhs_sample; c++) x[c * n2 + c % n2] = 1.0;
    auto t1 = std::chrono::steady_clock::now();
    const Sparse& in_blk = f.right_ifc >= 0 ? f.from_right : f.from_left;
    sparse_apply(in_blk, false, x.data(), nrhs_sample, tmp.data());
    f.lu.solve(tmp.data(), nrhs_sample, false);
    *t_trs = seconds_since(t1);
  })
}
// Times one stage-two sweep step at block size m (dgetrs with m RHS + dgemm +
// dgetrf on random well-conditioned blocks), inc/stage_two.hpp:135-147.
int orc_time_sweep_step(long m, double* t_step) {
  ORC_TRY({
    std::mt19937_64 rng(7);
    std::normal_distribution<double> g(0.0, 1.0);
    DenseLU prev;
    prev.n = m;
    prev.lu.resize(m * m);
    std::vector<double> sup(m * m), sub(m * m), d(m * m);
    for (auto& v : prev.lu) v = g(rng);
    for (long i = 0; i < m; i++) prev.lu[i * m + i] += 4.0 * std::sqrt((double)m);
    for (auto& v : sup) v = g(rng);
    for (auto& v : sub) v = g(rng);
    for (auto& v : d) v = g(rng);
    for (long i = 0; i < m; i++) d[i * m + i] += 4.0 * std::sqrt((double)m);
    prev.factor();
    auto t0 = std::chrono::steady_clock::now();
    std::vector<double> x = sup;
    prev.solve(x.data(), m, m);
    gemm(m, m, m, -1.0, sub.data(), m, x.data(), m, 1.0, d.data(), m);
    DenseLU cur;
    cur.n = m;
    cur.lu = std::move(d);
    cur.factor();
    *t_step = seconds_since(t0);
  })
}

// gaussian_matrix (inc/common.hpp:72-79): mt19937_64 + normal_distribution.
void orc_gaussian_matrix(long rows, long cols, uint64_t seed, double* out) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  for (long j = 0; j < cols; j++)
    for (long i = 0; i < rows; i++) out[j * rows + i] = gauss(rng);
}

// ---------------------------------------------------------------------------
// Per-slab staged checks (test infrastructure): one slab interior factored on
// its own (factor_one_interior, inc/stage_one.hpp:163-238), then the three
// per-slab terms of the reference's stage one / solve, so that parity can be
// checked at sizes where the whole oracle factorization does not fit:
//   contrib  : to_left/to_right . A_ii^{-1} permute_in(f_i)   (reduce_rhs :423-432)
//   T columns: to_X . A_ii^{-1} from_Y[:, cols]                (apply_T_block :276-283)
//   recover  : A_ii^{-1}(f_i - from_L u_L - from_R u_R)        (recover_interiors :447-459)
struct orc_slab {
  SlabFactor f;
  long N = 0, K = 0;
};
int orc_slab_factor(const orc_system* s, long b, long strip, orc_slab** out) {
  ORC_TRY({
    Partition p = partition(s->sys.n1, s->sys.n2, b);
    if (strip < 0 || strip >= p.nint()) fail(ERR_GENERIC, "slab_factor: strip out of range");
    auto* h = new orc_slab;
    try {
      h->f = factor_one_interior(s->sys, p, strip);
    } catch (...) {
      delete h;
      throw;
    }
    h->N = p.dim();
    h->K = p.nifc() * p.n2;
    *out = h;
  })
}
void orc_slab_free(orc_slab* h) { delete h; }
// [first_col, width, left_ifc, right_ifc]
void orc_slab_info(const orc_slab* h, long* info) {
  info[0] = h->f.first_col;
  info[1] = h->f.width;
  info[2] = h->f.left_ifc;
  info[3] = h->f.right_ifc;
}
// f: N x nrhs (ld N) natural order; outL/outR: n2 x nrhs (zero for an absent side)
int orc_slab_contrib(const orc_slab* h, const double* f, long nrhs, double* outL, double* outR) {
  ORC_TRY({
    const SlabFactor& fc = h->f;
    const long m = fc.rows(), n2 = fc.n2;
    std::vector<double> g(m * nrhs);
    fc.permute_in(f + fc.first_col * n2, h->N, nrhs, g.data());
    fc.lu.solve(g.data(), nrhs, false);
    std::fill(outL, outL + n2 * nrhs, 0.0);
    std::fill(outR, outR + n2 * nrhs, 0.0);
    if (fc.left_ifc >= 0) sparse_apply(fc.to_left, false, g.data(), nrhs, outL);
    if (fc.right_ifc >= 0) sparse_apply(fc.to_right, false, g.data(), nrhs, outR);
  })
}
// side: 0 from_left, 1 from_right; cols: ncol interface row indices (identity columns);
// outL/outR: n2 x ncol = to_left / to_right . A_ii^{-1} from_side[:, cols]
int orc_slab_T_columns(const orc_slab* h, int side, const long* cols, long ncol, double* outL, double* outR) {
  ORC_TRY({
    const SlabFactor& fc = h->f;
    const long m = fc.rows(), n2 = fc.n2;
    const Sparse& in_blk = side == 0 ? fc.from_left : fc.from_right;
    if ((side == 0 ? fc.left_ifc : fc.right_ifc) < 0) fail(ERR_GENERIC, "slab_T_columns: no interface on that side");
    std::vector<double> x(n2 * ncol, 0.0), tmp(m * ncol);
    for (long c = 0; c < ncol; c++) x[c * n2 + cols[c]] = 1.0;
    sparse_apply(in_blk, false, x.data(), ncol, tmp.data());
    fc.lu.solve(tmp.data(), ncol, false);
    std::fill(outL, outL + n2 * ncol, 0.0);
    std::fill(outR, outR + n2 * ncol, 0.0);
    if (fc.left_ifc >= 0) sparse_apply(fc.to_left, false, tmp.data(), ncol, outL);
    if (fc.right_ifc >= 0) sparse_apply(fc.to_right, false, tmp.data(), ncol, outR);
  })
}
// u_ifc: K x nrhs (ld K); out: (width*n2) x nrhs in natural order (ix*n2 + iy)
int orc_slab_recover(const orc_slab* h, const double* f, const double* u_ifc, long nrhs, double* out) {
  ORC_TRY({
    const SlabFactor& fc = h->f;
    const long m = fc.rows(), n2 = fc.n2;
    std::vector<double> rhs(m * nrhs), tmp(m * nrhs), ui(n2 * nrhs);
    fc.permute_in(f + fc.first_col * n2, h->N, nrhs, rhs.data());
    auto sub_coupling = [&](const Sparse& sp, long ifc) {
      for (long c = 0; c < nrhs; c++) std::memcpy(&ui[c * n2], u_ifc + c * h->K + ifc * n2, n2 * sizeof(double));
      sparse_apply(sp, false, ui.data(), nrhs, tmp.data());
      for (long i = 0; i < m * nrhs; i++) rhs[i] -= tmp[i];
    };
    if (fc.left_ifc >= 0) sub_coupling(fc.from_left, fc.left_ifc);
    if (fc.right_ifc >= 0) sub_coupling(fc.from_right, fc.right_ifc);
    fc.lu.solve(rhs.data(), nrhs, false);
    fc.permute_out(rhs.data(), nrhs, out, m);
  })
}

}  // extern "C"
