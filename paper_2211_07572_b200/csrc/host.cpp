// Host-side geometry and problem assembly for the SlabLU B200 engine.
// Integer maps (choose_b, partition) are bit-exact restatements of the
// reference; assembly evaluates the same formulas in the same order so the
// CSR it produces is bitwise identical to the reference's (compiled with
// -ffp-contract=off, as the oracle is).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>

#include "../../include/slablu_gpu.h"
#include "host.h"

namespace slb {

slablu_gpu_status make_status(int code, const std::string& msg, int64_t index, double residual) {
  slablu_gpu_status s;
  s.code = code;
  s.index = index;
  s.residual = residual;
  std::snprintf(s.msg, sizeof(s.msg), "%s", msg.c_str());
  return s;
}

// choose_b — proj/include/slablu/driver.hpp:55-66
int64_t choose_b(int64_t n1, int64_t n2, int64_t b, double c) {
  if (b > 0) return b;
  if (n2 < 8) throw HostError(SLABLU_ERR_CONFIG, "choose_b: n2 must be at least 8");
  if (!(c > 0.0) || c > 2.0) throw HostError(SLABLU_ERR_CONFIG, "choose_b: coefficient c must lie in (0, 2]");
  const double raw = c * std::pow(double(n2), 2.0 / 3.0);
  const int64_t rounded = 10 * static_cast<int64_t>(std::llround(raw / 10.0));
  const int64_t hi = std::max<int64_t>(1, n1 / 2);
  return std::clamp(rounded, std::min<int64_t>(10, hi), hi);
}

// partition — proj/include/slablu/partition.hpp:70-91
Partition partition(int64_t n1, int64_t n2, int64_t b) {
  if (n2 < 1) throw HostError(SLABLU_ERR_CONFIG, "partition: n2 must be positive");
  if (b < 1 || b > n1 - 2)
    throw HostError(SLABLU_ERR_CONFIG, "partition: slab width must satisfy 1 <= b <= n1 - 2");
  Partition p;
  p.n1 = n1;
  p.n2 = n2;
  p.b = b;
  int64_t col = 0;
  for (int64_t t = 1; col < n1; t++) {
    const int64_t ifc = t * (b + 1) - 1;
    const int64_t stop = std::min(ifc, n1);
    if (stop > col) p.interiors.push_back({col, stop - col});
    col = stop;
    if (col == ifc && col < n1) {
      p.interfaces.push_back({col, 1});
      col++;
    }
  }
  return p;
}

// bessel_j0 — proj/include/slablu/bessel.hpp:28-50
double bessel_j0(double t) {
  if (!std::isfinite(t)) throw HostError(SLABLU_ERR_GENERIC, "bessel_j0: argument must be finite");
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

namespace {

// Reference solutions — proj/include/slablu/problem.hpp:136-149
double poisson_solution(double x, double y) {
  const double r = std::hypot(x + 0.1, y - 0.5);
  if (r == 0.0) throw HostError(SLABLU_ERR_GENERIC, "true_solution_poisson: evaluated at the source point");
  return std::log(r);
}
double helmholtz_solution(double x, double y, double kappa) {
  return bessel_j0(kappa * std::hypot(x + 0.1, y - 0.5));
}

struct Canned {
  int kind;
  int64_t n1, n2;
  double kappa;
};
double canned_coef(double x, double y, void* u) {
  const Canned* c = static_cast<const Canned*>(u);
  if (c->kind != 2) return 1.0;
  // helmholtz_bump_problem coefficient — problem.hpp:245-251
  const double h = 1.0 / double(c->n2 + 1);
  const double cx = 0.5 * double(c->n1 + 1) * h, cy = 0.5;
  const double d2 = (x - cx) * (x - cx) + (y - cy) * (y - cy);
  return 1.0 - 0.9 * std::exp(-64.0 * d2);
}
double canned_dir(double x, double y, void* u) {
  const Canned* c = static_cast<const Canned*>(u);
  return c->kind == 0 ? poisson_solution(x, y) : helmholtz_solution(x, y, c->kappa);
}
double zero_field(double, double, void*) { return 0.0; }
double one_field(double, double, void*) { return 1.0; }

}  // namespace

// assemble_fd5 — proj/include/slablu/problem.hpp:78-132.  Columns within a
// row come out sorted (Eigen's compressed RowMajor order).
int64_t assemble_fd5(int64_t n1, int64_t n2, double h, double kappa, slablu_field_fn coef,
                     slablu_field_fn dir, slablu_field_fn load, void* user, int32_t* rp, int32_t* ci,
                     double* val, double* rhs) {
  if (n2 < 2 || n1 < n2) throw HostError(SLABLU_ERR_CONFIG, "assemble_fd5: grid must satisfy n1 >= n2 >= 2");
  if (!(h > 0.0)) throw HostError(SLABLU_ERR_CONFIG, "assemble_fd5: h must be positive");
  if (kappa < 0.0) throw HostError(SLABLU_ERR_CONFIG, "assemble_fd5: kappa must be nonnegative");
  if (n1 * n2 * 5 >= (int64_t)INT32_MAX)
    throw HostError(SLABLU_ERR_UNSUPPORTED, "assemble_fd5: nnz exceeds the int32 CSR index range");
  if (!coef) coef = one_field;
  if (!dir) dir = zero_field;
  if (!load) load = zero_field;
  const double inv_h2 = 1.0 / (h * h);
  int64_t nnz = 0;
  rp[0] = 0;
  for (int64_t i = 0; i < n1; i++) {
    for (int64_t j = 0; j < n2; j++) {
      const int64_t row = i * n2 + j;
      const double x = double(i + 1) * h;
      const double y = double(j + 1) * h;
      const double b = coef(x, y, user);
      if (b < 0.0) throw HostError(SLABLU_ERR_GENERIC, "assemble_fd5: coefficient field is negative at a node");
      const double diag = 4.0 * inv_h2 - kappa * kappa * b;
      double r = load(x, y, user);
      // neighbour order W, E, S, N (problem.hpp:114-125) for the Dirichlet fold
      const int64_t di[4] = {-1, 1, 0, 0};
      const int64_t dj[4] = {0, 0, -1, 1};
      bool inside[4];
      for (int s = 0; s < 4; s++) {
        const int64_t ii = i + di[s], jj = j + dj[s];
        inside[s] = ii >= 0 && ii < n1 && jj >= 0 && jj < n2;
        if (!inside[s]) r += dir(double(ii + 1) * h, double(jj + 1) * h, user) * inv_h2;
      }
      rhs[row] = r;
      // sorted columns: W (row-n2), S (row-1), diag, N (row+1), E (row+n2)
      if (inside[0]) { ci[nnz] = (int32_t)(row - n2); val[nnz++] = -inv_h2; }
      if (inside[2]) { ci[nnz] = (int32_t)(row - 1); val[nnz++] = -inv_h2; }
      ci[nnz] = (int32_t)row; val[nnz++] = diag;
      if (inside[3]) { ci[nnz] = (int32_t)(row + 1); val[nnz++] = -inv_h2; }
      if (inside[1]) { ci[nnz] = (int32_t)(row + n2); val[nnz++] = -inv_h2; }
      rp[row + 1] = (int32_t)nnz;
    }
  }
  return nnz;
}

int64_t assemble_canned(int kind, int64_t n1, int64_t n2, double kappa, int32_t* rp, int32_t* ci,
                        double* val, double* rhs) {
  if (kind < 0 || kind > 2) throw HostError(SLABLU_ERR_CONFIG, "assemble_canned: unknown problem kind");
  Canned c{kind, n1, n2, kind == 0 ? 0.0 : kappa};
  if (kind != 0 && kappa < 0.0) throw HostError(SLABLU_ERR_CONFIG, "assemble_fd5: kappa must be nonnegative");
  const double h = 1.0 / double(n2 + 1);
  return assemble_fd5(n1, n2, h, c.kappa, canned_coef, canned_dir, zero_field, &c, rp, ci, val, rhs);
}

void sample_solution(int kind, int64_t n1, int64_t n2, double kappa, double* out) {
  const double h = 1.0 / double(n2 + 1);
  for (int64_t i = 0; i < n1; i++)
    for (int64_t j = 0; j < n2; j++) {
      const double x = double(i + 1) * h, y = double(j + 1) * h;
      out[i * n2 + j] = kind == 0 ? poisson_solution(x, y) : helmholtz_solution(x, y, kappa);
    }
}

}  // namespace slb

using namespace slb;

extern "C" {

slablu_gpu_status slablu_gpu_assemble_fd5(int64_t n1, int64_t n2, double h, double kappa,
                                          slablu_field_fn coefficient, slablu_field_fn dirichlet,
                                          slablu_field_fn load, void* user, int32_t* row_ptr,
                                          int32_t* col_idx, double* val, double* rhs, int64_t* nnz) {
  try {
    *nnz = assemble_fd5(n1, n2, h, kappa, coefficient, dirichlet, load, user, row_ptr, col_idx, val, rhs);
    return make_status(SLABLU_OK, "", -1);
  } catch (const HostError& e) {
    return make_status(e.code, e.what(), e.index);
  }
}

slablu_gpu_status slablu_gpu_assemble_canned(int kind, int64_t n1, int64_t n2, double kappa,
                                             int32_t* row_ptr, int32_t* col_idx, double* val,
                                             double* rhs, int64_t* nnz) {
  try {
    *nnz = assemble_canned(kind, n1, n2, kappa, row_ptr, col_idx, val, rhs);
    return make_status(SLABLU_OK, "", -1);
  } catch (const HostError& e) {
    return make_status(e.code, e.what(), e.index);
  }
}

slablu_gpu_status slablu_gpu_sample_solution(int kind, int64_t n1, int64_t n2, double kappa, double* out) {
  try {
    sample_solution(kind, n1, n2, kappa, out);
    return make_status(SLABLU_OK, "", -1);
  } catch (const HostError& e) {
    return make_status(e.code, e.what(), e.index);
  }
}

// kappa_from_ppw — proj/include/slablu/problem.hpp:153-157 (NaN on invalid input)
double slablu_gpu_kappa_from_ppw(double ppw, int64_t n2) {
  if (!(ppw > 0.0) || n2 < 2) return std::nan("");
  return 2.0 * 3.14159265358979323846 * double(n2 + 1) / ppw;
}

double slablu_gpu_bessel_j0(double t) {
  try {
    return bessel_j0(t);
  } catch (const HostError&) {
    return std::nan("");
  }
}

void slablu_gpu_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  for (int64_t j = 0; j < cols; j++)
    for (int64_t i = 0; i < rows; i++) out[j * rows + i] = gauss(rng);
}

slablu_gpu_status slablu_gpu_choose_b(int64_t n1, int64_t n2, int64_t b, double c, int64_t* out) {
  try {
    *out = choose_b(n1, n2, b, c);
    return make_status(SLABLU_OK, "", -1);
  } catch (const HostError& e) {
    return make_status(e.code, e.what(), e.index);
  }
}

slablu_gpu_status slablu_gpu_partition(int64_t n1, int64_t n2, int64_t b, int64_t* n_interiors,
                                       int64_t* interiors, int64_t* n_interfaces, int64_t* interfaces,
                                       int64_t cap) {
  try {
    Partition p = partition(n1, n2, b);
    *n_interiors = (int64_t)p.interiors.size();
    *n_interfaces = (int64_t)p.interfaces.size();
    for (int64_t i = 0; i < (int64_t)p.interiors.size() && i < cap; i++) {
      interiors[2 * i] = p.interiors[i].first_col;
      interiors[2 * i + 1] = p.interiors[i].width;
    }
    for (int64_t i = 0; i < (int64_t)p.interfaces.size() && i < cap; i++) {
      interfaces[2 * i] = p.interfaces[i].first_col;
      interfaces[2 * i + 1] = p.interfaces[i].width;
    }
    return make_status(SLABLU_OK, "", -1);
  } catch (const HostError& e) {
    return make_status(e.code, e.what(), e.index);
  }
}

}  // extern "C"
