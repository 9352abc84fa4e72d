// C++ caller of the drop-in API (include/slablu_b200.hpp), written like the
// reference's own tests (proj/tests/test_partition.cpp, test_problem.cpp,
// test_driver.cpp).  `test_mirror host` runs the host-only checks; `test_mirror
// gpu` additionally factorizes and solves on the B200 and checks the residual.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "slablu_b200.hpp"

namespace S = slablu_b200;
static int failures = 0;
#define CHECK(cond)                                                     \
  do {                                                                  \
    if (!(cond)) {                                                      \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      failures++;                                                       \
    }                                                                   \
  } while (0)

static void host_checks() {
  // partition geometries (proj/tests/test_partition.cpp:49-94)
  S::SlabPartition p = S::partition(7, 5, 3);
  CHECK(p.interior_count() == 2 && p.interface_count() == 1);
  CHECK(p.interfaces[0].first_col == 3 && p.interiors[1].first_col == 4);
  p = S::partition(1000, 1000, 50);
  CHECK(p.interface_count() == 19 && p.interior_count() == 20 && p.interiors.back().width == 31);
  p = S::partition(8, 3, 3);
  CHECK(p.interface_count() == 2 && p.interior_count() == 2 && p.right_interior(1) == -1);
  bool threw = false;
  try {
    S::partition(10, 4, 9);
  } catch (const S::ConfigError&) {
    threw = true;
  }
  CHECK(threw);
  // choose_b (proj/tests/test_driver.cpp:54-78)
  S::SolverConfig c;
  c.c = 0.5;
  CHECK(S::choose_b(4000, 1000, c) == 50);
  c.c = 0.54;
  CHECK(S::choose_b(40000, 10000, c) == 250);
  c.c = 0.6;
  CHECK(S::choose_b(24, 1000, c) == 12);
  // assembly with std::function fields (proj/tests/test_problem.cpp:66-108)
  S::ProblemSpec spec;
  spec.n1 = spec.n2 = 3;
  spec.h = 0.25;
  spec.dirichlet_data = [](double x, double y) { return x + y; };
  spec.body_load = [](double, double) { return 7.0; };
  S::SparseSystem sys = S::assemble_fd5(spec);
  CHECK(sys.rhs[0] == 15.0 && sys.rhs[4] == 7.0);
  CHECK(sys.row_ptr[9] == 33);
  double dmax = 0, omin = 0;
  for (double v : sys.values) {
    dmax = std::fmax(dmax, v);
    omin = std::fmin(omin, v);
  }
  CHECK(dmax == 64.0 && omin == -16.0);
  CHECK(std::fabs(S::bessel_j0(5.0) - (-0.17759677131433830435)) <= 1e-13);
}

static void gpu_checks() {
  // factorize + solve, consistent right-hand side (proj/tests/test_driver.cpp:110-122)
  const S::SparseSystem sys = S::assemble_fd5(S::helmholtz_bump_problem(64, 48, 30.0));
  S::SolverConfig cfg;
  cfg.b = 6;
  const S::Factorization fact = S::factorize(sys, cfg);
  CHECK(!fact.single_slab() && fact.b == 6 && fact.t_stage1 > 0.0);
  const int64_t n = sys.dim();
  std::vector<double> w(n), f(n, 0.0);
  for (int64_t i = 0; i < n; i++) w[i] = std::sin(0.37 * double(i)) + 0.1;
  for (int64_t r = 0; r < n; r++)
    for (int32_t q = sys.row_ptr[r]; q < sys.row_ptr[r + 1]; q++) f[r] += sys.values[q] * w[sys.col_idx[q]];
  const std::vector<double> u = S::solve(fact, f);
  double num = 0, den = 0;
  for (int64_t i = 0; i < n; i++) {
    num += (u[i] - w[i]) * (u[i] - w[i]);
    den += w[i] * w[i];
  }
  std::printf("mirror gpu: rel err vs generating vector %.3e\n", std::sqrt(num / den));
  CHECK(std::sqrt(num / den) < 1e-10);
  bool threw = false;
  try {
    S::solve(fact, std::vector<double>(7, 0.0));
  } catch (const S::Error&) {
    threw = true;
  }
  CHECK(threw);
}

static void hbs_checks() {
  // hbs_compress of a diagonal-plus-rank-5 operator (test_hbs.cpp:307-341) and the failure at
  // the rank ceiling (:343-359), through the C++ mirror
  const int64_t n = 96;
  std::vector<double> m((size_t)(n * n), 0.0);
  for (int64_t j = 0; j < n; j++)
    for (int64_t i = 0; i < n; i++) {
      double v = i == j ? 20.0 : 0.0;
      for (int k = 0; k < 5; k++) v += std::sin(0.3 * double(i + 1) * (k + 1)) * std::cos(0.7 * double(j + 2) * (k + 1));
      m[(size_t)(i + j * n)] = v;
    }
  S::CompressStats st;
  const std::vector<double> h = S::hbs_compress_adaptive(m, n, 12, 2, 64, S::CompressOptions{1e-10, 1e-12, 37}, &st);
  double num = 0, den = 0;
  for (size_t e = 0; e < m.size(); e++) {
    num += (h[e] - m[e]) * (h[e] - m[e]);
    den += m[e] * m[e];
  }
  CHECK(std::sqrt(num / den) <= 1e-10);
  CHECK(st.final_rank <= 10 && st.rounds <= 3);
  bool threw = false;
  try {
    S::hbs_compress(m, n, 12, 2, S::CompressOptions{1e-10, 1e-12, 43});
  } catch (const S::CompressionError& e) {
    threw = e.residual_estimate > 1e-10;
  }
  CHECK(threw);
}

int main(int argc, char** argv) {
  if (argc > 1 && std::strcmp(argv[1], "sizes") == 0) {  // struct layouts for the ctypes mirror
    std::printf("%zu %zu %zu %zu\n", sizeof(slablu_gpu_config), sizeof(slablu_gpu_status), sizeof(slablu_gpu_stats_t),
                sizeof(slablu_gpu_hbs_stats));
    return 0;
  }
  host_checks();
  if (argc > 1 && std::strcmp(argv[1], "gpu") == 0) {
    gpu_checks();
    hbs_checks();
  }
  std::printf("%s (%d failures)\n", failures ? "FAIL" : "OK", failures);
  return failures ? 1 : 0;
}
