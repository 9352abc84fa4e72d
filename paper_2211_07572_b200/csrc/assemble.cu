// On-device problem assembly and validation.
//
// assemble_fd5 (proj/include/slablu/problem.hpp:78-132) for the canned problems
// (:210-261), the manufactured solutions (:136-149, bessel.hpp:28-50) and
// error_report (:160-196), as kernels: the 5-point operator of a 4000^2 grid is
// assembled in HBM in a few milliseconds instead of seconds of host work plus a
// 1.2 GB host->device copy.
//
// Bit-exactness: the CSR index arrays (row_ptr, col_idx) equal assemble_fd5's.
// Matrix values use the same operation order (inv_h2 = 1/(h h), diag = 4 inv_h2
// - kappa^2 b(x), off = -inv_h2); they are bit-identical except where b(x)
// goes through exp (the bump coefficient: device exp vs the host libm, <= 1 ulp
// in b).  The Dirichlet fold (order W, E, S, N) evaluates log/hypot, and J0 in
// double where the reference's bessel_j0 sums in long double: boundary rhs
// entries agree to ~1e-15 relative (Poisson) and ~1e-12 (Helmholtz, J0 of
// arguments up to ~3e3).
#include <cmath>
#include <vector>

#include "common.cuh"
#include "host.h"
#include "kernels.h"

namespace slb {
namespace {

// bessel_j0 (bessel.hpp:28-50): power series for t <= 8, midpoint rule of
// (1/pi) int_0^pi cos(t sin theta) dtheta above (compensated summation)
__device__ double bessel_j0_dev(double t) {
  t = fabs(t);
  if (t <= 8.0) {
    const double q = t / 2.0;
    double sum = 1.0, term = 1.0, comp = 0.0;
    for (int m = 1; m <= 64; m++) {
      term *= -(q * q) / ((double)m * m);
      const double y = term - comp, s2 = sum + y;
      comp = (s2 - sum) - y;
      sum = s2;
      if (fabs(term) < 1e-20) break;
    }
    return sum;
  }
  const int n = (int)ceil(0.75 * t) + 30;
  const double pi = 3.14159265358979323846;
  double sum = 0.0, comp = 0.0;
  for (int k = 0; k < n; k++) {
    const double theta = pi * ((double)k + 0.5) / n;
    const double y = cos(t * sin(theta)) - comp, s2 = sum + y;
    comp = (s2 - sum) - y;
    sum = s2;
  }
  return sum / n;
}

__device__ double true_solution_dev(int kind, double x, double y, double kappa) {
  const double r = hypot(x + 0.1, y - 0.5);
  return kind == 0 ? log(r) : bessel_j0_dev(kappa * r);
}

// helmholtz_bump_problem coefficient (problem.hpp:245-251); 1 otherwise
__device__ double coef_dev(int kind, int64_t n1, double h, double x, double y) {
  if (kind != 2) return 1.0;
  const double cx = 0.5 * double(n1 + 1) * h, cy = 0.5;
  const double d2 = (x - cx) * (x - cx) + (y - cy) * (y - cy);
  return 1.0 - 0.9 * exp(-64.0 * d2);
}

// one thread per grid node (i, j), row i * n2 + j; row_ptr in closed form:
// rp[r] = 5 r - (neighbours missing before row r)
__global__ void assemble_kernel(int kind, int64_t n1, int64_t n2, double h, double kappa, int32_t* rp, int32_t* ci,
                                double* v, double* rhs, int* bad) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t N = n1 * n2;
  if (r >= N) return;
  const int64_t i = r / n2, j = r % n2;
  const double inv_h2 = 1.0 / (h * h);
  const double x = double(i + 1) * h, y = double(j + 1) * h;
  const double b = coef_dev(kind, n1, h, x, y);
  if (b < 0.0) atomicOr(bad, 1);
  const double diag = 4.0 * inv_h2 - kappa * kappa * b;
  double f = 0.0;  // canned problems carry no body load
  const int64_t di[4] = {-1, 1, 0, 0};
  const int64_t dj[4] = {0, 0, -1, 1};
  bool inside[4];
#pragma unroll
  for (int s = 0; s < 4; s++) {  // W, E, S, N (problem.hpp:114-125)
    const int64_t ii = i + di[s], jj = j + dj[s];
    inside[s] = ii >= 0 && ii < n1 && jj >= 0 && jj < n2;
    if (!inside[s]) f += true_solution_dev(kind, double(ii + 1) * h, double(jj + 1) * h, kappa) * inv_h2;
  }
  rhs[r] = f;
  const int64_t missing = 2 * i + (i > 0 ? n2 : 0) + (j > 0 ? 1 : 0) + (i == 0 ? j : 0) + (i == n1 - 1 ? j : 0);
  int64_t p = 5 * r - missing;
  rp[r] = (int32_t)p;
  if (r == N - 1) rp[N] = (int32_t)(5 * N - 2 * (n1 + n2));
  // sorted columns: W (row - n2), S (row - 1), diag, N (row + 1), E (row + n2)
  if (inside[0]) { ci[p] = (int32_t)(r - n2); v[p++] = -inv_h2; }
  if (inside[2]) { ci[p] = (int32_t)(r - 1); v[p++] = -inv_h2; }
  ci[p] = (int32_t)r; v[p++] = diag;
  if (inside[3]) { ci[p] = (int32_t)(r + 1); v[p++] = -inv_h2; }
  if (inside[1]) { ci[p] = (int32_t)(r + n2); v[p++] = -inv_h2; }
}

__global__ void sample_solution_kernel(int kind, int64_t n1, int64_t n2, double kappa, double* out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n1 * n2) return;
  const double h = 1.0 / double(n2 + 1);
  out[r] = true_solution_dev(kind, double(r / n2 + 1) * h, double(r % n2 + 1) * h, kappa);
}

// per-block partial sums of squares of (A u - f), f, (u - u_true), u_true over all columns
// (fixed block order: the final sum is deterministic)
constexpr int ER_THREADS = 256;
__global__ void __launch_bounds__(ER_THREADS) error_partial_kernel(int64_t n, int64_t nrhs, const int32_t* rp,
                                                                   const int32_t* ci, const double* v,
                                                                   const double* f, const double* u,
                                                                   const double* ut, double* part) {
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t idx = (int64_t)blockIdx.x * ER_THREADS + threadIdx.x; idx < n * nrhs;
       idx += (int64_t)gridDim.x * ER_THREADS) {
    const int64_t row = idx % n, c = idx / n;
    const double* uc = u + c * n;
    double au = 0.0;
    for (int32_t q = rp[row]; q < rp[row + 1]; q++) au = fma(v[q], uc[ci[q]], au);
    const double res = au - f[idx];
    s[0] = fma(res, res, s[0]);
    s[1] = fma(f[idx], f[idx], s[1]);
    if (ut) {
      const double e = u[idx] - ut[idx];
      s[2] = fma(e, e, s[2]);
      s[3] = fma(ut[idx], ut[idx], s[3]);
    }
  }
  __shared__ double red[4][ER_THREADS];
#pragma unroll
  for (int k = 0; k < 4; k++) red[k][threadIdx.x] = s[k];
  __syncthreads();
  for (int w = ER_THREADS / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w)
#pragma unroll
      for (int k = 0; k < 4; k++) red[k][threadIdx.x] += red[k][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x < 4) part[blockIdx.x * 4 + threadIdx.x] = red[threadIdx.x][0];
}

}  // namespace
}  // namespace slb

using namespace slb;

namespace {
struct DevScope {  // current device for the call, restored afterwards
  int prev = -1;
  explicit DevScope(int d) {
    if (cudaGetDevice(&prev) != cudaSuccess) {
      cudaGetLastError();
      prev = -1;
    }
    SLB_CUDA_CHECK(cudaSetDevice(d));
  }
  ~DevScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
slablu_gpu_status cuda_status(const CudaFailure& e) {
  return make_status(e.err == cudaErrorMemoryAllocation ? SLABLU_ERR_OOM : SLABLU_ERR_CUDA,
                     std::string("CUDA error: ") + cudaGetErrorString(e.err) + " at " + e.file + ":" +
                         std::to_string(e.line) + " (" + e.expr + ")",
                     -1);
}
void need_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw HostError(SLABLU_ERR_CUDA, "no CUDA device available (the engine has no CPU fallback)");
  }
}

void error_report_impl(int64_t n, const int32_t* rp, const int32_t* ci, const double* v, const double* f,
                       const double* u, const double* ut, int64_t nrhs, double* out) {
  const int blocks = (int)std::min<int64_t>(cdiv(n * nrhs, ER_THREADS), 2048);
  double* part = nullptr;
  SLB_CUDA_CHECK(cudaMalloc(&part, (size_t)blocks * 4 * sizeof(double)));
  error_partial_kernel<<<blocks, ER_THREADS>>>(n, nrhs, rp, ci, v, f, u, ut, part); count_launch();
  cudaError_t e = cudaGetLastError();
  std::vector<double> h((size_t)blocks * 4);
  if (e == cudaSuccess) e = cudaMemcpy(h.data(), part, h.size() * sizeof(double), cudaMemcpyDeviceToHost);
  cudaFree(part);
  if (e != cudaSuccess) throw CudaFailure(e, "error_partial_kernel", __FILE__, __LINE__);
  double s[4] = {0, 0, 0, 0};
  for (int b = 0; b < blocks; b++)
    for (int k = 0; k < 4; k++) s[k] += h[(size_t)b * 4 + k];
  // problem.hpp:177-188: relative unless the reference norm vanishes
  const double res = std::sqrt(s[0]), fn = std::sqrt(s[1]), err = std::sqrt(s[2]), un = std::sqrt(s[3]);
  out[0] = fn > 0.0 ? res / fn : res;
  out[1] = ut ? (un > 0.0 ? err / un : err) : std::nan("");
  out[2] = fn > 0.0 ? 0.0 : 1.0;  // residual_norm_is_absolute
  out[3] = ut && un > 0.0 ? 0.0 : 1.0;  // solution_norm_is_absolute
}
}  // namespace

extern "C" {

slablu_gpu_status slablu_gpu_assemble_canned_device(int kind, int64_t n1, int64_t n2, double kappa, int device,
                                                    int32_t* d_rp, int32_t* d_ci, double* d_v, double* d_rhs,
                                                    int64_t* nnz) {
  try {
    need_device();
    if (kind < 0 || kind > 2) throw HostError(SLABLU_ERR_CONFIG, "assemble_canned: unknown problem kind");
    if (n2 < 2 || n1 < n2) throw HostError(SLABLU_ERR_CONFIG, "assemble_fd5: grid must satisfy n1 >= n2 >= 2");
    if (kind != 0 && kappa < 0.0) throw HostError(SLABLU_ERR_CONFIG, "assemble_fd5: kappa must be nonnegative");
    if (n1 * n2 * 5 >= (int64_t)INT32_MAX)
      throw HostError(SLABLU_ERR_UNSUPPORTED, "assemble_fd5: nnz exceeds the int32 CSR index range");
    DevScope ds(device);
    const int64_t N = n1 * n2;
    const double h = 1.0 / double(n2 + 1);
    int* bad = nullptr;
    SLB_CUDA_CHECK(cudaMalloc(&bad, sizeof(int)));
    SLB_CUDA_CHECK(cudaMemset(bad, 0, sizeof(int)));
    assemble_kernel<<<(unsigned)cdiv(N, 256), 256>>>(kind, n1, n2, h, kind == 0 ? 0.0 : kappa, d_rp, d_ci, d_v, d_rhs,
                                                      bad); count_launch();
    cudaError_t e = cudaGetLastError();
    int hb = 0;
    if (e == cudaSuccess) e = cudaMemcpy(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost);
    cudaFree(bad);
    if (e != cudaSuccess) throw CudaFailure(e, "assemble_kernel", __FILE__, __LINE__);
    if (hb) throw HostError(SLABLU_ERR_GENERIC, "assemble_fd5: coefficient field is negative at a node");
    *nnz = 5 * N - 2 * (n1 + n2);
    return make_status(SLABLU_OK, "", -1);
  } catch (const HostError& e) {
    return make_status(e.code, e.what(), e.index);
  } catch (const CudaFailure& e) {
    return cuda_status(e);
  }
}

slablu_gpu_status slablu_gpu_sample_solution_device(int kind, int64_t n1, int64_t n2, double kappa, int device,
                                                    double* d_out) {
  try {
    need_device();
    if (kind < 0 || kind > 2) throw HostError(SLABLU_ERR_CONFIG, "sample_solution: unknown problem kind");
    DevScope ds(device);
    sample_solution_kernel<<<(unsigned)cdiv(n1 * n2, 256), 256>>>(kind, n1, n2, kind == 0 ? 0.0 : kappa, d_out);
    count_launch();
    SLB_CUDA_CHECK(cudaGetLastError());
    SLB_CUDA_CHECK(cudaDeviceSynchronize());
    return make_status(SLABLU_OK, "", -1);
  } catch (const HostError& e) {
    return make_status(e.code, e.what(), e.index);
  } catch (const CudaFailure& e) {
    return cuda_status(e);
  }
}

slablu_gpu_status slablu_gpu_error_report_device(int64_t n, const int32_t* d_rp, const int32_t* d_ci,
                                                 const double* d_v, const double* d_f, const double* d_u,
                                                 const double* d_utrue, int64_t nrhs, int device, double* out) {
  try {
    need_device();
    if (n < 1 || nrhs < 1) throw HostError(SLABLU_ERR_GENERIC, "error_report: column counts must agree");
    DevScope ds(device);
    error_report_impl(n, d_rp, d_ci, d_v, d_f, d_u, d_utrue, nrhs, out);
    return make_status(SLABLU_OK, "", -1);
  } catch (const HostError& e) {
    return make_status(e.code, e.what(), e.index);
  } catch (const CudaFailure& e) {
    return cuda_status(e);
  }
}

slablu_gpu_status slablu_gpu_error_report(int64_t n, const int32_t* rp, const int32_t* ci, const double* v,
                                          const double* f, const double* u, const double* utrue, int64_t nrhs,
                                          int device, double* out) {
  try {
    need_device();
    if (n < 1 || nrhs < 1) throw HostError(SLABLU_ERR_GENERIC, "error_report: column counts must agree");
    DevScope ds(device);
    const int64_t nnz = rp[n];
    void* buf[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    const size_t sz[7] = {(size_t)(n + 1) * 4, (size_t)nnz * 4, (size_t)nnz * 8, (size_t)(n * nrhs) * 8,
                          (size_t)(n * nrhs) * 8, utrue ? (size_t)(n * nrhs) * 8 : 0, 0};
    const void* src[6] = {rp, ci, v, f, u, utrue};
    cudaError_t e = cudaSuccess;
    for (int k = 0; k < 6 && e == cudaSuccess; k++)
      if (sz[k]) {
        e = cudaMalloc(&buf[k], sz[k]);
        if (e == cudaSuccess) e = cudaMemcpy(buf[k], src[k], sz[k], cudaMemcpyHostToDevice);
      }
    if (e == cudaSuccess) {
      try {
        error_report_impl(n, (const int32_t*)buf[0], (const int32_t*)buf[1], (const double*)buf[2],
                          (const double*)buf[3], (const double*)buf[4], (const double*)buf[5], nrhs, out);
      } catch (...) {
        for (void* p : buf) cudaFree(p);
        throw;
      }
    }
    for (void* p : buf) cudaFree(p);
    if (e != cudaSuccess) throw CudaFailure(e, "error_report copies", __FILE__, __LINE__);
    return make_status(SLABLU_OK, "", -1);
  } catch (const HostError& e) {
    return make_status(e.code, e.what(), e.index);
  } catch (const CudaFailure& e) {
    return cuda_status(e);
  }
}

}  // extern "C"
