// Stage two building blocks: dense LU with partial pivoting, triangular
// solves and the explicit inverse of the sweep Schur blocks (sm_100a).
//
// Reference: DenseLU = LAPACKE_dgetrf / dgetrs (proj/include/slablu/dense.hpp:
// 31-61), used by SweepFactorization (stage_two.hpp:131-150, 170-188).
//
// getrf: recursive (Toledo) LU; the leaves are 32-column panels factored by
// one thread-block cluster (up to 16 CTAs, one panel row per thread held in
// registers, pivot search reduced through distributed shared memory).  All
// bulk work is DMMA GEMM (gemm.cu) with large K from the recursion.
// trsm: recursive, 64-row leaves solved per right-hand-side column.
#include <climits>
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace slb {
namespace {

constexpr int PNB = 32;          // panel width
constexpr int PTHREADS = 256;    // rows per CTA of the panel cluster (<= 16 CTAs)

// Factor rows [j, n) x cols [j, j + nb) of A in place.  Thread (rank, tid)
// owns panel row i = rank * 512 + tid.  ipiv[j + k] = global pivot row.
__global__ void __launch_bounds__(PTHREADS) panel_getrf_kernel(double* A, int64_t lda, int64_t n,
                                                               int64_t j, int nb, int32_t* ipiv,
                                                               DevStatus* status, int block_index) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int ncta = (int)cluster.num_blocks();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t m = n - j;
  const int64_t i = (int64_t)rank * PTHREADS + tid;
  const bool own = i < m;
  __shared__ double s_wv[PTHREADS / 32];
  __shared__ int s_wi[PTHREADS / 32];
  __shared__ double s_cv;      // CTA candidate |value|
  __shared__ int s_ci;         // CTA candidate row
  __shared__ double s_rowP[PNB];
  __shared__ double s_rowK[PNB];
  __shared__ double s_prow[PNB];
  __shared__ double s_krow[PNB];
  __shared__ int s_piv;

  double r[PNB];
#pragma unroll
  for (int c = 0; c < PNB; c++) r[c] = (own && c < nb) ? A[(j + c) * lda + j + i] : 0.0;

  for (int k = 0; k < nb; k++) {
    // (1) local argmax over rows i >= k (first max by row index)
    double v = -1.0;
    int vi = INT_MAX;
    if (own && i >= k) {
      double x = 0.0;
#pragma unroll
      for (int c = 0; c < PNB; c++)
        if (c == k) x = r[c];
      v = fabs(x);
      vi = (int)i;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int oi = __shfl_xor_sync(0xffffffffu, vi, o);
      if (ov > v || (ov == v && oi < vi)) {
        v = ov;
        vi = oi;
      }
    }
    if (lane == 0) {
      s_wv[warp] = v;
      s_wi[warp] = vi;
    }
    __syncthreads();
    if (warp == 0) {
      v = lane < PTHREADS / 32 ? s_wv[lane] : -1.0;
      vi = lane < PTHREADS / 32 ? s_wi[lane] : INT_MAX;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, vi, o);
        if (ov > v || (ov == v && oi < vi)) {
          v = ov;
          vi = oi;
        }
      }
      if (lane == 0) {
        s_cv = v;
        s_ci = vi;
      }
    }
    cluster.sync();
    // (2) cluster-wide pivot (every CTA computes the same answer); candidates read in parallel
    if (warp == 0) {
      double bv = -1.0;
      int bi = INT_MAX;
      if (lane < ncta) {
        bv = *cluster.map_shared_rank(&s_cv, lane);
        bi = *cluster.map_shared_rank(&s_ci, lane);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (lane == 0) {
        if (!(bv > 0.0)) {
          bi = k;
          if (rank == 0) {
            atomicOr(&status->flags, ERR_SINGULAR);
            atomicMin(&status->singular_block, block_index);
          }
        }
        s_piv = bi;
        if (rank == 0) ipiv[j + k] = (int32_t)(j + bi);
      }
    }
    __syncthreads();
    const int p = s_piv;
    // (3) owners publish rows p and k
    if (own && i == p)
#pragma unroll
      for (int c = 0; c < PNB; c++) s_rowP[c] = r[c];
    if (own && i == k)
#pragma unroll
      for (int c = 0; c < PNB; c++) s_rowK[c] = r[c];
    cluster.sync();
    // (4) local copies of both rows (parallel DSMEM reads), then swap
    if (tid < PNB) s_prow[tid] = *cluster.map_shared_rank(&s_rowP[tid], p / PTHREADS);
    else if (tid < 2 * PNB) s_krow[tid - PNB] = *cluster.map_shared_rank(&s_rowK[tid - PNB], k / PTHREADS);
    __syncthreads();
    if (p != k) {
      if (own && i == k) {
#pragma unroll
        for (int c = 0; c < PNB; c++) r[c] = s_prow[c];
      } else if (own && i == p) {
#pragma unroll
        for (int c = 0; c < PNB; c++) r[c] = s_krow[c];
      }
    }
    // (5) scale + rank-1 update of rows below k
    if (own && i > k) {
      const double pv = s_prow[k];
      const double inv = pv != 0.0 ? 1.0 / pv : 0.0;
      double l = 0.0;
#pragma unroll
      for (int c = 0; c < PNB; c++)
        if (c == k) l = r[c] * inv;
#pragma unroll
      for (int c = 0; c < PNB; c++) {
        if (c == k) r[c] = l;
        else if (c > k) r[c] = fma(-l, s_prow[c], r[c]);
      }
    }
  }
  cluster.sync();
  if (own)
#pragma unroll
    for (int c = 0; c < PNB; c++)
      if (c < nb) A[(j + c) * lda + j + i] = r[c];
}

// Row swaps ipiv[k1..k2) applied (in order) to columns [c0, c1).
__global__ void laswp_kernel(double* A, int64_t lda, int64_t c0, int64_t c1, const int32_t* ipiv,
                             int64_t k1, int64_t k2) {
  const int64_t c = c0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= c1) return;
  double* col = A + c * lda;
  for (int64_t k = k1; k < k2; k++) {
    const int64_t p = ipiv[k];
    if (p != k) {
      const double t = col[k];
      col[k] = col[p];
      col[p] = t;
    }
  }
}

__global__ void finite_kernel(const double* a, int64_t count, DevStatus* status) {
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(a[i])) bad = true;
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&status->flags, ERR_NONFINITE);
}

__global__ void identity_kernel(double* a, int64_t n) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n * n;
       idx += (int64_t)gridDim.x * blockDim.x)
    a[idx] = (idx % n == idx / n) ? 1.0 : 0.0;
}

void panel(cudaStream_t st, double* A, int64_t lda, int64_t n, int64_t j, int nb, int32_t* ipiv,
           DevStatus* status, int block_index) {
  const int64_t m = n - j;
  const int ncta = (int)cdiv(m, PTHREADS);
  if (ncta > 16)
    throw CudaFailure(cudaErrorInvalidValue, "dgetrf: block dimension > 4096 unsupported", __FILE__, __LINE__);
  static bool attr = false;
  if (!attr) {
    SLB_CUDA_CHECK(cudaFuncSetAttribute(panel_getrf_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ncta);
  cfg.blockDim = dim3(PTHREADS);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = ncta;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  SLB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, panel_getrf_kernel, A, lda, n, j, nb, ipiv, status, block_index));
}

void laswp(cudaStream_t st, double* A, int64_t lda, int64_t c0, int64_t c1, const int32_t* ipiv,
           int64_t k1, int64_t k2) {
  if (c1 <= c0 || k2 <= k1) return;
  laswp_kernel<<<(unsigned)cdiv(c1 - c0, 128), 128, 0, st>>>(A, lda, c0, c1, ipiv, k1, k2);
  SLB_CUDA_CHECK(cudaGetLastError());
}

// X = L^{-1} B (unit lower) or U^{-1} B (upper), L is m x m.
void trsm(cudaStream_t st, bool lower, const double* L, int64_t ldl, int64_t m, double* B, int64_t ldb,
          int64_t ncols) {
  if (m <= 0 || ncols <= 0) return;
  if (m <= 128) {
    trsm_small_batched(st, lower, (int)m, L, ldl, 0, B, ldb, 0, ncols, 1, /*rowmajor=*/false);
    return;
  }
  const int64_t h = round_up(m / 2, 64) < m ? round_up(m / 2, 64) : m / 2;
  const double* L11 = L;
  const double* L21 = L + h;              // rows h.., cols 0..h
  const double* L12 = L + h * ldl;        // rows 0..h, cols h..
  const double* L22 = L + h * ldl + h;
  if (lower) {
    trsm(st, true, L11, ldl, h, B, ldb, ncols);
    dgemm_batched(st, m - h, ncols, h, -1.0, L21, ldl, 0, B, ldb, 0, 1.0, B + h, ldb, 0, 1);
    trsm(st, true, L22, ldl, m - h, B + h, ldb, ncols);
  } else {
    trsm(st, false, L22, ldl, m - h, B + h, ldb, ncols);
    dgemm_batched(st, h, ncols, m - h, -1.0, L12, ldl, 0, B + h, ldb, 0, 1.0, B, ldb, 0, 1);
    trsm(st, false, L11, ldl, h, B, ldb, ncols);
  }
}

// Recursive LU of columns [c0, c1) (rows c0..n) of the n x n matrix A.
void getrf_rec(cudaStream_t st, double* A, int64_t n, int64_t c0, int64_t c1, int32_t* ipiv,
               DevStatus* status, int block_index) {
  const int64_t w = c1 - c0;
  if (w <= PNB) {
    panel(st, A, n, n, c0, (int)w, ipiv, status, block_index);
    return;
  }
  int64_t h = round_up(w / 2, PNB);
  if (h >= w) h = w - PNB;
  getrf_rec(st, A, n, c0, c0 + h, ipiv, status, block_index);
  laswp(st, A, n, c0 + h, c1, ipiv, c0, c0 + h);
  trsm(st, true, A + c0 * n + c0, n, h, A + (c0 + h) * n + c0, n, w - h);
  dgemm_batched(st, n - c0 - h, w - h, h, -1.0, A + c0 * n + c0 + h, n, 0, A + (c0 + h) * n + c0, n, 0, 1.0,
                A + (c0 + h) * n + c0 + h, n, 0, 1);
  getrf_rec(st, A, n, c0 + h, c1, ipiv, status, block_index);
  laswp(st, A, n, c0, c0 + h, ipiv, c0 + h, c1);
}

}  // namespace

void dgetrf(cudaStream_t st, int64_t n, double* a, int32_t* ipiv, double* /*work*/, DevStatus* status,
            int block_index) {
  getrf_rec(st, a, n, 0, n, ipiv, status, block_index);
}

void dgetrs(cudaStream_t st, int64_t n, int64_t nrhs, const double* lu, const int32_t* ipiv, double* b,
            int64_t ldb, double* /*work*/) {
  laswp(st, b, ldb, 0, nrhs, ipiv, 0, n);
  trsm(st, true, lu, n, n, b, ldb, nrhs);
  trsm(st, false, lu, n, n, b, ldb, nrhs);
}

void dset_identity(cudaStream_t st, double* a, int64_t n) {
  identity_kernel<<<(unsigned)std::min<int64_t>(cdiv(n * n, 256), 8192), 256, 0, st>>>(a, n);
  SLB_CUDA_CHECK(cudaGetLastError());
}

void check_finite(cudaStream_t st, const double* a, int64_t count, DevStatus* status) {
  if (count <= 0) return;
  finite_kernel<<<(unsigned)std::min<int64_t>(cdiv(count, 256), 4096), 256, 0, st>>>(a, count, status);
  SLB_CUDA_CHECK(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// y = beta*y + alpha*A*x for small nrhs (deterministic split-K).
namespace {
constexpr int GV_ROWS = 64;   // rows per CTA (lane -> 2 rows)
constexpr int GV_SPLIT = 8;   // K splits
__global__ void gemv_partial_kernel(int64_t m, int64_t n, int64_t nrhs, const double* A, int64_t lda,
                                    const double* x, int64_t ldx, double* part) {
  const int64_t r0 = (int64_t)blockIdx.x * GV_ROWS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t kc = cdiv(n, GV_SPLIT);
  const int64_t k0 = blockIdx.y * kc, k1 = min(n, k0 + kc);
  __shared__ double red[8][GV_ROWS];
  for (int64_t c = 0; c < nrhs; c++) {
    double a0 = 0.0, a1 = 0.0;
    const int64_t ra = r0 + 2 * lane, rb = ra + 1;
    for (int64_t k = k0 + warp; k < k1; k += nw) {
      const double xv = x[c * ldx + k];
      const double* col = A + k * lda;
      if (ra < m) a0 = fma(col[ra], xv, a0);
      if (rb < m) a1 = fma(col[rb], xv, a1);
    }
    red[warp][2 * lane] = a0;
    red[warp][2 * lane + 1] = a1;
    __syncthreads();
    if (threadIdx.x < GV_ROWS) {
      double s = 0.0;
      for (int w = 0; w < nw; w++) s += red[w][threadIdx.x];
      const int64_t r = r0 + threadIdx.x;
      if (r < m) part[((int64_t)blockIdx.y * nrhs + c) * m + r] = s;
    }
    __syncthreads();
  }
}
__global__ void gemv_reduce_kernel(int64_t m, int64_t nrhs, double alpha, const double* part, double beta,
                                   double* y, int64_t ldy) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= m * nrhs) return;
  const int64_t r = idx % m, c = idx / m;
  double s = 0.0;
  for (int k = 0; k < GV_SPLIT; k++) s += part[((int64_t)k * nrhs + c) * m + r];
  double* yy = y + c * ldy + r;
  *yy = beta == 0.0 ? alpha * s : fma(alpha, s, beta * *yy);
}
}  // namespace

void dgemv_batched_rhs(cudaStream_t st, int64_t m, int64_t n, int64_t nrhs, double alpha, const double* A,
                       int64_t lda, const double* x, int64_t ldx, double beta, double* y, int64_t ldy,
                       double* part) {
  if (nrhs >= 16) {
    dgemm_batched(st, m, nrhs, n, alpha, A, lda, 0, x, ldx, 0, beta, y, ldy, 0, 1);
    return;
  }
  dim3 grid((unsigned)cdiv(m, GV_ROWS), GV_SPLIT);
  gemv_partial_kernel<<<grid, 256, 0, st>>>(m, n, nrhs, A, lda, x, ldx, part);
  SLB_CUDA_CHECK(cudaGetLastError());
  gemv_reduce_kernel<<<(unsigned)cdiv(m * nrhs, 256), 256, 0, st>>>(m, nrhs, alpha, part, beta, y, ldy);
  SLB_CUDA_CHECK(cudaGetLastError());
}

}  // namespace slb
