// Batched small triangular solves on the DMMA pipe (sm_100a).
//
//   X = T^{-1} B   in place, T m x m (m <= 160, multiple of 8) stored row-major,
//   lower => unit lower (forward), else upper non-unit (backward).
//
// Used by the band-LU level chain (U12|U13 = L11^{-1} R1 per level, the
// dgbtrf/dgbtrs triangular factors of proj/include/slablu/banded.hpp:99-128
// in block form) and by the conversion of every level's LU factors into the
// GEMM-form sweep operators.  One CTA = one 32-column tile of one batch item;
// the tile lives in shared memory, T streams from L2.  Row blocks of 16: the
// off-diagonal update is a DMMA GEMM (two accumulators for ILP), the 16 x 16
// diagonal block is solved per column.
#include "common.cuh"
#include "kernels.h"

namespace slb {
namespace {

constexpr int TN = 32;       // columns per tile
constexpr int MMAX = 160;
constexpr int RB = 16;       // rows per block

__device__ __forceinline__ int sw32(int r, int n) { return r * TN + (n ^ ((r & 3) << 2)); }

template <bool LOWER, bool ROWMAJOR>
__global__ void __launch_bounds__(256) trsm_small_kernel(int m, const double* __restrict__ Tg, int64_t ldt,
                                                         int64_t sT, double* Bg, int64_t ldb, int64_t sB,
                                                         int64_t ncols) {
  __shared__ double X[MMAX * TN];
  __shared__ double Td[RB][RB + 1];
  const int64_t item = blockIdx.y;
  const double* T = Tg + item * sT;
  double* B = Bg + item * sB;
  const int64_t c0 = (int64_t)blockIdx.x * TN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  // load the tile
  for (int idx = tid; idx < m * TN; idx += 256) {
    const int n = idx / m, r = idx % m;
    const int64_t c = c0 + n;
    X[sw32(r, n)] = c < ncols ? B[c * ldb + r] : 0.0;
  }
  __syncthreads();
  const int nb = (m + RB - 1) / RB;
  const int mt = warp >> 2, nt = warp & 3;
  for (int bi = 0; bi < nb; bi++) {
    const int b = LOWER ? bi : nb - 1 - bi;
    const int r0 = b * RB, r1 = min(m, r0 + RB), h = r1 - r0;
    // diagonal block to smem (overlaps the GEMM below)
    for (int idx = tid; idx < h * h; idx += 256) {
      const int rr = idx / h, cc = idx % h;
      Td[rr][cc] = ROWMAJOR ? T[(int64_t)(r0 + rr) * ldt + r0 + cc] : T[(int64_t)(r0 + cc) * ldt + r0 + rr];
    }
    // off-diagonal update: X[r0:r1] -= T[r0:r1, K] X[K]
    if (mt * 8 < h) {
      const int row = r0 + mt * 8 + g;
      const bool rok = row < r1;
      const int kb = LOWER ? 0 : r1, ke = LOWER ? r0 : m;
      double a0 = X[sw32(row, nt * 8 + 2 * t)], a1 = X[sw32(row, nt * 8 + 2 * t + 1)];
      double b0 = 0.0, b1 = 0.0;
      auto tv = [&](int k) -> double {  // -T[row][k], zero outside
        if (!rok || k >= ke) return 0.0;
        return ROWMAJOR ? -T[(int64_t)row * ldt + k] : -T[(int64_t)k * ldt + row];
      };
      auto xv = [&](int k) -> double { return k < ke ? X[sw32(k, nt * 8 + g)] : 0.0; };
      int k = kb;
      for (; k + 8 <= ke; k += 8) {
        const double f0 = tv(k + t), f1 = tv(k + 4 + t);
        const double x0 = xv(k + t), x1 = xv(k + 4 + t);
        dmma884(a0, a1, f0, x0);
        dmma884(b0, b1, f1, x1);
      }
      for (; k < ke; k += 4) dmma884(a0, a1, tv(k + t), xv(k + t));
      if (rok) {
        X[sw32(row, nt * 8 + 2 * t)] = a0 + b0;
        X[sw32(row, nt * 8 + 2 * t + 1)] = a1 + b1;
      }
    }
    __syncthreads();
    // diagonal solve, one thread per column
    if (tid < TN) {
      const int n = tid;
      double x[RB];
#pragma unroll
      for (int rr = 0; rr < RB; rr++) x[rr] = rr < h ? X[sw32(r0 + rr, n)] : 0.0;
      if (LOWER) {
#pragma unroll
        for (int rr = 1; rr < RB; rr++) {
          double s = x[rr];
#pragma unroll
          for (int cc = 0; cc < RB; cc++)
            if (cc < rr) s = fma(-Td[rr][cc], x[cc], s);
          x[rr] = s;
        }
      } else {
#pragma unroll
        for (int rr = RB - 1; rr >= 0; rr--) {
          if (rr >= h) continue;
          double s = x[rr];
#pragma unroll
          for (int cc = 0; cc < RB; cc++)
            if (cc > rr && cc < h) s = fma(-Td[rr][cc], x[cc], s);
          x[rr] = s / Td[rr][rr];
        }
      }
#pragma unroll
      for (int rr = 0; rr < RB; rr++)
        if (rr < h) X[sw32(r0 + rr, n)] = x[rr];
    }
    __syncthreads();
  }
  for (int idx = tid; idx < m * TN; idx += 256) {
    const int n = idx / m, r = idx % m;
    const int64_t c = c0 + n;
    if (c < ncols) B[c * ldb + r] = X[sw32(r, n)];
  }
}

}  // namespace

void trsm_small_batched(cudaStream_t st, bool lower, int m, const double* T, int64_t ldt, int64_t sT, double* B,
                        int64_t ldb, int64_t sB, int64_t ncols, int64_t batch, bool rowmajor) {
  if (m <= 0 || ncols <= 0 || batch <= 0) return;
  if (m > MMAX)
    throw CudaFailure(cudaErrorInvalidValue, "trsm_small_batched: m must be <= 160", __FILE__, __LINE__);
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
    const int64_t nb = std::min<int64_t>(65535, batch - b0);
    dim3 grid((unsigned)cdiv(ncols, TN), (unsigned)nb);
    const double* Tb = T + b0 * sT;
    double* Bb = B + b0 * sB;
    if (lower && rowmajor) trsm_small_kernel<true, true><<<grid, 256, 0, st>>>(m, Tb, ldt, sT, Bb, ldb, sB, ncols);
    else if (lower) trsm_small_kernel<true, false><<<grid, 256, 0, st>>>(m, Tb, ldt, sT, Bb, ldb, sB, ncols);
    else if (rowmajor) trsm_small_kernel<false, true><<<grid, 256, 0, st>>>(m, Tb, ldt, sT, Bb, ldb, sB, ncols);
    else trsm_small_kernel<false, false><<<grid, 256, 0, st>>>(m, Tb, ldt, sT, Bb, ldb, sB, ncols);
    SLB_CUDA_CHECK(cudaGetLastError());
  }
}

}  // namespace slb
