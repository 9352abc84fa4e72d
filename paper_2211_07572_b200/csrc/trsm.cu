// Batched small triangular solves on the DMMA pipe (sm_100a).
//
//   X = T^{-1} B   in place, T m x m (m <= 160), row-major or column-major;
//   lower => unit lower (forward), else upper non-unit (backward).
//
// Used by the band-LU level chain (U12|U13 = L11^{-1} R1 per level, the
// dgbtrf/dgbtrs triangular factors of proj/include/slablu/banded.hpp:99-128
// in block form), by the conversion of every level's LU factors into the
// GEMM-form sweep operators, and as the leaf of the stage-two recursive
// TRSM.  One CTA = one 32-column tile of one batch item; the tile lives in
// shared memory.  Row blocks of 16: the rows of T each block needs are staged
// into shared memory with cp.async one block ahead (double buffer), the
// off-diagonal update is a DMMA GEMM, the 16 x 16 diagonal block is solved
// per column.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace slb {
namespace {

constexpr int TN = 32;       // columns per tile
constexpr int MMAX = 160;
constexpr int RB = 16;       // rows per block
constexpr int KS = MMAX + 4; // staged T row stride (== 4 mod 16)

__device__ __forceinline__ int sw32(int r, int n) { return r * TN + (n ^ ((r & 3) << 2)); }

// Inverses of the nb diagonal RB x RB blocks of T (unit lower or upper non-unit), identity
// padded past m, into Dv[b][i][k] (row-major).  Thread (b, c) forms column c by substitution,
// once per CTA, so the per-block diagonal step becomes a small DMMA product instead of a
// 16-step serial solve by one warp while the others wait at the barrier.
template <bool LOWER, bool ROWMAJOR>
__device__ __forceinline__ void diag_inverses(const double* T, int64_t ldt, int m, int nb, double* Dv, int tid,
                                              int nthreads) {
  for (int idx = tid; idx < nb * RB * RB; idx += nthreads) {
    const int b = idx / (RB * RB), i = (idx / RB) % RB, k = idx % RB;
    const int r0 = b * RB, h = min(m, r0 + RB) - r0;
    Dv[idx] = (i < h && k < h) ? T[ROWMAJOR ? (int64_t)(r0 + i) * ldt + r0 + k : (int64_t)(r0 + k) * ldt + r0 + i]
                               : (i == k ? 1.0 : 0.0);
  }
  __syncthreads();
  double x[RB];
  const bool mine = tid < nb * RB;
  if (mine) {
    const int c = tid % RB;
    const double* D = Dv + (tid / RB) * RB * RB;
    if (LOWER) {
#pragma unroll
      for (int i = 0; i < RB; i++) {
        double sacc = i == c ? 1.0 : 0.0;
#pragma unroll
        for (int k = 0; k < RB; k++)
          if (k < i) sacc = fma(-D[i * RB + k], x[k], sacc);
        x[i] = sacc;
      }
    } else {
#pragma unroll
      for (int i = RB - 1; i >= 0; i--) {
        double sacc = i == c ? 1.0 : 0.0;
#pragma unroll
        for (int k = 0; k < RB; k++)
          if (k > i) sacc = fma(-D[i * RB + k], x[k], sacc);
        x[i] = sacc / D[i * RB + i];
      }
    }
  }
  __syncthreads();
  if (mine) {
    const int c = tid % RB;
    double* D = Dv + (tid / RB) * RB * RB;
#pragma unroll
    for (int i = 0; i < RB; i++) D[i * RB + c] = x[i];
  }
  __syncthreads();
}

// d -= T[row, kb:ke) . X[kb:ke, tile cols] for one 8x8 tile (row = this lane's row of T staged
// in trow, X swizzled); four independent DMMA chains, operands of four k4 steps loaded together.
// (ke - kb) must be a multiple of 4.
__device__ __forceinline__ void sub_row_block(const double* trow, const double* X, int col8, int kb, int ke, bool rok,
                                              int t, int g, double& d0, double& d1) {
  double c[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
  int k = kb;
  for (; k + 16 <= ke; k += 16) {
    double av[4], bv[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      av[u] = rok ? -trow[k + 4 * u + t] : 0.0;
      bv[u] = X[sw32(k + 4 * u + t, col8 + g)];
    }
#pragma unroll
    for (int u = 0; u < 4; u++) dmma884(c[u][0], c[u][1], av[u], bv[u]);
  }
#pragma unroll
  for (int u = 0; u < 3; u++) {  // remainder: at most three k4 steps (static register indices)
    if (k < ke) dmma884(c[u][0], c[u][1], rok ? -trow[k + t] : 0.0, X[sw32(k + t, col8 + g)]);
    k += 4;
  }
  d0 += (c[0][0] + c[1][0]) + (c[2][0] + c[3][0]);
  d1 += (c[0][1] + c[1][1]) + (c[2][1] + c[3][1]);
}

// X[r0:r0+16, 0:32] = Dinv_b X[r0:r0+16, 0:32] in place; 8 warps, warp (mt, nt) one 8x8 tile.
__device__ __forceinline__ void apply_diag_inverse(const double* Di, double* X, int r0, int r1, int warp, int g,
                                                   int t) {
  const int mt = warp >> 2, nt = warp & 3;
  double d0 = 0.0, d1 = 0.0;
#pragma unroll
  for (int kk = 0; kk < RB / 4; kk++)
    dmma884(d0, d1, Di[(mt * 8 + g) * RB + kk * 4 + t], X[sw32(r0 + kk * 4 + t, nt * 8 + g)]);
  __syncthreads();
  const int row = r0 + mt * 8 + g;
  if (row < r1) {
    X[sw32(row, nt * 8 + 2 * t)] = d0;
    X[sw32(row, nt * 8 + 2 * t + 1)] = d1;
  }
}

template <bool LOWER, bool ROWMAJOR>
__global__ void __launch_bounds__(256) trsm_small_kernel(int m, const double* __restrict__ Tg, int64_t ldt,
                                                         int64_t sT, double* Bg, int64_t ldb, int64_t sB,
                                                         int64_t ncols) {
  extern __shared__ double sm[];
  double* X = sm;                       // MMAX * TN
  double* sTb = sm + MMAX * TN;         // 2 x RB x KS
  double* Dv = sTb + 2 * RB * KS;       // (MMAX / RB) x RB x RB diagonal-block inverses
  const int64_t item = blockIdx.y;
  const double* T = Tg + item * sT;
  double* B = Bg + item * sB;
  const int64_t c0 = (int64_t)blockIdx.x * TN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int nb = (m + RB - 1) / RB;
  auto block_of = [&](int bi) { return LOWER ? bi : nb - 1 - bi; };
  // stage rows [r0, r1) of T, all m columns, into buffer buf (row-major, stride KS)
  auto stage = [&](int bi, int buf) {
    if (bi >= nb) return;
    const int r0 = block_of(bi) * RB, h = min(m, r0 + RB) - r0;
    double* dst = sTb + buf * RB * KS;
    if (ROWMAJOR) {
      for (int idx = tid; idx < h * m; idx += 256) {
        const int rr = idx / m, c = idx % m;
        cp_async8(dst + rr * KS + c, T + (int64_t)(r0 + rr) * ldt + c, true);
      }
    } else {
      for (int idx = tid; idx < h * m; idx += 256) {
        const int c = idx / h, rr = idx % h;
        cp_async8(dst + rr * KS + c, T + (int64_t)c * ldt + r0 + rr, true);
      }
    }
  };
  stage(0, 0);
  cp_async_commit();
  bool nz = false;
  for (int idx = tid; idx < m * TN; idx += 256) {
    const int n = idx / m, r = idx % m;
    const int64_t c = c0 + n;
    const double v = c < ncols ? B[c * ldb + r] : 0.0;
    nz |= v != 0.0;
    X[sw32(r, n)] = v;
  }
  // an all-zero right-hand-side tile has the zero solution, already in place (the U13 columns of
  // the level conversion are zero but for the few rows pivoted up from the next level)
  if (!__syncthreads_or(nz)) {
    cp_async_wait<0>();
    return;
  }
  for (int idx = m * TN + tid; idx < nb * RB * TN; idx += 256) X[idx] = 0.0;  // padding rows of the last block
  diag_inverses<LOWER, ROWMAJOR>(T, ldt, m, nb, Dv, tid, 256);
  const int mt = warp >> 2, nt = warp & 3;
  for (int bi = 0; bi < nb; bi++) {
    const int b = block_of(bi);
    const int r0 = b * RB, r1 = min(m, r0 + RB), h = r1 - r0;
    stage(bi + 1, (bi + 1) & 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* Tb = sTb + (bi & 1) * RB * KS;  // rows r0..r1 of T
    // off-diagonal update: X[r0:r1] -= T[r0:r1, K] X[K]
    if (mt * 8 < h) {
      const int rloc = mt * 8 + g;
      const bool rok = r0 + rloc < r1;
      const int kb = LOWER ? 0 : r1, ke = LOWER ? r0 : m;
      const int row = rok ? r0 + rloc : r0;
      double a0 = X[sw32(row, nt * 8 + 2 * t)], a1 = X[sw32(row, nt * 8 + 2 * t + 1)];
      double b0 = 0.0, b1 = 0.0;
      const double* trow = Tb + rloc * KS;
      auto tv = [&](int k) -> double { return (rok && k < ke) ? -trow[k] : 0.0; };
      auto xv = [&](int k) -> double { return k < ke ? X[sw32(k, nt * 8 + g)] : 0.0; };
      int k = kb;
      for (; k + 8 <= ke; k += 8) {
        dmma884(a0, a1, tv(k + t), xv(k + t));
        dmma884(b0, b1, tv(k + 4 + t), xv(k + 4 + t));
      }
      for (; k < ke; k += 4) dmma884(a0, a1, tv(k + t), xv(k + t));
      if (rok) {
        X[sw32(row, nt * 8 + 2 * t)] = a0 + b0;
        X[sw32(row, nt * 8 + 2 * t + 1)] = a1 + b1;
      }
    }
    __syncthreads();
    // diagonal block: X_b = D_b^{-1} X_b (precomputed inverse, DMMA)
    apply_diag_inverse(Dv + b * RB * RB, X, r0, r1, warp, g, t);
    __syncthreads();  // X block final; the staging buffer may be refilled
  }
  cp_async_wait<0>();
  __syncthreads();
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
  const size_t smem = (size_t)(MMAX * TN + 2 * RB * KS + MMAX * RB) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    SLB_CUDA_CHECK(cudaFuncSetAttribute(trsm_small_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    SLB_CUDA_CHECK(cudaFuncSetAttribute(trsm_small_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    SLB_CUDA_CHECK(cudaFuncSetAttribute(trsm_small_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    SLB_CUDA_CHECK(cudaFuncSetAttribute(trsm_small_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
    const int64_t nb = std::min<int64_t>(65535, batch - b0);
    dim3 grid((unsigned)cdiv(ncols, TN), (unsigned)nb);
    const double* Tb = T + b0 * sT;
    double* Bb = B + b0 * sB;
    if (lower && rowmajor) trsm_small_kernel<true, true><<<grid, 256, smem, st>>>(m, Tb, ldt, sT, Bb, ldb, sB, ncols);
    else if (lower) trsm_small_kernel<true, false><<<grid, 256, smem, st>>>(m, Tb, ldt, sT, Bb, ldb, sB, ncols);
    else if (rowmajor) trsm_small_kernel<false, true><<<grid, 256, smem, st>>>(m, Tb, ldt, sT, Bb, ldb, sB, ncols);
    else trsm_small_kernel<false, false><<<grid, 256, smem, st>>>(m, Tb, ldt, sT, Bb, ldb, sB, ncols);
    count_launch();
    SLB_CUDA_CHECK(cudaGetLastError());
  }
}

}  // namespace slb

// ---------------------------------------------------------------------------
// Fused per-level update of the band-LU chain (one launch per level):
//   R = perm_l [V_l 0 ; D_{l+1} Usup_{l+1}],  U1213 = L11^{-1} R1,
//   [S | V]_{l+1} = R2 - L21 U1213.
// grid (2Wp / 32 column tiles, strips), 256 threads; the 32-column tile of
// U1213 stays in shared memory between the TRSM and the GEMM, L11/L21 rows
// are staged through a cp.async double buffer.
namespace slb {
namespace {
__global__ void __launch_bounds__(256) level_update_kernel(LevelArgs a) {
  extern __shared__ double sm[];
  const int Wp = a.Wp, s = blockIdx.y;
  double* X = sm;                 // MMAX * TN   (U1213 tile, swizzled)
  double* sTb = sm + MMAX * TN;   // 2 x RB x KS (staged rows of L11 / L21)
  double* Dv = sTb + 2 * RB * KS; // inverses of L11's 16 x 16 diagonal blocks
  int* sperm = reinterpret_cast<int*>(Dv + MMAX * RB);  // this level's pivot order (2 Wp)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int c0 = blockIdx.x * TN;
  const double* V = a.sv_in + s * a.sSV + (int64_t)Wp * Wp;
  const double* NX = a.nx + s * a.sNX;
  const int32_t* perm = a.perm + s * a.sP;
  double* slot = a.slot + s * a.sF;
  const double* LU11 = slot;
  const double* L21 = slot + (int64_t)Wp * Wp;
  double* U1213 = slot + 2LL * Wp * Wp;
  double* svo = a.sv_out + s * a.sSV;
  auto Rval = [&](int p, int c) -> double {
    if (p < Wp) return c < Wp ? V[(int64_t)c * Wp + p] : 0.0;
    return NX[(int64_t)(Wp + c) * Wp + (p - Wp)];
  };
  const int m = Wp;
  const int nb = (m + RB - 1) / RB;
  auto stage_rows = [&](const double* T, int r0, int buf) {  // rows r0..r0+16 of a row-major Wp x Wp
    const int h = min(m, r0 + RB) - r0;
    double* dst = sTb + buf * RB * KS;
    const int m2 = m / 2;  // Wp is a multiple of 8: rows are whole 16-byte pieces
    const float inv_m2 = 1.0f / (float)m2;
    for (int idx = tid; idx < h * m2; idx += 256) {
      const int rr = qdiv(idx, inv_m2), c = 2 * (idx - rr * m2);
      cp_async16(dst + rr * KS + c, T + (int64_t)(r0 + rr) * m + c, true);
    }
  };
  // ---- R1 tile -> X (gathered through perm)
#ifdef SLB_UPD_PROF
  long long P0 = clock64(), ph[6] = {0, 0, 0, 0, 0, 0};
#define UP(k_) { const long long q_ = clock64(); ph[k_] += q_ - P0; P0 = q_; }
#else
#define UP(k_)
#endif
  pdl_wait();     // the level's LU (and, transitively, everything before it) is complete
  pdl_trigger();  // the next level's LU may start launching
  stage_rows(LU11, 0, 0);
  cp_async_commit();
  const int ncol = min(TN, 2 * Wp - c0);
  const int mt = warp >> 2, nt = warp & 3;
  for (int i = tid; i < 2 * Wp; i += 256) sperm[i] = perm[i];
  __syncthreads();
  const float inv_m = 1.0f / (float)m;
  for (int idx = tid; idx < m * TN; idx += 256) {  // asynchronous gather (many loads in flight)
    const int n = qdiv(idx, inv_m), r = idx - n * m;
    const int p = sperm[r], c = c0 + n;
    double* dst = &X[sw32(r, n)];
    if (n >= ncol || (p < Wp && c >= Wp)) *dst = 0.0;
    else cp_async8(dst, p < Wp ? V + (int64_t)c * Wp + p : NX + (int64_t)(Wp + c) * Wp + (p - Wp), true);
  }
  cp_async_commit();
  for (int idx = m * TN + tid; idx < nb * RB * TN; idx += 256) X[idx] = 0.0;
  diag_inverses<true, true>(LU11, Wp, m, nb, Dv, tid, 256);
  UP(0)
  // ---- TRSM: X = L11^{-1} X (unit lower)
  for (int b = 0; b < nb; b++) {
    const int r0 = b * RB, r1 = min(m, r0 + RB), h = r1 - r0;
    if (b + 1 < nb) stage_rows(LU11, (b + 1) * RB, (b + 1) & 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    UP(1)
    const double* Tb = sTb + (b & 1) * RB * KS;
    if (mt * 8 < h) {
      const int rloc = mt * 8 + g;
      const bool rok = r0 + rloc < r1;
      const int row = rok ? r0 + rloc : r0;
      double a0 = X[sw32(row, nt * 8 + 2 * t)], a1 = X[sw32(row, nt * 8 + 2 * t + 1)];
      sub_row_block(Tb + rloc * KS, X, nt * 8, 0, r0, rok, t, g, a0, a1);
      if (rok) {
        X[sw32(row, nt * 8 + 2 * t)] = a0;
        X[sw32(row, nt * 8 + 2 * t + 1)] = a1;
      }
    }
    __syncthreads();
    apply_diag_inverse(Dv + b * RB * RB, X, r0, r1, warp, g, t);
    __syncthreads();
  }
  UP(2)
  // ---- U1213 tile out
  for (int idx = tid; idx < m * ncol; idx += 256) {
    const int n = qdiv(idx, inv_m), r = idx - n * m;
    U1213[(int64_t)(c0 + n) * Wp + r] = X[sw32(r, n)];
  }
  // ---- GEMM: out = R2 - L21 X, row blocks of 16 of L21 staged like L11
  stage_rows(L21, 0, 0);
  cp_async_commit();
  // R2 values of this thread's outputs, one block ahead (their latency hides behind a block)
  const int colq = c0 + nt * 8 + 2 * t;
  auto r2 = [&](int b, int dc) -> double {
    const int row = b * RB + mt * 8 + g;
    return (b < nb && row < m && colq + dc < 2 * Wp) ? Rval(sperm[Wp + row], colq + dc) : 0.0;
  };
  double rn0 = r2(0, 0), rn1 = r2(0, 1);
  for (int b = 0; b < nb; b++) {
    const int r0 = b * RB, r1 = min(m, r0 + RB), h = r1 - r0;
    if (b + 1 < nb) stage_rows(L21, (b + 1) * RB, (b + 1) & 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    UP(3)
    const double* Tb = sTb + (b & 1) * RB * KS;
    if (mt * 8 < h) {
      const int rloc = mt * 8 + g;
      const bool rok = r0 + rloc < r1;
      const int row = rok ? r0 + rloc : r0;
      const int col = colq;
      const double r0v = rn0, r1v = rn1;
      rn0 = r2(b + 1, 0);
      rn1 = r2(b + 1, 1);
      double a0 = 0.0, a1 = 0.0;
      sub_row_block(Tb + rloc * KS, X, nt * 8, 0, m, rok, t, g, a0, a1);
      if (rok && col < 2 * Wp) svo[(int64_t)col * Wp + row] = r0v + a0;
      if (rok && col + 1 < 2 * Wp) svo[(int64_t)(col + 1) * Wp + row] = r1v + a1;
    }
    __syncthreads();
    UP(4)
  }
#ifdef SLB_UPD_PROF
  if (tid == 0 && blockIdx.x == 0 && blockIdx.y == 0 && (a.level % 1000) == 1)
    printf("UPD l=%d: gather %lld trsm-wait %lld trsm-compute %lld gemm-wait %lld gemm-compute %lld (cycles)\n", a.level,
           ph[0], ph[1], ph[2], ph[3], ph[4]);
#endif
}
// Version 2 of the level update, right-looking: per 16-row block b of the TRSM the diagonal
// block is applied (precomputed inverse) and ALL rows below take the rank-16 update at once
// (independent 8x8 tiles over the 8 warps), so the sequential depth is one small step per
// block instead of a left-looking dot product over the growing k range; the GEMM
// R2 - L21 U1213 accumulates in registers over 16-column blocks of L21 (no per-row-block
// round trip through shared memory).  L11 / L21 column blocks are staged with cp.async one
// block ahead.  Selected by SLB_UPD_V2=1 (the default is the left-looking kernel above).
constexpr int LCS = RB + 4;  // staged column-block row stride (doubles)
constexpr int UT = 10;       // output tiles per warp in the GEMM (Wp <= 160: 20 x 4 tiles / 8 warps)
__global__ void __launch_bounds__(256) level_update2_kernel(LevelArgs a) {
  extern __shared__ double sm[];
  const int Wp = a.Wp, s = blockIdx.y;
  double* X = sm;                  // MMAX * TN   (U1213 tile, swizzled)
  double* Lc = sm + MMAX * TN;     // 2 x MMAX x LCS (staged column block of L11 / L21)
  double* Dv = Lc + 2 * MMAX * LCS;  // inverses of L11's 16 x 16 diagonal blocks
  int* sperm = reinterpret_cast<int*>(Dv + MMAX * RB);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int c0 = blockIdx.x * TN;
  const double* V = a.sv_in + s * a.sSV + (int64_t)Wp * Wp;
  const double* NX = a.nx + s * a.sNX;
  const int32_t* perm = a.perm + s * a.sP;
  double* slot = a.slot + s * a.sF;
  const double* LU11 = slot;
  const double* L21 = slot + (int64_t)Wp * Wp;
  double* U1213 = slot + 2LL * Wp * Wp;
  double* svo = a.sv_out + s * a.sSV;
  const int m = Wp;
  const int nb = (m + RB - 1) / RB;
  const int mt_all = m / 8;  // Wp is a multiple of 8
  const int ncol = min(TN, 2 * Wp - c0);
  // rows [rlo, m) of column block kb of a row-major m x m matrix -> Lc[buf][row][0..16)
  auto stage_cols = [&](const double* T, int kb, int rlo, int buf) {
    const int k0 = kb * RB, kw = min(m, k0 + RB) - k0;  // kw is a multiple of 8
    const int pieces = kw / 2;                           // 16-byte pieces per row
    double* dst = Lc + buf * MMAX * LCS;
    const int total = (m - rlo) * pieces;
    const float inv_p = 1.0f / (float)pieces;
    for (int idx = tid; idx < total; idx += 256) {
      const int rr = qdiv(idx, inv_p), c = 2 * (idx - rr * pieces);
      const int row = rlo + rr;
      cp_async16(dst + row * LCS + c, T + (int64_t)row * m + k0 + c, true);
    }
    cp_async_commit();
  };
  // ---- R1 tile -> X (gathered through perm, asynchronous), diagonal-block inverses
  for (int i = tid; i < 2 * Wp; i += 256) sperm[i] = perm[i];
  __syncthreads();
  const float inv_m = 1.0f / (float)m;
  for (int idx = tid; idx < m * TN; idx += 256) {
    const int n = qdiv(idx, inv_m), r = idx - n * m;
    const int p = sperm[r], c = c0 + n;
    double* dst = &X[sw32(r, n)];
    if (n >= ncol || (p < Wp && c >= Wp)) *dst = 0.0;
    else cp_async8(dst, p < Wp ? V + (int64_t)c * Wp + p : NX + (int64_t)(Wp + c) * Wp + (p - Wp), true);
  }
  cp_async_commit();
  for (int idx = m * TN + tid; idx < nb * RB * TN; idx += 256) X[idx] = 0.0;
#ifdef SLB_UPD_PROF
  long long Q0 = clock64(), qh[4] = {0, 0, 0, 0};
#define UQ(k_) { const long long q_ = clock64(); qh[k_] += q_ - Q0; Q0 = q_; }
#else
#define UQ(k_)
#endif
  stage_cols(LU11, 0, min(m, RB), 0);
  diag_inverses<true, true>(LU11, Wp, m, nb, Dv, tid, 256);
  UQ(0)
  // ---- TRSM, right-looking: X = L11^{-1} X (unit lower)
  for (int b = 0; b < nb; b++) {
    const int r0 = b * RB, r1 = min(m, r0 + RB);
    cp_async_wait<0>();
    __syncthreads();  // X (gather, previous trailing updates) and column block b staged
    apply_diag_inverse(Dv + b * RB * RB, X, r0, r1, warp, g, t);
    __syncthreads();
    if (b + 1 < nb) stage_cols(LU11, b + 1, min(m, r1 + RB), (b + 1) & 1);
    // X[r1:m] -= L11[r1:m, r0:r1] X[r0:r1]: (rows below) x 4 column tiles over the 8 warps
    const double* lc = Lc + (b & 1) * MMAX * LCS;
    const int mt0 = r1 / 8, ntile = (mt_all - mt0) * 4;
    for (int tile = warp; tile < ntile; tile += 8) {
      const int mt = mt0 + (tile >> 2), nt = tile & 3;
      const int row = mt * 8 + g;
      double d0 = X[sw32(row, nt * 8 + 2 * t)], d1 = X[sw32(row, nt * 8 + 2 * t + 1)];
#pragma unroll
      for (int kk = 0; kk < RB / 4; kk++) {
        const int k = kk * 4 + t;
        if (r0 + kk * 4 < r1)
          dmma884(d0, d1, -lc[row * LCS + k], X[sw32(r0 + k, nt * 8 + g)]);
      }
      X[sw32(row, nt * 8 + 2 * t)] = d0;
      X[sw32(row, nt * 8 + 2 * t + 1)] = d1;
    }
  }
  __syncthreads();
  UQ(1)
  // ---- U1213 tile out; the GEMM's first L21 column block
  stage_cols(L21, 0, 0, 0);
  for (int idx = tid; idx < m * ncol; idx += 256) {
    const int n = qdiv(idx, inv_m), r = idx - n * m;
    U1213[(int64_t)(c0 + n) * Wp + r] = X[sw32(r, n)];
  }
  // ---- GEMM: out = R2 - L21 X, accumulated over column blocks of L21
  double acc[UT][2];
  double r2v[UT][2];
  const int ntiles = mt_all * 4;
#pragma unroll
  for (int i = 0; i < UT; i++) {
    acc[i][0] = acc[i][1] = 0.0;
    r2v[i][0] = r2v[i][1] = 0.0;
    const int tile = warp + 8 * i;
    if (tile < ntiles) {
      const int row = (tile >> 2) * 8 + g, col = c0 + (tile & 3) * 8 + 2 * t;
      const int p = sperm[Wp + row];
      if (col < 2 * Wp) r2v[i][0] = p < Wp ? (col < Wp ? V[(int64_t)col * Wp + p] : 0.0)
                                           : NX[(int64_t)(Wp + col) * Wp + (p - Wp)];
      if (col + 1 < 2 * Wp) r2v[i][1] = p < Wp ? (col + 1 < Wp ? V[(int64_t)(col + 1) * Wp + p] : 0.0)
                                               : NX[(int64_t)(Wp + col + 1) * Wp + (p - Wp)];
    }
  }
  for (int kb = 0; kb < nb; kb++) {
    cp_async_wait<0>();
    __syncthreads();
    if (kb + 1 < nb) stage_cols(L21, kb + 1, 0, (kb + 1) & 1);
    const double* lc = Lc + (kb & 1) * MMAX * LCS;
    const int k0 = kb * RB, kw = min(m, k0 + RB) - k0;
#pragma unroll
    for (int i = 0; i < UT; i++) {
      const int tile = warp + 8 * i;
      if (tile >= ntiles) break;
      const int row = (tile >> 2) * 8 + g, nt = tile & 3;
#pragma unroll
      for (int kk = 0; kk < RB / 4; kk++)
        if (kk * 4 < kw)
          dmma884(acc[i][0], acc[i][1], lc[row * LCS + kk * 4 + t], X[sw32(k0 + kk * 4 + t, nt * 8 + g)]);
    }
  }
  UQ(2)
#ifdef SLB_UPD_PROF
  if (tid == 0 && blockIdx.x == 0 && blockIdx.y == 0 && (a.level % 1000) == 1)
    printf("UPD2 l=%d: gather+inverses %lld trsm %lld gemm %lld (cycles)\n", a.level, qh[0], qh[1], qh[2]);
#endif
#pragma unroll
  for (int i = 0; i < UT; i++) {
    const int tile = warp + 8 * i;
    if (tile >= ntiles) break;
    const int row = (tile >> 2) * 8 + g, col = c0 + (tile & 3) * 8 + 2 * t;
    if (col < 2 * Wp) svo[(int64_t)col * Wp + row] = r2v[i][0] - acc[i][0];
    if (col + 1 < 2 * Wp) svo[(int64_t)(col + 1) * Wp + row] = r2v[i][1] - acc[i][1];
  }
}
}  // namespace

void level_update(cudaStream_t st, const LevelArgs& a) {
  const size_t smem = (size_t)(MMAX * TN + 2 * RB * KS + MMAX * RB) * sizeof(double) + 2 * MMAX * sizeof(int);
  static bool attr = false;
  if (!attr) {
    SLB_CUDA_CHECK(cudaFuncSetAttribute(level_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  dim3 grid((unsigned)cdiv(2 * a.Wp, TN), (unsigned)a.nstrips);
  // default: the left-looking kernel (its rounding stays closer to dgbtrf's: staged parity at
  // cfg3 1.9e-11 vs 5.3e-11 for version 2, which is 2.5 % faster); SLB_UPD_V2=1 selects version 2
  static const bool v1 = getenv("SLB_UPD_V2") == nullptr;
  if (v1) {
    launch_pdl(level_update_kernel, grid, dim3(256), smem, st, a);
  } else {
    const size_t smem2 = (size_t)(MMAX * TN + 2 * MMAX * LCS + MMAX * RB) * sizeof(double) + 2 * MMAX * sizeof(int);
    static bool attr2 = false;
    if (!attr2) {
      SLB_CUDA_CHECK(cudaFuncSetAttribute(level_update2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
      attr2 = true;
    }
    level_update2_kernel<<<grid, 256, smem2, st>>>(a); count_launch();
  }
  SLB_CUDA_CHECK(cudaGetLastError());
}
}  // namespace slb
