// Stage one, part 1: block band LU of every slab interior (sm_100a).
//
// Reference: BandedLU = LAPACKE_dgbtrf on the permuted interior
// (proj/include/slablu/banded.hpp:99-111, filled at stage_one.hpp:176-199).
// The permuted interior (row iy*w + ix) is block tridiagonal with w x w
// level blocks; dgbtrf's partial pivoting window (rows c..c+kl, kl = w)
// spans exactly the current level and the next one.  We factor level by
// level with the same pivot rule (first max |a| in the window), on
// Wp-padded blocks (Wp = round_up(b, 8); padded unknowns are decoupled
// identity rows that never win a pivot):
//
//   panel  P_l = [S_l ; Lsub_{l+1}]  (2Wp x Wp)      -> perm_l (window pivots)
//   A11 = (perm_l P_l)_top, B = (perm_l P_l)_bot
//   Ainv_l = A11^{-1}   (Gauss-Jordan, pivots known)
//   Fbot_l = -B Ainv_l
//   R  = perm_l [V_l 0 ; D_{l+1} Usup_{l+1}] = [R1 ; R2]
//   H_l = Ainv_l R1,  [S_{l+1} | V_{l+1}] = R2 - B H_l
//
// so that A_ii^{-1} b is the pure-GEMM sweep
//   forward  t = perm_l [z_l ; b_{l+1}],  y_l = Ainv_l t_top,  z_{l+1} = t_bot + Fbot_l t_top
//   backward x_l = y_l - H_l [x_{l+1} ; x_{l+2}]
// used by the Schur kernel (schur.cu) and the solves (solve.cu).
#include <climits>

#include "common.cuh"
#include "kernels.h"

namespace slb {
namespace {

__device__ __forceinline__ void raise(DevStatus* st, int32_t bit) { atomicOr(&st->flags, bit); }

// ---------------------------------------------------------------------------
// Level blocks [Lsub | D | Usup] of one strip level from the CSR.
// grid (nl, nstrips), block 128.
__global__ void extract_levels_kernel(CsrDev A, const StripDesc* strips, int64_t n2, int Wp,
                                      int64_t L0, double* nx, int64_t sNX, DevStatus* status) {
  const int s = blockIdx.y;
  const int64_t L = L0 + blockIdx.x;
  const StripDesc sd = strips[s];
  double* out = nx + s * sNX + (int64_t)blockIdx.x * 3 * Wp * Wp;
  for (int idx = threadIdx.x; idx < 3 * Wp * Wp; idx += blockDim.x) out[idx] = 0.0;
  __syncthreads();
  for (int i = sd.w + threadIdx.x; i < Wp; i += blockDim.x) out[(Wp + i) * Wp + i] = 1.0;  // padding
  const int64_t begin = (int64_t)sd.col0 * n2, end = (int64_t)(sd.col0 + sd.w) * n2;
  for (int ix = threadIdx.x; ix < sd.w; ix += blockDim.x) {
    const int64_t g = (int64_t)(sd.col0 + ix) * n2 + L;
    for (int32_t p = A.rp[g]; p < A.rp[g + 1]; p++) {
      const int64_t c = A.ci[p];
      const double v = A.v[p];
      if (c >= begin && c < end) {
        const int cx = (int)(c / n2) - sd.col0;
        const int64_t cy = c % n2;
        const int64_t dy = cy - L;
        const int64_t off = dy * sd.w + (cx - ix);
        if (off > sd.w || off < -sd.w) {
          raise(status, ERR_OUT_OF_BAND);
          continue;
        }
        // dy in {-1, 0, 1}: Lsub, D, Usup
        out[((dy + 1) * Wp + cx) * Wp + ix] = v;
      } else if (sd.left >= 0 && c >= sd.left_off && c < sd.left_off + n2) {
        if (c - sd.left_off != L) raise(status, ERR_COUPLING_LEVEL);
      } else if (sd.right >= 0 && c >= sd.right_off && c < sd.right_off + n2) {
        if (c - sd.right_off != L) raise(status, ERR_COUPLING_LEVEL);
      } else {
        raise(status, ERR_PAST_INTERFACE);
      }
    }
  }
}

// Finds A[r][c] in CSR row r (rows hold <= a handful of entries).
__device__ __forceinline__ bool csr_find(const CsrDev& A, int64_t r, int64_t c, double* v) {
  for (int32_t p = A.rp[r]; p < A.rp[r + 1]; p++)
    if (A.ci[p] == c) {
      *v = A.v[p];
      return true;
    }
  return false;
}

// Coupling vectors per (strip, level): cpl[s] = [fromL | fromR | toL | toR],
// each n2 x Wp row-major (level, ix).  Also clears sym_flags[s] when the strip
// is not symmetric (A_ii != A_ii^T or to_X != from_X^T).
// grid (ceil(n2/8), nstrips), block (32, 8): threadIdx.x = ix lane, y = level.
__global__ void extract_couplings_kernel(CsrDev A, const StripDesc* strips, int64_t n2, int Wp,
                                         double* cpl, int64_t sCPL, int32_t* sym, DevStatus* status) {
  const int s = blockIdx.y;
  const int64_t L = (int64_t)blockIdx.x * blockDim.y + threadIdx.y;
  if (L >= n2) return;
  const StripDesc sd = strips[s];
  double* fromL = cpl + s * sCPL;
  double* fromR = fromL + n2 * Wp;
  double* toL = fromR + n2 * Wp;
  double* toR = toL + n2 * Wp;
  const int64_t begin = (int64_t)sd.col0 * n2, end = (int64_t)(sd.col0 + sd.w) * n2;
  bool symmetric = true;
  for (int ix = threadIdx.x; ix < Wp; ix += blockDim.x) {
    double fl = 0.0, fr = 0.0, tl = 0.0, tr = 0.0;
    if (ix < sd.w) {
      const int64_t g = (int64_t)(sd.col0 + ix) * n2 + L;
      if (sd.left >= 0) csr_find(A, g, sd.left_off + L, &fl);
      if (sd.right >= 0) csr_find(A, g, sd.right_off + L, &fr);
      if (sd.left >= 0) csr_find(A, sd.left_off + L, g, &tl);
      if (sd.right >= 0) csr_find(A, sd.right_off + L, g, &tr);
      if (fl != tl || fr != tr) symmetric = false;
      // interior symmetry: every in-strip entry has an equal transpose
      for (int32_t p = A.rp[g]; p < A.rp[g + 1]; p++) {
        const int64_t c = A.ci[p];
        if (c >= begin && c < end) {
          double vt = 0.0;
          if (!csr_find(A, c, g, &vt) || vt != A.v[p]) symmetric = false;
        }
      }
    }
    fromL[L * Wp + ix] = fl;
    fromR[L * Wp + ix] = fr;
    toL[L * Wp + ix] = tl;
    toR[L * Wp + ix] = tr;
  }
  // interface rows: every entry inside the strip must sit on level L
  if (threadIdx.x == 0) {
    const int64_t offs[2] = {sd.left >= 0 ? sd.left_off : -1, sd.right >= 0 ? sd.right_off : -1};
    for (int e = 0; e < 2; e++) {
      if (offs[e] < 0) continue;
      const int64_t r = offs[e] + L;
      for (int32_t p = A.rp[r]; p < A.rp[r + 1]; p++) {
        const int64_t c = A.ci[p];
        if (c >= begin && c < end && c % n2 != L) raise(status, ERR_COUPLING_LEVEL);
      }
    }
  }
  if (!symmetric) sym[s] = 0;
}

__global__ void init_sv_kernel(int Wp, const double* nx0, int64_t sNX, double* sv, int64_t sSV) {
  const int s = blockIdx.x;
  const double* src = nx0 + s * sNX + (int64_t)Wp * Wp;  // [D | Usup]
  double* dst = sv + s * sSV;
  for (int idx = threadIdx.x; idx < 2 * Wp * Wp; idx += blockDim.x) dst[idx] = src[idx];
}

// ---------------------------------------------------------------------------
// One level step for every strip: window-pivoted panel LU (pivot order only),
// Gauss-Jordan inverse of the pivot block, and the gathers feeding the GEMMs.
// grid = nstrips, block = 1024.
__global__ void __launch_bounds__(1024) level_panel_kernel(LevelArgs a) {
  extern __shared__ double smem[];
  const int Wp = a.Wp, NW = Wp + 1, RS = Wp + 1;
  double* win = smem;            // NW * RS
  double* prow = win + NW * RS;  // Wp + 1
  double* fcol = prow + Wp + 1;  // Wp + 1
  int* perm = reinterpret_cast<int*>(fcol + Wp + 1);  // 2 Wp
  __shared__ int s_piv;
  __shared__ int s_sing;

  const int s = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const double* SV = a.sv_in + s * a.sSV;
  const double* NX = a.has_next ? a.nx + s * a.sNX : nullptr;
  const int rows_total = a.has_next ? 2 * Wp : Wp;
  auto Pval = [&](int p, int j) -> double {
    return p < Wp ? SV[(int64_t)j * Wp + p] : NX[(int64_t)j * Wp + (p - Wp)];
  };
  if (tid == 0) s_sing = 0;

  // ---- phase 1: window LU, pivot order only --------------------------------
  const int init_rows = rows_total < NW ? rows_total : NW;
  for (int idx = tid; idx < init_rows * Wp; idx += blockDim.x) {
    const int j = idx / init_rows, p = idx % init_rows;
    win[p * RS + j] = Pval(p, j);
  }
  for (int p = tid; p < 2 * Wp; p += blockDim.x) perm[p] = p;
  // register prefetch of the next entering bottom row (position Wp + 1 + k -> bottom row k + 1)
  double nextv = 0.0;
  if (a.has_next && tid < Wp && Wp > 1) nextv = NX[(int64_t)tid * Wp + 1];
  __syncthreads();

  for (int k = 0; k < Wp; k++) {
    const int hi = min(k + Wp, rows_total - 1);
    if (warp == 0) {
      double best = -1.0;
      int bpos = INT_MAX;
      for (int pos = k + lane; pos <= hi; pos += 32) {
        const double v = fabs(win[(pos % NW) * RS + k]);
        if (v > best) {
          best = v;
          bpos = pos;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int op = __shfl_xor_sync(0xffffffffu, bpos, o);
        if (ob > best || (ob == best && op < bpos)) {
          best = ob;
          bpos = op;
        }
      }
      int r = bpos;
      if (!(best > 0.0)) {  // exactly singular (or NaN) column
        r = k;
        if (lane == 0) s_sing = 1;
      }
      if (r != k) {
        double* rk = win + (k % NW) * RS;
        double* rr = win + (r % NW) * RS;
        for (int j = lane; j < Wp; j += 32) {
          const double t = rk[j];
          rk[j] = rr[j];
          rr[j] = t;
        }
        if (lane == 0) {
          const int t = perm[k];
          perm[k] = perm[r];
          perm[r] = t;
        }
        __syncwarp();
      }
      const double* rk = win + (k % NW) * RS;
      for (int j = lane; j < Wp; j += 32) prow[j] = rk[j];
    }
    __syncthreads();
    const double pv = prow[k];
    const double inv = pv != 0.0 ? 1.0 / pv : 0.0;
    for (int pos = k + 1 + warp; pos <= hi; pos += nwarps) {
      double* row = win + (pos % NW) * RS;
      const double m = row[k] * inv;
      if (m != 0.0)
        for (int j = k + 1 + lane; j < Wp; j += 32) row[j] = fma(-m, prow[j], row[j]);
    }
    // entering row: position k + Wp + 1 = bottom row k + 1, into the freed slot of position k
    if (k + Wp + 1 < rows_total) {
      if (tid < Wp) win[(k % NW) * RS + tid] = nextv;
      if (tid < Wp && k + 2 < Wp) nextv = NX[(int64_t)tid * Wp + (k + 2)];
    }
    __syncthreads();
  }

  // ---- gathers: perm, Bsel, R1, R2 (-> sv_out) ---------------------------------
  int32_t* perm_out = a.perm + s * a.sP;
  for (int p = tid; p < 2 * Wp; p += blockDim.x) perm_out[p] = perm[p];
  if (a.has_next) {
    const double* V = SV + (int64_t)Wp * Wp;
    auto Rval = [&](int p, int c) -> double {
      if (p < Wp) return c < Wp ? V[(int64_t)c * Wp + p] : 0.0;
      return NX[(int64_t)(Wp + c) * Wp + (p - Wp)];  // [D | Usup] columns Wp..3Wp-1 of NX
    };
    double* bsel = a.bsel + s * a.sScr;
    double* r1 = a.r1 + s * a.sScr;
    double* r2 = a.sv_out + s * a.sSV;
    for (int idx = tid; idx < Wp * Wp; idx += blockDim.x) {
      const int j = idx / Wp, i = idx % Wp;
      bsel[idx] = Pval(perm[Wp + i], j);
    }
    for (int idx = tid; idx < 2 * Wp * Wp; idx += blockDim.x) {
      const int c = idx / Wp, i = idx % Wp;
      r1[idx] = Rval(perm[i], c);
      r2[idx] = Rval(perm[Wp + i], c);
    }
  }
  // A11 = pivot-ordered top rows of the original panel, row-major in win
  for (int idx = tid; idx < Wp * Wp; idx += blockDim.x) {
    const int j = idx / Wp, i = idx % Wp;
    win[i * RS + j] = Pval(perm[i], j);
  }
  __syncthreads();

  // ---- phase 2: in-place Gauss-Jordan inverse of A11 (pivots known) -------------
  for (int k = 0; k < Wp; k++) {
    const double piv = win[k * RS + k];
    const double ip = piv != 0.0 ? 1.0 / piv : 0.0;
    if (piv == 0.0 && tid == 0) s_sing = 1;
    if (tid < Wp) fcol[tid] = tid == k ? 0.0 : win[tid * RS + k];
    else if (tid < 2 * Wp) {
      const int j = tid - Wp;
      prow[j] = (j == k ? 1.0 : win[k * RS + j]) * ip;
    }
    __syncthreads();
    for (int i = warp; i < Wp; i += nwarps) {
      double* row = win + i * RS;
      if (i == k) {
        for (int j = lane; j < Wp; j += 32) row[j] = prow[j];
      } else {
        const double f = fcol[i];
        for (int j = lane; j < Wp; j += 32) {
          const double base = j == k ? 0.0 : row[j];
          row[j] = fma(-f, prow[j], base);
        }
      }
    }
    __syncthreads();
  }
  double* ainv = a.ainv + s * a.sF;
  for (int idx = tid; idx < Wp * Wp; idx += blockDim.x) {
    const int j = idx / Wp, i = idx % Wp;
    ainv[idx] = win[i * RS + j];
  }
  if (tid == 0 && s_sing) {
    atomicOr(&a.status->flags, ERR_SINGULAR);
    atomicMin(&a.status->singular_strip, s);
  }
}

}  // namespace

void extract_levels(cudaStream_t st, CsrDev A, const StripDesc* strips, int nstrips, int64_t n2,
                    int Wp, int64_t L0, int64_t nl, double* nx, int64_t sNX, DevStatus* status) {
  if (nl <= 0) return;
  extract_levels_kernel<<<dim3((unsigned)nl, (unsigned)nstrips), 128, 0, st>>>(A, strips, n2, Wp, L0,
                                                                            nx, sNX, status);
  SLB_CUDA_CHECK(cudaGetLastError());
}

void extract_couplings(cudaStream_t st, CsrDev A, const StripDesc* strips, int nstrips, int64_t n2,
                       int Wp, double* cpl, int64_t sCPL, int32_t* sym, DevStatus* status) {
  dim3 block(32, 8);
  dim3 grid((unsigned)cdiv(n2, 8), (unsigned)nstrips);
  extract_couplings_kernel<<<grid, block, 0, st>>>(A, strips, n2, Wp, cpl, sCPL, sym, status);
  SLB_CUDA_CHECK(cudaGetLastError());
}

void init_sv(cudaStream_t st, int nstrips, int Wp, const double* nx0, int64_t sNX, double* sv,
             int64_t sSV) {
  init_sv_kernel<<<nstrips, 256, 0, st>>>(Wp, nx0, sNX, sv, sSV);
  SLB_CUDA_CHECK(cudaGetLastError());
}

void level_panel(cudaStream_t st, const LevelArgs& a) {
  const int Wp = a.Wp;
  const size_t smem = (size_t)((Wp + 1) * (Wp + 1) + 2 * (Wp + 1)) * sizeof(double) + 2 * Wp * sizeof(int);
  static size_t attr = 0;
  if (smem > attr) {
    SLB_CUDA_CHECK(cudaFuncSetAttribute(level_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  level_panel_kernel<<<a.nstrips, 1024, smem, st>>>(a);
  SLB_CUDA_CHECK(cudaGetLastError());
}

}  // namespace slb

// ---------------------------------------------------------------------------
// Pack one level's col-major factors into the DMMA fragment order used by
// the sweeps (schur.cu, solve.cu).  Per level (4 Wp^2 doubles):
//   F = [Ainv ; Fbot]  (2Wp x Wp):  [k4 step][m8 tile][lane]  (lane = 4g + t -> F[8mt+g][4ks+t])
//   H                  (Wp x 2Wp):  same order, at offset 2 Wp^2
namespace slb {
namespace {
__global__ void pack_level_kernel(int Wp, const double* ainv, const double* fbot, const double* h,
                                  int64_t sScr, double* out, int64_t sF) {
  const int s = blockIdx.y;
  const double* A0 = ainv + s * sScr;
  const double* F1 = fbot + s * sScr;
  const double* H = h + s * sScr;
  double* o = out + s * sF;
  const int64_t nF = 2LL * Wp * Wp;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < 2 * nF;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int lane = (int)(idx & 31);
    const int g = lane >> 2, t = lane & 3;
    if (idx < nF) {
      const int64_t q = idx >> 5;
      const int MT = 2 * Wp / 8;
      const int mt = (int)(q % MT), ks = (int)(q / MT);
      const int m = mt * 8 + g, k = ks * 4 + t;
      o[idx] = m < Wp ? A0[(int64_t)k * Wp + m] : F1[(int64_t)k * Wp + (m - Wp)];
    } else {
      const int64_t q = (idx - nF) >> 5;
      const int MT = Wp / 8;
      const int mt = (int)(q % MT), ks = (int)(q / MT);
      const int m = mt * 8 + g, k = ks * 4 + t;
      o[idx] = H[(int64_t)k * Wp + m];
    }
  }
}
}  // namespace

void pack_level(cudaStream_t st, int nstrips, int Wp, const double* ainv, const double* fbot,
                const double* h, int64_t sScr, double* out, int64_t sF) {
  const int64_t total = 4LL * Wp * Wp;
  dim3 grid((unsigned)std::min<int64_t>(cdiv(total, 256), 64), (unsigned)nstrips);
  pack_level_kernel<<<grid, 256, 0, st>>>(Wp, ainv, fbot, h, sScr, out, sF);
  SLB_CUDA_CHECK(cudaGetLastError());
}
}  // namespace slb
