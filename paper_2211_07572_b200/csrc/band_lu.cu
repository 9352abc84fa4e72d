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
//   panel  perm_l [S_l ; Lsub_{l+1}] = [L11 ; L21] U11   (window pivots, 2Wp x Wp)
//   R = perm_l [V_l 0 ; D_{l+1} Usup_{l+1}] = [R1 ; R2]
//   U1213 = L11^{-1} R1,  [S_{l+1} | V_{l+1}] = R2 - L21 U1213      (the chain)
// and, after the chain, for every level in parallel (convert_levels):
//   Ainv_l = U11^{-1} L11^{-1},  Fbot_l = -L21 L11^{-1},  H_l = U11^{-1} U1213
//
// so that A_ii^{-1} b is the pure-GEMM sweep
//   forward  t = perm_l [z_l ; b_{l+1}],  y_l = Ainv_l t_top,  z_{l+1} = t_bot + Fbot_l t_top
//   backward x_l = y_l - H_l [x_{l+1} ; x_{l+2}]
// used by the Schur kernel (schur.cu) and the solves (solve.cu).
#include <climits>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace slb {
namespace {

__device__ __forceinline__ void raise(DevStatus* st, int32_t bit) { atomicOr(&st->flags, bit); }

// ---------------------------------------------------------------------------
// Level blocks [Lsub | D | Usup] of one strip level from the CSR.
// grid (nl, nstrips), block 128.
__global__ void extract_levels_kernel(CsrDev A, const StripDesc* strips, int64_t n2, int Wp,
                                      int64_t L0, double* nx, int64_t sNX, DevStatus* status, double* dsub,
                                      uint8_t* lnd) {
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
        if (dy == -1) {
          if (cx == ix) dsub[((int64_t)s * n2 + L - 1) * Wp + ix] = v;
          else if (v != 0.0) lnd[(int64_t)s * n2 + L] = 1;
        } else if (dy == 1 && cx != ix && v != 0.0) {
          lnd[((int64_t)gridDim.y + s) * n2 + L] = 1;  // second plane: Usup_L not diagonal
        }
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
// One level step for every strip: LU with partial pivoting of the panel
// P_l = [S_l ; Lsub_{l+1}] (2Wp x Wp) restricted to dgbtrf's window (rows
// k..k+Wp at column k), blocked by 8 columns:
//   (a) warp 0 factors the 8-column panel (pivot search, swaps, multipliers),
//   (b) all threads apply its 8 row swaps to the other columns,
//   (c) U block = L_bb^{-1} (pivot rows, trailing columns),
//   (d) rank-8 trailing update of the window on the DMMA pipe,
//   (e) the 8 finished rows retire to LU11, 8 bottom rows enter.
// The window is a circular buffer of Wp+8 rows in shared memory.
// Outputs into the level slot (LU form, converted later by convert_levels):
//   LU11 (row-major Wp x Wp: unit-lower multipliers + U11), L21 (row-major),
//   U1213 <- R1 = top rows of perm_l [V_l 0 ; D_{l+1} Usup_{l+1}] (col-major Wp x 2Wp),
// and sv_out <- R2 = bottom rows.  The chain then forms
//   U1213 = L11^{-1} R1 (trsm_small_batched) and [S|V]_{l+1} = R2 - L21 U1213 (GEMM).
// grid = nstrips, block = 512.
template <int PW>  // warps factoring the 8-column panel (1 or 4; 4 is used)
__global__ void __launch_bounds__(512) level_lu_kernel(LevelArgs a) {
  extern __shared__ double smem[];
  const int Wp = a.Wp, NW = Wp + 8;
  const int RS = ((Wp + 15) / 16) * 16 + 4;  // row stride = 4 mod 16 doubles
  double* win = smem;                        // NW * RS
  int* perm = reinterpret_cast<int*>(win + NW * RS + 32 + 8 * Wp);  // 2 Wp (after panel scratch + entering rows)
  __shared__ int s_sing;
  __shared__ int s_piv[8];

  const int s = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const double* SV = a.sv_in + s * a.sSV;
  const double* NX = a.has_next ? a.nx + s * a.sNX : nullptr;
  double* slot = a.slot + s * a.sF;
  double* LU11 = slot;
  double* L21 = slot + (int64_t)Wp * Wp;
  double* U1213 = slot + 2LL * Wp * Wp;
  const int rows_total = a.has_next ? 2 * Wp : Wp;
  auto rowp = [&](int pos) -> double* { return win + (pos < NW ? pos : pos - NW) * RS; };
  auto Pval = [&](int p, int j) -> double {
    return p < Wp ? SV[(int64_t)j * Wp + p] : NX[(int64_t)j * Wp + (p - Wp)];
  };
  if (tid == 0) s_sing = -1;

  const int init_rows = rows_total < NW ? rows_total : NW;
  // the window's first rows: asynchronous 8-byte copies (transposing gather), so every thread has
  // many loads in flight instead of one load-store pair at a time
  const float inv_ir = 1.0f / (float)init_rows, inv_wp = 1.0f / (float)Wp;
  for (int idx = tid; idx < init_rows * Wp; idx += blockDim.x) {
    const int j = qdiv(idx, inv_ir), p = idx - j * init_rows;
    cp_async8(rowp(p) + j, p < Wp ? SV + (int64_t)j * Wp + p : NX + (int64_t)j * Wp + (p - Wp), true);
  }
  cp_async_commit();
  for (int p = tid; p < 2 * Wp; p += blockDim.x) perm[p] = p;
  __syncthreads();

  double* ent = win + NW * RS + 32;  // 8 x Wp staging for the entering rows
#ifdef SLB_LU_PROF
  long long L0 = clock64(), lp[6] = {0, 0, 0, 0, 0, 0};
#define LP(k_) { const long long q_ = clock64(); lp[k_] += q_ - L0; L0 = q_; }
#else
#define LP(k_)
#endif
#ifdef SLB_PANEL8_PROF
  long long pq[5] = {0, 0, 0, 0, 0};
#endif
  for (int kb = 0; kb < Wp; kb += 8) {
    const int kend = kb + 8;
    // prefetch the 8 bottom rows entering after this block (overlaps (a)-(d))
    for (int idx = tid; idx < 8 * Wp; idx += blockDim.x) {
      const int q = idx / Wp, j = idx % Wp;
      const int pe = kend + Wp + q;
      if (pe < rows_total) cp_async8(ent + idx, NX + (int64_t)j * Wp + (pe - Wp), true);
    }
    cp_async_commit();
    // (a) panel factorization by warps 0-3 (128 threads) with the panel in
    //     registers: thread p owns the rows initially at positions
    //     kb + p + 128 i (i < 2), 8 panel columns each.  Interchanges only
    //     update each row's position register (pos); the data move happens
    //     once, when the panel is written back.  Two named barriers per column.
    if (warp < PW) {
      constexpr int NT = PW * 32;                  // panel threads
      constexpr int RPL = PW == 1 ? 5 : 2;         // rows per thread (Wp + 8 <= NT * RPL)
      const int pt = tid;
      const int rlast = min(kb + 7 + Wp, rows_total - 1);
      double v[RPL][8];
      int pos[RPL];
#pragma unroll
      for (int i = 0; i < RPL; i++) {
        pos[i] = kb + pt + NT * i;
        if (pos[i] <= rlast) {
          const double* row = rowp(pos[i]);
#pragma unroll
          for (int q = 0; q < 8; q++) v[i][q] = row[kb + q];
        } else {
          pos[i] = 0x3fffffff;  // inactive
#pragma unroll
          for (int q = 0; q < 8; q++) v[i][q] = 0.0;
        }
      }
      double* pcand = win + NW * RS;  // scratch: [2][4] (value) + [2][4] (pos as double) + [2][8] (pivot row)
#ifdef SLB_PANEL8_PROF
      long long Q0 = clock64();
#define QP(k_) { const long long q_ = clock64(); pq[k_] += q_ - Q0; Q0 = q_; }
#else
#define QP(k_)
#endif
      auto panel_sync = [&]() {
        if (PW == 1) __syncwarp();
        else asm volatile("bar.sync 1, %0;\n" ::"n"(NT) : "memory");
      };
#pragma unroll
      for (int q = 0; q < 8; q++) {
        const int c = kb + q, par = q & 1;
        const int hi = min(c + Wp, rows_total - 1);
        double best = 0.0;
        int bpos = 0x7fffffff;
#pragma unroll
        for (int i = 0; i < RPL; i++) {
          const double av = fabs(v[i][q]);
          if (pos[i] >= c && pos[i] <= hi && (av > best || (av == best && pos[i] < bpos))) {
            best = av;
            bpos = pos[i];
          }
        }
        // warp arg-max with hardware reductions: non-negative doubles order like their bit
        // patterns, so max(hi word), then max(lo word) among those lanes, then the smallest
        // position among exact maxima (dgbtrf's first-max rule)
        const unsigned long long key = (unsigned long long)__double_as_longlong(best);
        const unsigned khi = (unsigned)(key >> 32), klo = (unsigned)key;
        const unsigned mhi = __reduce_max_sync(0xffffffffu, khi);
        const unsigned mlo = __reduce_max_sync(0xffffffffu, khi == mhi ? klo : 0u);
        const bool ismax = khi == mhi && klo == mlo;
        const int rw = (int)__reduce_min_sync(0xffffffffu, ismax ? (unsigned)bpos : 0x7fffffffu);
        const double mx = __longlong_as_double((long long)(((unsigned long long)mhi << 32) | mlo));
        QP(0)
        double gm = mx;
        int r = rw;
        if (PW > 1) {  // combine the warps' candidates through shared memory
          if (lane == 0) {
            pcand[par * 4 + warp] = mx;
            pcand[8 + par * 4 + warp] = (double)rw;
          }
          panel_sync();
          gm = pcand[par * 4];
          r = (int)pcand[8 + par * 4];
#pragma unroll
          for (int w2 = 1; w2 < PW; w2++) {
            const double cv = pcand[par * 4 + w2];
            const int cr = (int)pcand[8 + par * 4 + w2];
            if (cv > gm || (cv == gm && cr < r)) {
              gm = cv;
              r = cr;
            }
          }
        }
        QP(1)
        if (!(gm > 0.0)) {
          r = c;
          if (pt == 0 && s_sing < 0) s_sing = c;  // first zero pivot column of this level
        }
        // the winner publishes its row; positions c and r exchange
#pragma unroll
        for (int i = 0; i < RPL; i++)
          if (pos[i] == r)
#pragma unroll
            for (int qq = 0; qq < 8; qq++) pcand[16 + par * 8 + qq] = v[i][qq];
#pragma unroll
        for (int i = 0; i < RPL; i++) {
          if (pos[i] == r) pos[i] = c;
          else if (pos[i] == c) pos[i] = r;
        }
        if (pt == 0) s_piv[q] = r;  // perm is updated after the panel (off the critical path)
        QP(2)
        panel_sync();
        QP(3)
        double pr[8];
#pragma unroll
        for (int qq = 0; qq < 8; qq++) pr[qq] = pcand[16 + par * 8 + qq];
        const double inv = pr[q] != 0.0 ? __drcp_rn(pr[q]) : 0.0;
#pragma unroll
        for (int i = 0; i < RPL; i++) {
          if (pos[i] > c && pos[i] <= hi) {
            const double m = v[i][q] * inv;
            v[i][q] = m;
#pragma unroll
            for (int qq = q + 1; qq < 8; qq++) v[i][qq] = fma(-m, pr[qq], v[i][qq]);
          }
        }
        QP(4)
      }
#pragma unroll
      for (int i = 0; i < RPL; i++) {
        if (pos[i] <= rlast) {
          double* row = rowp(pos[i]);
#pragma unroll
          for (int q = 0; q < 8; q++) row[kb + q] = v[i][q];
        }
      }
    }
    __syncthreads();
    LP(0)
    // pivot-order bookkeeping for the panel (one thread, beside the swaps)
    if (tid == blockDim.x - 1)
      for (int q = 0; q < 8; q++) {
        const int c = kb + q, r = s_piv[q];
        if (r != c) {
          const int tp = perm[c];
          perm[c] = perm[r];
          perm[r] = tp;
        }
      }
    // (b) the panel's row swaps on all other columns, in pivot order
    for (int jj = tid; jj < Wp - 8; jj += blockDim.x) {
      const int col = jj < kb ? jj : jj + 8;
#pragma unroll
      for (int q = 0; q < 8; q++) {
        const int c = kb + q, r = s_piv[q];
        if (r != c) {
          double* rc = rowp(c);
          double* rr = rowp(r);
          const double tv = rc[col];
          rc[col] = rr[col];
          rr[col] = tv;
        }
      }
    }
    __syncthreads();
    LP(1)
    // (c) U block: pivot rows kb..kb+7 on the trailing columns, U = L_bb^{-1} A
    for (int j = kend + tid; j < Wp; j += blockDim.x) {
      double u[8];
#pragma unroll
      for (int q = 0; q < 8; q++) u[q] = rowp(kb + q)[j];
#pragma unroll
      for (int q = 1; q < 8; q++) {
        const double* lq = rowp(kb + q);
#pragma unroll
        for (int p = 0; p < 8; p++)
          if (p < q) u[q] = fma(-lq[kb + p], u[p], u[q]);
      }
#pragma unroll
      for (int q = 1; q < 8; q++) rowp(kb + q)[j] = u[q];
    }
    __syncthreads();
    LP(2)
    // (d) trailing update on the DMMA pipe: rows kend..kb+7+Wp, cols kend..Wp-1.
    //     A warp owns m tiles (8 rows) and sweeps the n tiles; its A fragments
    //     (the 8 multipliers of each row) are loaded once.
    {
      const int rlast = min(kb + 7 + Wp, rows_total - 1);
      const int mt_n = (rlast - kend + 1 + 7) / 8;
      const int nt_n = (Wp - kend) / 8;
      const double* u0 = rowp(kb + t);
      const double* u1 = rowp(kb + 4 + t);
      // units = (m tile, half of the n tiles): 2 mt_n units over the warps (whole rows per warp
      // left a few warps with twice the work)
      const int nh = (nt_n + 1) / 2;
      for (int unit = warp; unit < 2 * mt_n; unit += nwarps) {
        const int mi = unit >> 1;
        const int nbeg = (unit & 1) * nh, nend = min(nt_n, nbeg + nh);
        const int p = kend + mi * 8 + g;
        const bool ok = p <= rlast;
        double* row = rowp(ok ? p : kend);
        const double a0 = ok ? -row[kb + t] : 0.0, a1 = ok ? -row[kb + 4 + t] : 0.0;
        // four n tiles per step: their loads issue together, the DMMA chains interleave
        int ni = nbeg;
        for (; ni + 4 <= nend; ni += 4) {
          double b0[4], b1[4], d0[4], d1[4];
#pragma unroll
          for (int u = 0; u < 4; u++) {
            const int c0 = kend + (ni + u) * 8;
            b0[u] = u0[c0 + g];
            b1[u] = u1[c0 + g];
            d0[u] = row[c0 + 2 * t];
            d1[u] = row[c0 + 2 * t + 1];
          }
#pragma unroll
          for (int u = 0; u < 4; u++) {
            dmma884(d0[u], d1[u], a0, b0[u]);
            dmma884(d0[u], d1[u], a1, b1[u]);
          }
          if (ok) {
#pragma unroll
            for (int u = 0; u < 4; u++) {
              const int c0 = kend + (ni + u) * 8;
              row[c0 + 2 * t] = d0[u];
              row[c0 + 2 * t + 1] = d1[u];
            }
          }
        }
        for (; ni < nend; ni++) {
          const int c0 = kend + ni * 8;
          const double b0 = u0[c0 + g], b1 = u1[c0 + g];
          double d0 = row[c0 + 2 * t], d1 = row[c0 + 2 * t + 1];
          dmma884(d0, d1, a0, b0);
          dmma884(d0, d1, a1, b1);
          if (ok) {
            row[c0 + 2 * t] = d0;
            row[c0 + 2 * t + 1] = d1;
          }
        }
      }
    }
    __syncthreads();
    LP(3)
    // (e) retire positions kb..kb+7; bottom rows kend..kend+7 enter at positions kend+Wp..
    cp_async_wait<0>();
    for (int idx = tid; idx < 8 * Wp; idx += blockDim.x) {
      const int q = idx / Wp, j = idx % Wp;
      double* rr = rowp(kb + q);
      LU11[(int64_t)(kb + q) * Wp + j] = rr[j];
      const int pe = kend + Wp + q;
      if (pe < rows_total) rr[j] = ent[idx];
    }
    __syncthreads();
    LP(4)
  }
#ifdef SLB_LU_PROF
  if (tid == 0 && s == 0 && (a.level % 1000) == 1)
    printf("LEVEL_LU l=%d: panel %lld swap %lld ublock %lld trailing %lld retire %lld (cycles)\n", a.level, lp[0], lp[1],
           lp[2], lp[3], lp[4]);
#endif

#ifdef SLB_PANEL8_PROF
  if (tid == 0 && s == 0 && (a.level % 1000) == 1)
    printf("PANEL8 l=%d: argmax %lld bar1 %lld resolve %lld bar2 %lld update %lld (cycles, %d columns)\n", a.level,
           pq[0], pq[1], pq[2], pq[3], pq[4], Wp);
#endif
  int32_t* perm_out = a.perm + s * a.sP;
  for (int p = tid; p < 2 * Wp; p += blockDim.x) perm_out[p] = perm[p];
  {
    // U13 != 0 iff a row of level l+1 was pivoted into the top half
    // bits: 0 U13 != 0, 1 Lsub_{l+1} not diagonal, 2..5 rows of level l+1 pivoted up (15 = more)
    const int nup = __syncthreads_count(tid < Wp && perm[tid] >= Wp);
    const int nd = a.has_next ? a.lnd[s * a.sU13] : 0;
    const int ud = a.has_next ? a.lnd[(a.nstrips + s) * a.sU13] : 0;
    // bit 6: Usup_{l+1} not diagonal (the x_{l+2} half of H is then not confined to the
    // columns of the rows pivoted up)
    if (tid == 0)
      a.u13[s * a.sU13] = (uint8_t)((nup ? 1 : 0) | (nd ? 2 : 0) | (min(nup, 15) << 2) | (ud ? 64 : 0));
  }
  if (a.has_next) {
    for (int idx = tid; idx < Wp * Wp; idx += blockDim.x) {
      const int i = idx / Wp, j = idx % Wp;
      L21[idx] = rowp(Wp + i)[j];
    }
  } else {
    for (int idx = tid; idx < 3 * Wp * Wp; idx += blockDim.x) L21[idx] = 0.0;  // L21 and U1213
  }
  if (tid == 0 && s_sing >= 0) {
    atomicOr(&a.status->flags, ERR_SINGULAR);
    atomicMin(&a.status->singular_strip, s);
    if (a.nstrips == 1) atomicMin(&a.status->singular_pos, a.level * Wp + s_sing);  // single-slab path
  }
}

// Look-ahead form of level_lu_kernel (same arithmetic and outputs).  Per 8-column block kb:
//   X  trailing update of block kb on the next panel's 8 columns (all warps)
//   Y  warps 0-3 factor panel kb+8 (its entering rows read from the staging buffer) while
//      warps 4-15 finish the trailing update of block kb on the remaining columns
//   R  rows kb..kb+7 retire to LU11, the entering rows take their physical rows
//   S  panel kb+8's interchanges on the other columns;  U  its U block
// so the serial pivot search of panel kb+8 runs beside the DMMA update of block kb.
template <int PW>  // warps factoring the panel: 4 (two rows per lane) or 2 (three rows per lane)
__global__ void __launch_bounds__(512) level_lu_la_kernel(LevelArgs a) {
  extern __shared__ double smem[];
  const int Wp = a.Wp, NW = Wp + 8;
  const int RS = ((Wp + 15) / 16) * 16 + 4;
  double* win = smem;
  double* pcand = win + NW * RS;  // [2][4] values, [2][4] positions, [2][8] pivot rows
  double* ent = pcand + 32;       // [2][8 x Wp] entering rows
  int* perm = reinterpret_cast<int*>(ent + 16 * Wp);
  __shared__ int s_sing;
  __shared__ int s_piv[8];
  constexpr int NT = PW * 32, RPL = PW == 4 ? 2 : 3;  // NT * RPL >= Wp + 8 (Wp <= 160)

  const int s = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const double* SV = a.sv_in + s * a.sSV;
  const double* NX = a.has_next ? a.nx + s * a.sNX : nullptr;
  double* slot = a.slot + s * a.sF;
  double* LU11 = slot;
  double* L21 = slot + (int64_t)Wp * Wp;
  const int rows_total = a.has_next ? 2 * Wp : Wp;
  auto rowp = [&](int pos) -> double* { return win + (pos < NW ? pos : pos - NW) * RS; };
  auto Pval = [&](int p, int j) -> double {
    return p < Wp ? SV[(int64_t)j * Wp + p] : NX[(int64_t)j * Wp + (p - Wp)];
  };
  if (tid == 0) s_sing = -1;
  const int init_rows = rows_total < NW ? rows_total : NW;
  // the window's first rows: asynchronous 8-byte copies (transposing gather), so every thread has
  // many loads in flight instead of one load-store pair at a time.  The rows of level l + 1 (NX,
  // extracted long before) are requested before the wait for the previous level's update (PDL).
  const float inv_wp = 1.0f / (float)Wp;
  if (init_rows > Wp) {
    const int nxr = init_rows - Wp;
    const float inv_n = 1.0f / (float)nxr;
    for (int idx = tid; idx < nxr * Wp; idx += blockDim.x) {
      const int j = qdiv(idx, inv_n), p = idx - j * nxr;
      cp_async8(rowp(Wp + p) + j, NX + (int64_t)j * Wp + p, true);
    }
  }
  pdl_wait();
  for (int idx = tid; idx < Wp * Wp; idx += blockDim.x) {
    const int j = qdiv(idx, inv_wp), p = idx - j * Wp;
    cp_async8(rowp(p) + j, SV + (int64_t)j * Wp + p, true);
  }
  cp_async_commit();
  for (int p = tid; p < 2 * Wp; p += blockDim.x) perm[p] = p;

  auto prefetch = [&](int kb_in, int buf) {  // rows entering at positions kb_in + Wp + q
    for (int idx = tid; idx < 8 * Wp; idx += blockDim.x) {
      const int q = qdiv(idx, inv_wp), j = idx - q * Wp;
      const int pe = kb_in + Wp + q;
      if (pe < rows_total) cp_async8(ent + buf * 8 * Wp + idx, NX + (int64_t)j * Wp + (pe - Wp), true);
    }
    cp_async_commit();
  };
  // panel [kb, kb+8) on warps 0..PW-1; rows at positions >= kb + Wp live in entp (if given)
  auto panel = [&](int kb, double* entp) {
    const int pt = tid;
    const int rlast = min(kb + 7 + Wp, rows_total - 1);
    auto rowsrc = [&](int P) -> double* { return (entp && P >= kb + Wp) ? entp + (P - kb - Wp) * Wp : rowp(P); };
    double v[RPL][8];
    int pos[RPL];
#pragma unroll
    for (int i = 0; i < RPL; i++) {
      pos[i] = kb + pt + NT * i;
      if (pos[i] <= rlast) {
        const double* row = rowsrc(pos[i]);
#pragma unroll
        for (int q = 0; q < 8; q++) v[i][q] = row[kb + q];
      } else {
        pos[i] = 0x3fffffff;
#pragma unroll
        for (int q = 0; q < 8; q++) v[i][q] = 0.0;
      }
    }
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const int c = kb + q, par = q & 1;
      const int hi = min(c + Wp, rows_total - 1);
      double best = 0.0;
      int bpos = 0x7fffffff;
#pragma unroll
      for (int i = 0; i < RPL; i++) {
        const double av = fabs(v[i][q]);
        if (pos[i] >= c && pos[i] <= hi && (av > best || (av == best && pos[i] < bpos))) {
          best = av;
          bpos = pos[i];
        }
      }
      const unsigned long long key = (unsigned long long)__double_as_longlong(best);
      const unsigned khi = (unsigned)(key >> 32), klo = (unsigned)key;
      const unsigned mhi = __reduce_max_sync(0xffffffffu, khi);
      const unsigned mlo = __reduce_max_sync(0xffffffffu, khi == mhi ? klo : 0u);
      const bool ismax = khi == mhi && klo == mlo;
      const int rw = (int)__reduce_min_sync(0xffffffffu, ismax ? (unsigned)bpos : 0x7fffffffu);
      const double mx = __longlong_as_double((long long)(((unsigned long long)mhi << 32) | mlo));
      if (lane == 0) {
        pcand[par * 4 + warp] = mx;
        pcand[8 + par * 4 + warp] = (double)rw;
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(NT) : "memory");
      double gm = pcand[par * 4];
      int r = (int)pcand[8 + par * 4];
#pragma unroll
      for (int w2 = 1; w2 < PW; w2++) {
        const double cv = pcand[par * 4 + w2];
        const int cr = (int)pcand[8 + par * 4 + w2];
        if (cv > gm || (cv == gm && cr < r)) {
          gm = cv;
          r = cr;
        }
      }
      if (!(gm > 0.0)) {
        r = c;
        if (pt == 0 && s_sing < 0) s_sing = c;  // first zero pivot column of this level
      }
#pragma unroll
      for (int i = 0; i < RPL; i++)
        if (pos[i] == r)
#pragma unroll
          for (int qq = 0; qq < 8; qq++) pcand[16 + par * 8 + qq] = v[i][qq];
#pragma unroll
      for (int i = 0; i < RPL; i++) {
        if (pos[i] == r) pos[i] = c;
        else if (pos[i] == c) pos[i] = r;
      }
      if (pt == 0) s_piv[q] = r;
      asm volatile("bar.sync 1, %0;\n" ::"n"(NT) : "memory");
      double pr[8];
#pragma unroll
      for (int qq = 0; qq < 8; qq++) pr[qq] = pcand[16 + par * 8 + qq];
      const double inv = pr[q] != 0.0 ? __drcp_rn(pr[q]) : 0.0;
#pragma unroll
      for (int i = 0; i < RPL; i++) {
        if (pos[i] > c && pos[i] <= hi) {
          const double m = v[i][q] * inv;
          v[i][q] = m;
#pragma unroll
          for (int qq = q + 1; qq < 8; qq++) v[i][qq] = fma(-m, pr[qq], v[i][qq]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < RPL; i++) {
      if (pos[i] <= rlast) {
        double* row = rowsrc(pos[i]);
#pragma unroll
        for (int q = 0; q < 8; q++) row[kb + q] = v[i][q];
      }
    }
  };
  auto swaps = [&](int kb) {  // panel kb's interchanges on the other columns; pivot-order bookkeeping
    if (tid == blockDim.x - 1)
      for (int q = 0; q < 8; q++) {
        const int c = kb + q, r = s_piv[q];
        if (r != c) {
          const int tp = perm[c];
          perm[c] = perm[r];
          perm[r] = tp;
        }
      }
    for (int jj = tid; jj < Wp - 8; jj += blockDim.x) {
      const int col = jj < kb ? jj : jj + 8;
#pragma unroll
      for (int q = 0; q < 8; q++) {
        const int c = kb + q, r = s_piv[q];
        if (r != c) {
          double* rc = rowp(c);
          double* rr = rowp(r);
          const double tv = rc[col];
          rc[col] = rr[col];
          rr[col] = tv;
        }
      }
    }
  };
  auto ublock = [&](int kb) {
    for (int j = kb + 8 + tid; j < Wp; j += blockDim.x) {
      double u[8];
#pragma unroll
      for (int q = 0; q < 8; q++) u[q] = rowp(kb + q)[j];
#pragma unroll
      for (int q = 1; q < 8; q++) {
        const double* lq = rowp(kb + q);
#pragma unroll
        for (int p = 0; p < 8; p++)
          if (p < q) u[q] = fma(-lq[kb + p], u[p], u[q]);
      }
#pragma unroll
      for (int q = 1; q < 8; q++) rowp(kb + q)[j] = u[q];
    }
  };
  // rank-8 update of block kb on columns [c0, c1), rows kb+8..kb+7+Wp, by warps w0, w0+1, ...
  auto trailing = [&](int kb, int c0, int c1, int w0, int nw) {
    if (c1 <= c0 || warp < w0) return;
    const int kend = kb + 8;
    const int rlast = min(kb + 7 + Wp, rows_total - 1);
    const int mt_n = (rlast - kend + 1 + 7) / 8;
    const int nt_n = (c1 - c0) / 8;
    const double* u0 = rowp(kb + t);
    const double* u1 = rowp(kb + 4 + t);
    const int nh = (nt_n + 1) / 2;
    for (int unit = warp - w0; unit < 2 * mt_n; unit += nw) {
      const int mi = unit >> 1;
      const int nbeg = (unit & 1) * nh, nend = min(nt_n, nbeg + nh);
      const int p = kend + mi * 8 + g;
      const bool ok = p <= rlast;
      double* row = rowp(ok ? p : kend);
      const double a0 = ok ? -row[kb + t] : 0.0, a1 = ok ? -row[kb + 4 + t] : 0.0;
      int ni = nbeg;
      for (; ni + 4 <= nend; ni += 4) {
        double b0[4], b1[4], d0[4], d1[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int cc = c0 + (ni + u) * 8;
          b0[u] = u0[cc + g];
          b1[u] = u1[cc + g];
          d0[u] = row[cc + 2 * t];
          d1[u] = row[cc + 2 * t + 1];
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
          dmma884(d0[u], d1[u], a0, b0[u]);
          dmma884(d0[u], d1[u], a1, b1[u]);
        }
        if (ok) {
#pragma unroll
          for (int u = 0; u < 4; u++) {
            const int cc = c0 + (ni + u) * 8;
            row[cc + 2 * t] = d0[u];
            row[cc + 2 * t + 1] = d1[u];
          }
        }
      }
      for (; ni < nend; ni++) {
        const int cc = c0 + ni * 8;
        const double b0 = u0[cc + g], b1 = u1[cc + g];
        double d0 = row[cc + 2 * t], d1 = row[cc + 2 * t + 1];
        dmma884(d0, d1, a0, b0);
        dmma884(d0, d1, a1, b1);
        if (ok) {
          row[cc + 2 * t] = d0;
          row[cc + 2 * t + 1] = d1;
        }
      }
    }
  };

#ifdef SLB_LU_PROF
  long long Q0 = clock64(), lq[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define LQ(k_) { const long long q_ = clock64(); lq[k_] += q_ - Q0; Q0 = q_; }
#else
#define LQ(k_)
#endif
  if (8 < Wp) {
    prefetch(8, 0);
    cp_async_wait<1>();  // the window (the entering rows of block 8 may still be in flight)
  } else {
    cp_async_wait<0>();
  }
  __syncthreads();
  LQ(0)
  if (warp < PW) panel(0, nullptr);  // block 0: every row is in the window
  __syncthreads();
  swaps(0);
  __syncthreads();
  ublock(0);
  __syncthreads();
  LQ(1)
  int eb = 0;
  // first warp of the trailing update beside the panel: 8 of the 12 non-panel warps suffice
  // (trailing ~81k vs panel ~147k cycles per level) and leave the panel warps more issue slots
  // on their SMSPs: cfg3 chain 0.823 -> 0.816 s; with two panel warps, 10 trailing warps
  // (SLB_LU_TW0 overrides, measurement)
  const int tw0 = a.tw0 > PW ? a.tw0 : (PW == 2 ? 6 : 8);
  for (int kb = 0; kb < Wp; kb += 8) {
    const int kend = kb + 8;
    const bool more = kend < Wp;
    if (more) trailing(kb, kend, kend + 8, 0, nwarps);  // X
    cp_async_wait<0>();
    __syncthreads();
    LQ(2)
    if (warp < PW) {  // Y
      if (more) panel(kend, ent + eb * 8 * Wp);
    } else if (warp >= tw0) {
      trailing(kb, more ? kend + 8 : kend, Wp, tw0, nwarps - tw0);
    }
    LQ(3)
    __syncthreads();
    LQ(4)
    if (more && kend + 8 < Wp) prefetch(kend + 8, eb ^ 1);
    // R, S and U fused per column (one thread per column, no barrier between them): rows
    // kb..kb+7 retire and the entering rows take their slots (R); panel kend's interchanges (S)
    // and its U block (U) on the column.  Column j touches only column j of the window, and
    // reads the panel's L values, final since the barrier above.
    if (more && tid == blockDim.x - 1)
      for (int q = 0; q < 8; q++) {  // pivot-order bookkeeping of panel kend
        const int c = kend + q, r = s_piv[q];
        if (r != c) {
          const int tp = perm[c];
          perm[c] = perm[r];
          perm[r] = tp;
        }
      }
    for (int j = tid; j < Wp; j += blockDim.x) {
#pragma unroll
      for (int q = 0; q < 8; q++) {  // R
        double* rr = rowp(kb + q);
        LU11[(int64_t)(kb + q) * Wp + j] = rr[j];
        if (kend + Wp + q < rows_total) rr[j] = ent[eb * 8 * Wp + q * Wp + j];
      }
      if (!more || (j >= kend && j < kend + 8)) continue;
#pragma unroll
      for (int q = 0; q < 8; q++) {  // S
        const int c = kend + q, r = s_piv[q];
        if (r != c) {
          double* rc = rowp(c);
          double* rw = rowp(r);
          const double tv = rc[j];
          rc[j] = rw[j];
          rw[j] = tv;
        }
      }
      if (j < kend + 8) continue;
      double u[8];  // U
#pragma unroll
      for (int q = 0; q < 8; q++) u[q] = rowp(kend + q)[j];
#pragma unroll
      for (int q = 1; q < 8; q++) {
        const double* lq = rowp(kend + q);
#pragma unroll
        for (int p2 = 0; p2 < 8; p2++)
          if (p2 < q) u[q] = fma(-lq[kend + p2], u[p2], u[q]);
      }
#pragma unroll
      for (int q = 1; q < 8; q++) rowp(kend + q)[j] = u[q];
    }
    __syncthreads();
    LQ(5)
    LQ(6)
    eb ^= 1;
  }
#ifdef SLB_LU_PROF
  if ((tid == 0 || tid == 511) && s == 0 && (a.level % 1000) == 1)
    printf("LEVEL_LU_LA l=%d tid %d: prologue %lld block0 %lld X %lld Y %lld Ywait %lld R %lld SU %lld (cycles)\n", a.level,
           tid, lq[0], lq[1], lq[2], lq[3], lq[4], lq[5], lq[6]);
#endif

  pdl_trigger();  // the level update may start launching (it waits for this grid's completion)
  int32_t* perm_out = a.perm + s * a.sP;
  for (int p = tid; p < 2 * Wp; p += blockDim.x) perm_out[p] = perm[p];
  {
    const int nup = __syncthreads_count(tid < Wp && perm[tid] >= Wp);
    const int nd = a.has_next ? a.lnd[s * a.sU13] : 0;
    const int ud = a.has_next ? a.lnd[(a.nstrips + s) * a.sU13] : 0;
    if (tid == 0)
      a.u13[s * a.sU13] = (uint8_t)((nup ? 1 : 0) | (nd ? 2 : 0) | (min(nup, 15) << 2) | (ud ? 64 : 0));
  }
  if (a.has_next) {
    for (int idx = tid; idx < Wp * Wp; idx += blockDim.x) {
      const int i = idx / Wp, j = idx % Wp;
      L21[idx] = rowp(Wp + i)[j];
    }
  } else {
    for (int idx = tid; idx < 3 * Wp * Wp; idx += blockDim.x) L21[idx] = 0.0;  // L21 and U1213
  }
  if (tid == 0 && s_sing >= 0) {
    atomicOr(&a.status->flags, ERR_SINGULAR);
    atomicMin(&a.status->singular_strip, s);
    if (a.nstrips == 1) atomicMin(&a.status->singular_pos, a.level * Wp + s_sing);  // single-slab path
  }
}

// R = perm_l [V_l 0 ; D_{l+1} Usup_{l+1}]: R1 -> U1213 slot, R2 -> sv_out.
__global__ void gather_r_kernel(LevelArgs a) {
  const int s = blockIdx.y, Wp = a.Wp;
  const double* V = a.sv_in + s * a.sSV + (int64_t)Wp * Wp;
  const double* NX = a.nx + s * a.sNX;
  const int32_t* perm = a.perm + s * a.sP;
  double* U1213 = a.slot + s * a.sF + 2LL * Wp * Wp;
  double* r2 = a.sv_out + s * a.sSV;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < 2 * Wp * Wp; idx += gridDim.x * blockDim.x) {
    const int c = idx / Wp, i = idx % Wp;
    auto Rval = [&](int p) -> double {
      if (p < Wp) return c < Wp ? V[(int64_t)c * Wp + p] : 0.0;
      return NX[(int64_t)(Wp + c) * Wp + (p - Wp)];
    };
    U1213[idx] = Rval(perm[i]);
    r2[idx] = Rval(perm[Wp + i]);
  }
}

// Conversion helpers (per strip, batched over levels): X = [I | U1213], and
// the final packing of [Ainv | H] and Fbot into DMMA fragment order.
__global__ void convert_init_kernel(int Wp, const double* slots, int64_t lvl, double* X, int64_t sX) {
  const int64_t l = blockIdx.y;
  const double* U = slots + l * lvl + 2LL * Wp * Wp;
  double* x = X + l * sX;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < 3 * Wp * Wp; idx += gridDim.x * blockDim.x) {
    const int c = idx / Wp, r = idx % Wp;
    x[idx] = c < Wp ? (r == c ? 1.0 : 0.0) : U[(int64_t)(c - Wp) * Wp + r];
  }
}

// out (per level, 4 Wp^2): F = [Ainv ; Fbot] (2Wp x Wp) then H (Wp x 2Wp), fragment order
__global__ void convert_pack_kernel(int Wp, const double* X, int64_t sX, const double* Fb, int64_t sFb,
                                    double* slots, int64_t lvl) {
  const int64_t l = blockIdx.y;
  const double* AH = X + l * sX;    // [Ainv | H] col-major Wp x 3Wp
  const double* F1 = Fb + l * sFb;  // Fbot col-major Wp x Wp
  double* o = slots + l * lvl;
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
      o[idx] = m < Wp ? AH[(int64_t)k * Wp + m] : F1[(int64_t)k * Wp + (m - Wp)];
    } else {
      const int64_t q = (idx - nF) >> 5;
      const int MT = Wp / 8;
      const int mt = (int)(q % MT), ks = (int)(q / MT);
      const int m = mt * 8 + g, k = ks * 4 + t;
      o[idx] = AH[(int64_t)(Wp + k) * Wp + m];
    }
  }
}

}  // namespace

void extract_levels(cudaStream_t st, CsrDev A, const StripDesc* strips, int nstrips, int64_t n2,
                    int Wp, int64_t L0, int64_t nl, double* nx, int64_t sNX, DevStatus* status, double* dsub,
                    uint8_t* lnd) {
  if (nl <= 0) return;
  extract_levels_kernel<<<dim3((unsigned)nl, (unsigned)nstrips), 128, 0, st>>>(A, strips, n2, Wp, L0,
                                                                            nx, sNX, status, dsub, lnd); count_launch();
  SLB_CUDA_CHECK(cudaGetLastError());
}

void extract_couplings(cudaStream_t st, CsrDev A, const StripDesc* strips, int nstrips, int64_t n2,
                       int Wp, double* cpl, int64_t sCPL, int32_t* sym, DevStatus* status) {
  dim3 block(32, 8);
  dim3 grid((unsigned)cdiv(n2, 8), (unsigned)nstrips);
  extract_couplings_kernel<<<grid, block, 0, st>>>(A, strips, n2, Wp, cpl, sCPL, sym, status); count_launch();
  SLB_CUDA_CHECK(cudaGetLastError());
}

void init_sv(cudaStream_t st, int nstrips, int Wp, const double* nx0, int64_t sNX, double* sv,
             int64_t sSV) {
  init_sv_kernel<<<nstrips, 256, 0, st>>>(Wp, nx0, sNX, sv, sSV); count_launch();
  SLB_CUDA_CHECK(cudaGetLastError());
}

void level_lu(cudaStream_t st, const LevelArgs& a) {
  const int Wp = a.Wp;
  const int RS = ((Wp + 15) / 16) * 16 + 4;
  const size_t smem = (size_t)((Wp + 8) * RS + 32 + 8 * Wp) * sizeof(double) + 2 * Wp * sizeof(int);
  static size_t attr = 0;
  if (smem > attr) {
    SLB_CUDA_CHECK(cudaFuncSetAttribute(level_lu_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  // 4 panel warps: measured faster than one warp with 5 rows per lane (register pressure)
  static const bool no_la = getenv("SLB_LU_NOLA") != nullptr;
  if (no_la) {
    level_lu_kernel<4><<<a.nstrips, 512, smem, st>>>(a); count_launch();
  } else {
    const size_t smem2 = (size_t)((Wp + 8) * RS + 32 + 16 * Wp) * sizeof(double) + 2 * Wp * sizeof(int);
    static size_t attr2 = 0;
    if (smem2 > attr2) {
      SLB_CUDA_CHECK(cudaFuncSetAttribute(level_lu_la_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
      SLB_CUDA_CHECK(cudaFuncSetAttribute(level_lu_la_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
      attr2 = smem2;
    }
    static const int tw0 = getenv("SLB_LU_TW0") ? atoi(getenv("SLB_LU_TW0")) : 0;
    LevelArgs a2 = a;
    a2.tw0 = tw0;
    // two panel warps with three rows per lane (cfg3 chain 0.793 -> 0.789 s; the per-column
    // critical path barely depends on the panel's warp count), SLB_LU_PW=4 selects four
    static const int pw = getenv("SLB_LU_PW") ? atoi(getenv("SLB_LU_PW")) : 2;
    if (pw == 2) launch_pdl(level_lu_la_kernel<2>, dim3(a.nstrips), dim3(512), smem2, st, a2);
    else launch_pdl(level_lu_la_kernel<4>, dim3(a.nstrips), dim3(512), smem2, st, a2);
  }
  SLB_CUDA_CHECK(cudaGetLastError());
}

// LU form -> GEMM form for levels [0, nl) of one strip (slots at stride lvl):
//   X = [I | U1213];  X[:, :Wp] = L11^{-1} (lower TRSM);  Fbot = -L21 L11^{-1} (GEMM);
//   X = U11^{-1} X = [Ainv | H] (upper TRSM);  pack [Ainv ; Fbot] and H.
// work: 4 Wp^2 doubles per level.  Runs on a low-priority stream behind the
// chain (one launch group per chunk of levels).
// Rows of Fbot at the bottom positions i that hold a row pivoted down from level l (perm[Wp+i] < Wp):
// the only rows where Fbot t_top differs from -diag(Lsub_{l+1}) y_l.  Up to 8 per level, in
// position order, into exc[level][e][k] (row-major) and excpos[level][e] (-1 unused).
__global__ void convert_exc_kernel(int Wp, const int32_t* perm, const double* Fb, int64_t w2, double* exc,
                                   int32_t* excpos) {
  const int64_t l = blockIdx.x;
  const int32_t* p = perm + l * 2 * Wp;
  __shared__ int pos[8];
  __shared__ int cnt;
  if (threadIdx.x == 0) {
    int c = 0;
    for (int i = 0; i < Wp && c < 8; i++)
      if (p[Wp + i] < Wp) pos[c++] = i;
    cnt = c;
    for (int e = 0; e < 8; e++) excpos[l * 8 + e] = e < c ? pos[e] : -1;
  }
  __syncthreads();
  const double* f = Fb + l * w2;
  for (int idx = threadIdx.x; idx < cnt * Wp; idx += blockDim.x) {
    const int e = idx / Wp, k = idx % Wp;
    exc[(l * 8 + e) * Wp + k] = f[(int64_t)k * Wp + pos[e]];
  }
}

// The x_{l+2} half of H (columns 2Wp.. of [Ainv | H]) is nonzero only in the columns r of the
// level-(l+1) rows pivoted up (Usup diagonal): up to 8 such columns per level into hcol[level][e][i]
// with hidx[level][e] = r (-1 unused), in top-position order.
__global__ void convert_hcol_kernel(int Wp, const int32_t* perm, const double* X, int64_t sX, double* hcol,
                                    int32_t* hidx) {
  const int64_t l = blockIdx.x;
  const int32_t* p = perm + l * 2 * Wp;
  __shared__ int cols[8];
  __shared__ int cnt;
  if (threadIdx.x == 0) {
    int c = 0;
    for (int i = 0; i < Wp && c < 8; i++)
      if (p[i] >= Wp) cols[c++] = p[i] - Wp;
    cnt = c;
    for (int e = 0; e < 8; e++) hidx[l * 8 + e] = e < c ? cols[e] : -1;
  }
  __syncthreads();
  const double* x = X + l * sX;
  for (int idx = threadIdx.x; idx < cnt * Wp; idx += blockDim.x) {
    const int e = idx / Wp, i = idx % Wp;
    hcol[(l * 8 + e) * Wp + i] = x[(int64_t)(2 * Wp + cols[e]) * Wp + i];
  }
}

void convert_levels(cudaStream_t st, int Wp, double* slots, int64_t lvl, int64_t nl, double* work,
                    const int32_t* perm, double* exc, int32_t* excpos, double* hcol, int32_t* hidx) {
  const int64_t w2 = (int64_t)Wp * Wp, sX = 3 * w2;
  double* X = work;
  double* Fb = work + nl * sX;
  convert_init_kernel<<<dim3((unsigned)cdiv(3 * Wp * Wp, 256), (unsigned)nl), 256, 0, st>>>(Wp, slots, lvl, X, sX); count_launch();
  SLB_CUDA_CHECK(cudaGetLastError());
  trsm_small_batched(st, true, Wp, slots, Wp, lvl, X, Wp, sX, Wp, nl);
  dgemm_batched(st, Wp, Wp, Wp, -1.0, slots + w2, Wp, lvl, X, Wp, sX, 0.0, Fb, Wp, w2, nl, true);
  trsm_small_batched(st, false, Wp, slots, Wp, lvl, X, Wp, sX, 3 * Wp, nl);
  convert_pack_kernel<<<dim3((unsigned)std::min<int64_t>(cdiv(4LL * Wp * Wp, 256), 64), (unsigned)nl), 256, 0, st>>>(
      Wp, X, sX, Fb, w2, slots, lvl); count_launch();
  convert_exc_kernel<<<(unsigned)nl, 256, 0, st>>>(Wp, perm, Fb, w2, exc, excpos); count_launch();
  convert_hcol_kernel<<<(unsigned)nl, 256, 0, st>>>(Wp, perm, X, sX, hcol, hidx); count_launch();
  SLB_CUDA_CHECK(cudaGetLastError());
}

}  // namespace slb

