// Stage one, part 2: dense Schur blocks T = A_JJ - A_JI A_II^{-1} A_IJ (sm_100a).
//
// Reference: build_reduced dense branch (proj/include/slablu/stage_one.hpp:
// 357-411) applies apply_T_block (:258-299) to Identity(n2): one dgbtrs with
// n2 right-hand sides per adjacent strip side (banded.hpp:116-128).
//
// Here every strip side Y in {L, R} contributes the n2 x n2 blocks
//   C_XY[p][q] = to_X[p] . (A_ii^{-1} from_Y[:, q])[level p]     (X in {L, R})
// computed by a persistent kernel: one task = (strip, side, C = 64 columns
// starting at level q0).  Column q of from_Y lives on level q only, so the
// forward sweep starts at level q0 - 1 (sparse start).  For symmetric strips
// (A_ii = A_ii^T, to = from^T, detected at factorize time) C is symmetric over
// (X,p)x(Y,q) and the backward sweep stops at level q0 (rows p >= q0 are the
// only ones needed); the mirror half is filled in assemble_T.
//
// Per level, both sweeps are one FP64 GEMM on the DMMA pipe (mma.sync m8n8k4):
//   forward  [y_l ; z_{l+1} - t_bot] = [Ainv ; Fbot] (2Wp x Wp) * t_top (Wp x C)
//   backward x_l = y_l - H_l (Wp x 2Wp) * [x_{l+1} ; x_{l+2}] (2Wp x C)
// A operands stream from HBM/L2 in fragment order (16-byte cp.async, 3-stage
// ring, continuous across levels); B operands stay in shared memory; y_l is
// spilled to a per-CTA HBM slab between the two sweeps.
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace slb {
namespace {

constexpr int THREADS = 512;
// The operand-ring producer thread: lane 0 of the last warp, whose m group holds the fewest row
// tiles (19 = 5 + 5 + 5 + 4 at Wp = 152), so the issue work lands on the least-loaded warp.
constexpr int PRODUCER = THREADS - 32;

// Compile-time layout of a sweep kernel with C right-hand-side columns.
template <int C>
struct Lay {
  // operand ring: SK k4 steps per slice, STAGES slices (measured at cfg3: k8 slices x 3 beat
  // k4 slices x 6 by 17%, the per-slice synchronisation outweighs the deeper prefetch)
  static constexpr int SK = 2;
  static constexpr int STAGES = C >= 32 ? 3 : 8;
  static constexpr int NT = C / 8;                    // n8 tiles
  static constexpr int FWN = NT >= 2 ? 2 : 1;         // forward n groups (per half)
  static constexpr int FWM = 8 / FWN;                 // forward m groups (per half)
  static constexpr int FNT = NT / FWN;                // forward n tiles per warp
  static constexpr int SWN = NT >= 4 ? 4 : NT;        // shortcut forward (Ainv rows only): n groups
  static constexpr int SWM = 16 / SWN;                // ... m groups
  static constexpr int SNT = NT / SWN;                // ... n tiles per warp
  static constexpr int BWN = NT >= 4 ? 4 : NT;        // backward n groups
  static constexpr int BWM = 16 / BWN;                // backward m groups
  static constexpr int BNT = NT / BWN;                // backward n tiles per warp
};

// Calls f with the warp's m-tile count as a compile-time constant (1..MTMAX): the DMMA loops
// then have no per-tile exit branches, and every A fragment of a k4 step is loaded up front.
template <int MTMAX, class F>
__device__ __forceinline__ void dispatch_mt(int cnt, F&& f) {
  switch (cnt) {
    case 5:
      if constexpr (MTMAX >= 5) f(std::integral_constant<int, 5>{});
      break;
    case 4:
      if constexpr (MTMAX >= 4) f(std::integral_constant<int, 4>{});
      break;
    case 3:
      if constexpr (MTMAX >= 3) f(std::integral_constant<int, 3>{});
      break;
    case 2:
      if constexpr (MTMAX >= 2) f(std::integral_constant<int, 2>{});
      break;
    case 1:
      f(std::integral_constant<int, 1>{});
      break;
    default:
      break;
  }
}

template <int C>
__device__ __forceinline__ int swz(int r, int n) {
  if constexpr (C >= 16) return r * C + (n ^ ((r & 3) << 2));
  else return r * C + n;
}

struct TaskGeom {
  int s, side, q0, l0, lstop;
  int64_t nf, nslices;  // forward slices, total slices (upper bound; U13-free levels skip half)
};

template <int C, int MTMAX>
__global__ void __launch_bounds__(THREADS, 1) sweep_kernel(SchurArgs a) {
  using L = Lay<C>;
  constexpr int STAGES = L::STAGES;
  extern __shared__ double sm[];
  const int Wp = a.Wp;
  const int64_t n2 = a.n2;
  double* zb = sm;                       // forward: z      | backward: x buffer 0
  double* tb = sm + Wp * C;              // forward: t_top  | backward: x buffer 1
  double* stg = sm + 2 * Wp * C;         // STAGES slots of 16*Wp doubles
  int* spermb = reinterpret_cast<int*>(stg + STAGES * 8 * L::SK * Wp);  // [2][2 Wp] pivot orders (level l, l+1)
  double* sdsub = reinterpret_cast<double*>(spermb + 4 * Wp);    // [2][Wp] diag(Lsub_{l+1}) (level l, l+1)
  uint8_t* su13 = reinterpret_cast<uint8_t*>(sdsub + 2 * Wp);    // n2 level flags of the current strip
  __shared__ int s_task;
  __shared__ __align__(8) uint64_t full_bar[L::STAGES];
  __shared__ __align__(8) uint64_t empty_bar[L::STAGES];
  // Ring state persists across tasks: slot = global slice counter % STAGES.
  // The producer (thread PRODUCER) fills slot s for slice q after all warps released
  // slice q - STAGES from it; consumers wait on full_bar[s] with parity
  // (q / STAGES) & 1 and release with one arrive per warp.
  // ring positions + phases (producer state lives in thread PRODUCER only)
  int p_slot = 0, c_slot = 0;
  uint32_t p_round = 0, c_phase = 0;  // p_round: completed passes over the ring (producer)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int MTH = Wp / 8;                       // m8 tiles per Wp rows
  const int FMT = (MTH + L::FWM - 1) / L::FWM;  // forward m tiles per warp
  const int BMT = (MTH + L::BWM - 1) / L::BWM;  // backward m tiles per warp
  constexpr int SK = L::SK;
  const int fslice = 8 * SK * Wp;               // doubles per forward slice (SK k4 steps of [Ainv ; Fbot])
  const int bslice = 4 * SK * Wp;               // doubles per backward slice (SK k4 steps of H)
  const int64_t lvl_stride = 4LL * Wp * Wp;
  const int kf = Wp / (4 * SK), kb = Wp / (2 * SK);  // slices per level (fwd, bwd)
  double* ybase = a.ybuf + (int64_t)blockIdx.x * a.sY;
  if (tid == 0) {
    for (int i = 0; i < STAGES; i++) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], THREADS / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();

  for (;;) {
    if (tid == 0) s_task = atomicAdd(a.task_counter, 1);
    __syncthreads();
    const int task = s_task;
    __syncthreads();
    if (task >= a.ntasks) break;
    TaskGeom T;
    T.s = a.tasks[3 * task];
    T.side = a.tasks[3 * task + 1];
    T.q0 = a.tasks[3 * task + 2];
    const bool schur = a.mode == SWEEP_SCHUR;
    T.l0 = (schur && T.q0 > 0) ? T.q0 - 1 : 0;
    T.lstop = (schur && a.sym[T.s]) ? T.q0 : 0;
    T.nf = (n2 - T.l0) * kf;
    const StripDesc sd = a.strips[T.s];
    const double* fac = a.fac + T.s * a.sF;
    const int32_t* permg = a.perm + T.s * a.sP;
    {
      const uint8_t* u13g = a.u13 + T.s * n2;
      for (int64_t i = tid; i < n2; i += THREADS) su13[i] = u13g[i];
      __syncthreads();
    }
    const double* cpl = a.cpl + T.s * a.sCPL;
    const double* fromY = cpl + (T.side == 0 ? 0 : n2 * Wp);
    const double* toL = cpl + 2 * n2 * Wp;
    const double* toR = cpl + 3 * n2 * Wp;
    double* gb = a.gbuf + T.s * a.sG;
    const int64_t rem = schur ? n2 - T.q0 : a.nrhs - T.q0;
    const int ncols = (int)(rem < C ? rem : C);
    // dense right-hand side of level Lv (solve modes): b_Lv[i][n]
    auto rhs_val = [&](int64_t Lv, int i, int n) -> double {
      if (i >= sd.w || n >= ncols) return 0.0;
      const int64_t col = T.q0 + n;
      double v = a.f[col * a.N + (int64_t)(sd.col0 + i) * n2 + Lv];
      if (a.mode == SWEEP_RECOVER) {
        if (sd.left >= 0) v -= cpl[Lv * Wp + i] * a.u_ifc[col * a.K + (int64_t)sd.left * n2 + Lv];
        if (sd.right >= 0) v -= cpl[n2 * Wp + Lv * Wp + i] * a.u_ifc[col * a.K + (int64_t)sd.right * n2 + Lv];
      }
      return v;
    };

    // Slice stream: forward levels l0..n2-1 (kf slices each), then backward
    // levels n2-1..lstop (kb slices, or kb/2 when U13 = 0 on that level).
    // The producer (thread PRODUCER) walks it with an incremental cursor; the U13
    // flags of the strip sit in shared memory (loaded at task start).
    const double* p_src = fac + (int64_t)T.l0 * lvl_stride;
    int p_len = fslice, p_left = kf;
    int64_t p_lvl = T.l0;
    bool p_fwd = true, p_done = false;
    // backward level streams the full H (kb slices) only if U13 != 0 and its x_{l+2} half cannot
    // be applied as the few columns of the rows pivoted up (Usup not diagonal or > 8 such rows)
    auto bwd_full = [&](uint8_t f) -> bool {
      return (f & 1) && !(a.bsc && !(f & 64) && ((f >> 2) & 15) <= 8);
    };
    auto issue = [&]() {
      if (tid != PRODUCER || p_done) return;
      const double* src = p_src;
      const int len = p_len;
      // shortcut level (flags == 0): only the Ainv half of each k4 block of [Ainv ; Fbot]
      const bool split = a.fsc && p_fwd && (su13[p_lvl] & 2) == 0 && (su13[p_lvl] >> 2) <= 8;
      if (--p_left > 0) {
        p_src += p_len;
      } else if (p_fwd) {
        if (++p_lvl == n2) {
          p_fwd = false;
          p_lvl = n2 - 1;
          if (p_lvl < T.lstop) {
            p_done = true;
          } else {
            p_src = fac + p_lvl * lvl_stride + 2LL * Wp * Wp;
            p_len = bslice;
            p_left = bwd_full(su13[p_lvl]) ? kb : kb / 2;
          }
        } else {
          p_src += p_len + (lvl_stride - (int64_t)kf * fslice);
          p_left = kf;
        }
      } else {
        if (--p_lvl < T.lstop) {
          p_done = true;
        } else {
          p_src = fac + p_lvl * lvl_stride + 2LL * Wp * Wp;
          p_left = bwd_full(su13[p_lvl]) ? kb : kb / 2;
        }
      }
      const int sl = p_slot;
      if (p_round > 0) mbar_wait(&empty_bar[sl], (p_round - 1) & 1u);
      if (split) {
        const uint32_t hb = (uint32_t)(4 * Wp * sizeof(double));  // MTH m8 tiles of one k4 step
        mbar_arrive_expect_tx(&full_bar[sl], SK * hb);
#pragma unroll
        for (int kk = 0; kk < SK; kk++) bulk_g2s(stg + sl * fslice + kk * 4 * Wp, src + kk * 8 * Wp, hb, &full_bar[sl]);
      } else {
        mbar_arrive_expect_tx(&full_bar[sl], (uint32_t)(len * sizeof(double)));
        bulk_g2s(stg + sl * fslice, src, (uint32_t)(len * sizeof(double)), &full_bar[sl]);
      }
      if (++p_slot == STAGES) {
        p_slot = 0;
        p_round++;
      }
    };
    // consumer side: wait for the current slice, release it after use
    auto acquire = [&]() -> const double* {
      mbar_wait(&full_bar[c_slot], c_phase);
      return stg + c_slot * fslice;
    };
    auto release = [&]() {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[c_slot]);
      if (++c_slot == STAGES) {
        c_slot = 0;
        c_phase ^= 1u;
      }
    };

    for (int i = 0; i < STAGES - 1; i++) issue();

    // ---------------- forward sweep ----------------
    for (int idx = tid; idx < Wp * C; idx += THREADS) zb[idx] = 0.0;
    __syncthreads();
    if (schur) {
      if (T.q0 == 0)  // column 0 lives on level 0: z_0 = from_Y[level 0]
        for (int i = tid; i < Wp; i += THREADS) zb[swz<C>(i, 0)] = fromY[i];
    } else {
      for (int idx = tid; idx < Wp * C; idx += THREADS) {
        const int r = idx / C, n = idx % C;
        zb[swz<C>(r, n)] = rhs_val(0, r, n);
      }
    }

    const int half = warp >> 3;            // 0: Ainv rows (y), 1: Fbot rows (z')
    const int fwm = (warp & 7) / L::FWN;   // m group
    const int fwn = (warp & 7) % L::FWN;   // n group
    // pivot order of the first level now; each level prefetches the next one (cp.async)
    const double* dsubg = a.dsub + (int64_t)T.s * n2 * Wp;
    for (int i = tid; i < 2 * Wp; i += THREADS) spermb[i] = permg[T.l0 * 2 * Wp + i];
    for (int i = tid; i < Wp; i += THREADS) sdsub[i] = dsubg[T.l0 * Wp + i];
    int pcur = 0;
#ifdef SLB_SCHUR_PROF
    long long S0 = clock64(), sp[6] = {0, 0, 0, 0, 0, 0}, wacq = 0, nsc = 0, ep[3] = {0, 0, 0};
#define SP(k_) { const long long q_ = clock64(); sp[k_] += q_ - S0; S0 = q_; }
#else
#define SP(k_)
#endif
    for (int64_t l = T.l0; l < n2; l++) {
      const bool has_next = l + 1 < n2;
      const int cstar = (schur && has_next) ? (int)(l + 1 - T.q0) : -1;  // column injected
      const bool inj = cstar >= 0 && cstar < ncols;
      const double* fvec = inj ? fromY + (l + 1) * Wp : nullptr;
      SP(4)
      cp_async_wait<0>();
      __syncthreads();  // sperm (this level) and z_l complete
      SP(0)
      const int* sperm = spermb + pcur * 2 * Wp;
      const double* dsl = sdsub + pcur * Wp;
      if (has_next && tid < Wp / 2)  // 2 Wp int32 = Wp / 2 16-byte pieces
        cp_async16(spermb + (pcur ^ 1) * 2 * Wp + 4 * tid, permg + (l + 1) * 2 * Wp + 4 * tid, true);
      else if (has_next && tid >= 256 && tid < 256 + Wp / 2)  // Wp doubles = Wp / 2 pieces
        cp_async16(sdsub + (pcur ^ 1) * Wp + 2 * (tid - 256), dsubg + (l + 1) * Wp + 2 * (tid - 256), true);
      cp_async_commit();
      pcur ^= 1;
      // shortcut level: no level-(l+1) row pivoted up and Lsub_{l+1} diagonal, so
      // Fbot t_top = -diag(Lsub_{l+1}) y_l: stream Ainv only, all warps on its rows
      const bool sc = a.fsc && (su13[l] & 2) == 0 && (su13[l] >> 2) <= 8;
#ifdef SLB_SCHUR_PROF
      nsc += sc ? 1 : 0;
#endif
      // shortcut: all 16 warps on the MTH rows of Ainv, as SWM m groups x SWN n groups
      const int hf = sc ? 0 : half;
      const int fm = sc ? warp / L::SWN : fwm;
      const int fmt = sc ? (MTH + L::SWM - 1) / L::SWM : FMT;
      const int fnb = sc ? (warp % L::SWN) * L::SNT : fwn * L::FNT;  // first n tile of this warp
      const int fnn = sc ? L::SNT : L::FNT;                          // n tiles of this warp
      auto vval = [&](int src, int n) -> double {
        if (src < Wp) return zb[swz<C>(src, n)];
        if (!schur) return has_next ? rhs_val(l + 1, src - Wp, n) : 0.0;
        return (inj && n == cstar) ? fvec[src - Wp] : 0.0;
      };
      // t_top = rows perm[0..Wp) of [z_l ; b_{l+1}]: one row per warp step, two columns per lane
      for (int r = warp; r < Wp; r += THREADS / 32) {
        const int src = sperm[r];
        if (2 * lane < C) {
          double2 v;
          if (src < Wp) {
            v = *reinterpret_cast<const double2*>(&zb[swz<C>(src, 2 * lane)]);
          } else {
            v.x = vval(src, 2 * lane);
            v.y = vval(src, 2 * lane + 1);
          }
          *reinterpret_cast<double2*>(&tb[swz<C>(r, 2 * lane)]) = v;
        }
      }
      double acc[MTMAX][L::FNT][2];
#pragma unroll
      for (int mi = 0; mi < MTMAX; mi++)
#pragma unroll
        for (int nj = 0; nj < L::FNT; nj++) {
          acc[mi][nj][0] = acc[mi][nj][1] = 0.0;
          const int mt = fm * fmt + mi;
          if (hf == 1 && mi < fmt && mt < MTH) {
            const int row = mt * 8 + g;
            const int col = (fwn * L::FNT + nj) * 8 + 2 * t;
            const int src = sperm[Wp + row];
            acc[mi][nj][0] = vval(src, col);
            acc[mi][nj][1] = vval(src, col + 1);
          }
        }
      SP(1)
      __syncthreads();
      SP(2)
      for (int j = 0; j < kf; j++) {
#ifdef SLB_SCHUR_PROF
        long long W0 = clock64();
        issue();
        long long W1 = clock64();
        const double* A = acquire();
        long long W2 = clock64();
        sp[5] += W1 - W0;
        wacq += W2 - W1;
#else
        issue();
        const double* A = acquire();
#endif
        if (sc) {  // Ainv rows only: SNT n tiles per warp
          const int cnt = min(fmt, MTH - fm * fmt);
          dispatch_mt<MTMAX>(cnt, [&](auto MTc) {
            constexpr int MT = decltype(MTc)::value;
#pragma unroll
            for (int kk = 0; kk < SK; kk++) {
              const int k = j * 4 * SK + kk * 4 + t;  // B row
              double bf[L::SNT], af[MT];
#pragma unroll
              for (int nj = 0; nj < L::SNT; nj++) bf[nj] = tb[swz<C>(k, (fnb + nj) * 8 + g)];
              const double* Ak = A + kk * MTH * 32 + (fm * fmt) * 32 + lane;
#pragma unroll
              for (int mi = 0; mi < MT; mi++) af[mi] = Ak[mi * 32];
#pragma unroll
              for (int mi = 0; mi < MT; mi++)
#pragma unroll
                for (int nj = 0; nj < L::SNT; nj++) dmma884(acc[mi][nj][0], acc[mi][nj][1], af[mi], bf[nj]);
            }
          });
        } else {
          // predicated-off DMMAs would still occupy the pipe: the tile count is a template constant
          const int cnt = min(fmt, MTH - fm * fmt);
          dispatch_mt<MTMAX>(cnt, [&](auto MTc) {
            constexpr int MT = decltype(MTc)::value;
#pragma unroll
            for (int kk = 0; kk < SK; kk++) {
              const int k = j * 4 * SK + kk * 4 + t;  // B row
              double bf[L::FNT], af[MT];
#pragma unroll
              for (int nj = 0; nj < L::FNT; nj++) bf[nj] = tb[swz<C>(k, (fwn * L::FNT + nj) * 8 + g)];
              const double* Ak = A + kk * (2 * MTH) * 32 + hf * MTH * 32 + (fm * fmt) * 32 + lane;
#pragma unroll
              for (int mi = 0; mi < MT; mi++) af[mi] = Ak[mi * 32];
#pragma unroll
              for (int mi = 0; mi < MT; mi++)
#pragma unroll
                for (int nj = 0; nj < L::FNT; nj++) dmma884(acc[mi][nj][0], acc[mi][nj][1], af[mi], bf[nj]);
            }
          });
        }
        release();
      }
      SP(3)
      // epilogue: y_l -> HBM slab (canonical tile order), z_{l+1} -> smem
      double* ylev = ybase + (l - T.l0) * (int64_t)Wp * C;
#pragma unroll
      for (int mi = 0; mi < MTMAX; mi++) {
        const int mt = fm * fmt + mi;
        if (mi >= fmt || mt >= MTH) continue;
#pragma unroll
        for (int nj = 0; nj < L::FNT; nj++) {
          if (nj >= fnn) break;
          const int nt = fnb + nj;
          if (hf == 0) {
            double2* dst = reinterpret_cast<double2*>(ylev + ((int64_t)(mt * L::NT + nt) * 32 + lane) * 2);
            *dst = make_double2(acc[mi][nj][0], acc[mi][nj][1]);
          } else {
            const int row = mt * 8 + g, col = nt * 8 + 2 * t;
            zb[swz<C>(row, col)] = acc[mi][nj][0];
            zb[swz<C>(row, col + 1)] = acc[mi][nj][1];
          }
        }
      }
#ifdef SLB_SCHUR_PROF
      { const long long q_ = clock64(); ep[0] += q_ - S0; S0 = q_; }
#endif
      if (sc) {
        // z_{l+1}[i] = t_bot[i] - d_i y_l[i], except at the (few) bottom positions holding a row
        // pivoted down from level l, where z_{l+1}[i] = t_bot[i] + Fbot[i,:] t_top.  Every t_bot
        // value (old z_l rows) is read first; z is overwritten in place after the barrier.
        const int ncx = (su13[l] >> 2) & 15;
        const int64_t li = (int64_t)T.s * n2 + l;
        const int kn = tid >> 3, kp = tid & 7;  // exceptional rows: column kn, k-part kp of 8
        double exv[8];
#pragma unroll
        for (int e = 0; e < 8; e++) {  // t_bot at the exceptional positions (old z rows)
          exv[e] = 0.0;
          if (e < ncx && kp == 0 && kn < C) exv[e] = vval(sperm[Wp + a.excpos[li * 8 + e]], kn);
        }
#pragma unroll
        for (int mi = 0; mi < MTMAX; mi++) {
          const int mt = fm * fmt + mi;
          if (mi >= fmt || mt >= MTH) continue;
          // unswapped bottom position i keeps level-(l+1) row i: t_bot[i] = b_{l+1}[i] (the
          // exceptional positions are rewritten below)
          const int row = mt * 8 + g;
          const double dd = dsl[row];
#pragma unroll
          for (int nj = 0; nj < L::FNT; nj++) {
            if (nj >= fnn) break;
            const int col = (fnb + nj) * 8 + 2 * t;
            acc[mi][nj][0] = fma(-dd, acc[mi][nj][0], vval(Wp + row, col));
            acc[mi][nj][1] = fma(-dd, acc[mi][nj][1], vval(Wp + row, col + 1));
          }
        }
#ifdef SLB_SCHUR_PROF
        { const long long q_ = clock64(); ep[1] += q_ - S0; S0 = q_; }
#endif
        __syncthreads();
#ifdef SLB_SCHUR_PROF
        { const long long q_ = clock64(); ep[2] += q_ - S0; S0 = q_; }
#endif
#pragma unroll
        for (int mi = 0; mi < MTMAX; mi++) {
          const int mt = fm * fmt + mi;
          if (mi >= fmt || mt >= MTH) continue;
#pragma unroll
          for (int nj = 0; nj < L::FNT; nj++) {
            if (nj >= fnn) break;
            const int row = mt * 8 + g, col = (fnb + nj) * 8 + 2 * t;
            zb[swz<C>(row, col)] = acc[mi][nj][0];
            zb[swz<C>(row, col + 1)] = acc[mi][nj][1];
          }
        }
        if (ncx > 0) {
          // + Fbot[i,:] t_top (t_top is intact until the next level's build): every thread takes
          // an eighth of the k range of one column, the parts meet through three shuffles
#pragma unroll
          for (int e = 0; e < 8; e++) {
            if (e >= ncx) break;
            double q = 0.0;
            if (kn < C) {
              const double* er = a.exc + (li * 8 + e) * Wp;
              for (int k = kp; k < Wp; k += 8) q = fma(er[k], tb[swz<C>(k, kn)], q);
            }
            q += __shfl_xor_sync(0xffffffffu, q, 1);
            q += __shfl_xor_sync(0xffffffffu, q, 2);
            q += __shfl_xor_sync(0xffffffffu, q, 4);
            exv[e] += q;
          }
          __syncthreads();  // the generic rows above also wrote these positions
          if (kp == 0 && kn < C) {
#pragma unroll
            for (int e = 0; e < 8; e++) {
              if (e >= ncx) break;
              zb[swz<C>(a.excpos[li * 8 + e], kn)] = exv[e];
            }
          }
        }
      }
    }

#ifdef SLB_SCHUR_PROF
    if ((tid == 0 || tid == 160 || tid == PRODUCER) && blockIdx.x == 0)
      printf("SCHUR tid %d task %d levels %lld: topsync %lld build %lld presync %lld kloop %lld (issue %lld acquire-wait %lld) epi %lld [ystore %lld zcomp %lld bar1 %lld] shortcut-levels %lld\n",
             tid, task, (long long)(n2 - T.l0), sp[0], sp[1], sp[2], sp[3], sp[5], wacq, sp[4], ep[0], ep[1], ep[2], nsc);
#endif
    // ---------------- backward sweep ----------------
    __syncthreads();
    for (int idx = tid; idx < 2 * Wp * C; idx += THREADS) sm[idx] = 0.0;  // x_{n2}, x_{n2+1} = 0
    __syncthreads();
    const int bwm = warp / L::BWN;    // m group
    const int bwn = warp % L::BWN;    // n group
    int p_buf = 0;                    // buffer holding x_{l+1}; the other holds x_{l+2}
    for (int64_t l = n2 - 1; l >= T.lstop; l--) {
      const double* ylev = ybase + (l - T.l0) * (int64_t)Wp * C;
      if (l - 1 >= T.lstop) {  // y_{l-1} was written long ago (HBM): pull it into L2 one level ahead
        const char* yn = reinterpret_cast<const char*>(ylev - (int64_t)Wp * C);
        for (int off = tid * 128; off < Wp * C * 8; off += THREADS * 128)
          asm volatile("prefetch.global.L2 [%0];\n" ::"l"(yn + off));
      }
      const uint8_t fl = su13[l];
      const int kbl = bwd_full(fl) ? kb : kb / 2;  // else x_{l+2} enters through <= 8 columns of H
      const int nhc = ((fl & 1) && !bwd_full(fl)) ? ((fl >> 2) & 15) : 0;
      double acc[MTMAX][L::BNT][2];
#pragma unroll
      for (int mi = 0; mi < MTMAX; mi++) {
        const int mt = bwm * BMT + mi;
#pragma unroll
        for (int nj = 0; nj < L::BNT; nj++) {
          acc[mi][nj][0] = acc[mi][nj][1] = 0.0;
          if (mi < BMT && mt < MTH) {
            const int nt = bwn * L::BNT + nj;
            const double2 v = *reinterpret_cast<const double2*>(ylev + ((int64_t)(mt * L::NT + nt) * 32 + lane) * 2);
            acc[mi][nj][0] = -v.x;  // accumulate -x, negate at the end
            acc[mi][nj][1] = -v.y;
          }
        }
      }
      const double* xp = sm + p_buf * Wp * C;        // x_{l+1}
      const double* xq = sm + (1 - p_buf) * Wp * C;  // x_{l+2}
      for (int j = 0; j < kbl; j++) {
        issue();
        const double* A = acquire();
        const int kj = j * 4 * SK;
        const double* xs = (kj < Wp) ? xp : xq;
        const int kbase = (kj < Wp) ? kj : kj - Wp;
        dispatch_mt<MTMAX>(min(BMT, MTH - bwm * BMT), [&](auto MTc) {
          constexpr int MT = decltype(MTc)::value;
#pragma unroll
          for (int kk = 0; kk < SK; kk++) {
            const int k = kbase + kk * 4 + t;
            double bf[L::BNT], af[MT];
#pragma unroll
            for (int nj = 0; nj < L::BNT; nj++) bf[nj] = xs[swz<C>(k, (bwn * L::BNT + nj) * 8 + g)];
            const double* Ak = A + kk * MTH * 32 + (bwm * BMT) * 32 + lane;
#pragma unroll
            for (int mi = 0; mi < MT; mi++) af[mi] = Ak[mi * 32];
#pragma unroll
            for (int mi = 0; mi < MT; mi++)
#pragma unroll
              for (int nj = 0; nj < L::BNT; nj++) dmma884(acc[mi][nj][0], acc[mi][nj][1], af[mi], bf[nj]);
          }
        });
        release();
      }
      if (nhc > 0) {  // acc (= -x) += H[:, r] x_{l+2}[r, :] for the columns r of the rows pivoted up
        const int64_t li = (int64_t)T.s * n2 + l;
#pragma unroll
        for (int e = 0; e < 8; e++) {
          if (e >= nhc) break;
          const int r = a.hidx[li * 8 + e];
          const double* hc = a.hcol + (li * 8 + e) * Wp;
#pragma unroll
          for (int mi = 0; mi < MTMAX; mi++) {
            const int mt = bwm * BMT + mi;
            if (mi >= BMT || mt >= MTH) break;
            const double hv = hc[mt * 8 + g];
#pragma unroll
            for (int nj = 0; nj < L::BNT; nj++) {
              const int col = (bwn * L::BNT + nj) * 8 + 2 * t;
              acc[mi][nj][0] = fma(hv, xq[swz<C>(r, col)], acc[mi][nj][0]);
              acc[mi][nj][1] = fma(hv, xq[swz<C>(r, col + 1)], acc[mi][nj][1]);
            }
          }
        }
      }
      __syncthreads();  // everyone done reading x_{l+2}
      double* xo = sm + (1 - p_buf) * Wp * C;  // x_l overwrites x_{l+2}
#pragma unroll
      for (int mi = 0; mi < MTMAX; mi++) {
        const int mt = bwm * BMT + mi;
        if (mi >= BMT || mt >= MTH) continue;
#pragma unroll
        for (int nj = 0; nj < L::BNT; nj++) {
          const int row = mt * 8 + g, col = (bwn * L::BNT + nj) * 8 + 2 * t;
          xo[swz<C>(row, col)] = -acc[mi][nj][0];
          xo[swz<C>(row, col + 1)] = -acc[mi][nj][1];
        }
      }
      __syncthreads();
      if (a.mode == SWEEP_RECOVER) {
        for (int idx = tid; idx < sd.w * ncols; idx += THREADS) {
          const int i = idx % sd.w, n = idx / sd.w;
          a.out[(T.q0 + n) * a.N + (int64_t)(sd.col0 + i) * n2 + l] = xo[swz<C>(i, n)];
        }
      } else {
        // boundary extraction: C_XY[l][q0 + n] = to_X[l] . x_l[:, n]
        constexpr int PARTS = THREADS / (2 * C);  // threads per (X, n) dot product
        const int X = tid / (THREADS / 2);
        const int n = (tid / PARTS) % C;
        const int part = tid % PARTS;
        const double* tv = (X == 0 ? toL : toR) + l * Wp;
        double sum = 0.0;
        for (int i = part; i < Wp; i += PARTS) sum = fma(tv[i], xo[swz<C>(i, n)], sum);
#pragma unroll
        for (int o = 1; o < PARTS; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        const bool has = X == 0 ? sd.left >= 0 : sd.right >= 0;
        if (part == 0 && has && n < ncols) {
          if (schur) gb[((int64_t)(X * 2 + T.side) * n2 + l) * n2 + T.q0 + n] = sum;
          else a.out[((int64_t)(T.s * 2 + X) * a.nrhs + T.q0 + n) * n2 + l] = sum;  // contrib[s][X][col][l]
        }
      }
      p_buf = 1 - p_buf;
    }
    __syncthreads();
  }
}

template <int C>
void launch_sweep(cudaStream_t st, const SchurArgs& a, int nslots) {
  using L = Lay<C>;
  const int Wp = a.Wp;
  const size_t smem =
      (size_t)(2 * Wp * C + L::STAGES * 8 * L::SK * Wp + 2 * Wp) * sizeof(double) + 4 * Wp * sizeof(int) + a.n2;
  const int mth = Wp / 8;
  const int mt = std::max((mth + L::FWM - 1) / L::FWM, (mth + L::BWM - 1) / L::BWM);
  auto go = [&](auto kern) {
    SLB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<nslots, THREADS, smem, st>>>(a); count_launch();
  };
  if (mt <= 1) go(sweep_kernel<C, 1>);
  else if (mt <= 2) go(sweep_kernel<C, 2>);
  else if (mt <= 3) go(sweep_kernel<C, 3>);
  else if (mt <= 4) go(sweep_kernel<C, 4>);
  else if (mt <= 5) go(sweep_kernel<C, 5>);
  else throw CudaFailure(cudaErrorInvalidValue, "sweep: slab width > 160 unsupported", __FILE__, __LINE__);
  SLB_CUDA_CHECK(cudaGetLastError());
}

}  // namespace

void sweep(cudaStream_t st, const SchurArgs& a, int nslots) {
  if (a.chunk == 8) launch_sweep<8>(st, a, nslots);
  else launch_sweep<64>(st, a, nslots);
}

// ---------------------------------------------------------------------------
// T assembly (reference order: direct term, then the strip left of the
// interface (its right side), then the strip right of it (its left side);
// inc/stage_one.hpp:284-297).  T blocks are n2 x n2 column major.
namespace {

__device__ __forceinline__ double cval(const double* gb, int64_t n2, int sym, int X, int Y, int64_t p,
                                       int64_t q) {
  if (sym && p < q) return gb[((int64_t)(Y * 2 + X) * n2 + q) * n2 + p];
  return gb[((int64_t)(X * 2 + Y) * n2 + p) * n2 + q];
}

// grid (ceil(n2/32), ceil(n2/32), nblocks) with blocks ordered diag j (k), super j (k-1), sub j (k-1);
// blocks outside the shard's ranges are skipped, strip terms from non-local strips are left out
__global__ void assemble_T_kernel(int64_t n2, int nifc, int nstrips, const int32_t* sym,
                                  const double* gbuf, int64_t sG, double* Tdiag, double* Tsup,
                                  double* Tsub, TRanges tr) {
  __shared__ double tile[32][33];
  const int b = blockIdx.z;
  int kind, j;
  if (b < nifc) {
    kind = 0;
    j = b;
  } else if (b < 2 * nifc - 1) {
    kind = 1;
    j = b - nifc;
  } else {
    kind = 2;
    j = b - (2 * nifc - 1);
  }
  if (kind == 0 ? (j < tr.dlo || j >= tr.dhi) : (j < tr.ulo || j >= tr.uhi)) return;
  double* T = (kind == 0 ? Tdiag : kind == 1 ? Tsup : Tsub) + (int64_t)j * n2 * n2;
  const int64_t p0 = (int64_t)blockIdx.x * 32, q0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  // The two (or one) strip terms, each (strip, X, Y):
  //  diag j: strip j (X=R,Y=R), strip j+1 (X=L,Y=L) if it exists
  //  super j (T_{j,j+1}): strip j+1 (X=L, Y=R);  sub j (T_{j+1,j}): strip j+1 (X=R, Y=L)
  int ns = 0, st_[2], X_[2], Y_[2];
  if (kind == 0) {
    st_[ns] = j; X_[ns] = 1; Y_[ns] = 1; ns++;
    if (j + 1 < tr.nstrips_global) { st_[ns] = j + 1; X_[ns] = 0; Y_[ns] = 0; ns++; }
  } else if (kind == 1) {
    st_[ns] = j + 1; X_[ns] = 0; Y_[ns] = 1; ns++;
  } else {
    st_[ns] = j + 1; X_[ns] = 1; Y_[ns] = 0; ns++;
  }
  // element (p, q) of T at T[q*n2 + p]; thread (tx, ty..) handles p = p0 + tx, q = q0 + ty + 8r
  double val[4];
#pragma unroll
  for (int r = 0; r < 4; r++) {
    const int64_t p = p0 + tx, q = q0 + ty + 8 * r;
    val[r] = (p < n2 && q < n2) ? T[q * n2 + p] : 0.0;
  }
  for (int e = 0; e < ns; e++) {
    const int ls = st_[e] - tr.sbase;  // local strip
    if (ls < 0 || ls >= nstrips) continue;
    const double* gb = gbuf + ls * sG;
    const int sy = sym[ls];
    // coalesced path: load the 32x32 tile with q fastest (row-major gbuf) then transpose
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 4; r++) {
      const int64_t p = p0 + ty + 8 * r, q = q0 + tx;
      tile[ty + 8 * r][tx] = (p < n2 && q < n2) ? cval(gb, n2, sy, X_[e], Y_[e], p, q) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 4; r++) val[r] -= tile[tx][ty + 8 * r];
  }
#pragma unroll
  for (int r = 0; r < 4; r++) {
    const int64_t p = p0 + tx, q = q0 + ty + 8 * r;
    if (p < n2 && q < n2) T[q * n2 + p] = val[r];
  }
}

// Direct interface blocks from the CSR: grid = owned interfaces, each block scans the
// interface's rows and scatters into the zeroed T blocks.
__global__ void direct_T_kernel(CsrDev A, int64_t n2, int nifc, const int64_t* ifc_off,
                                const StripDesc* strips, int nstrips, double* Tdiag, double* Tsup,
                                double* Tsub, DevStatus* status, TRanges tr) {
  const int j = tr.olo + blockIdx.x;
  const int64_t off = ifc_off[j];
  for (int64_t p = threadIdx.x; p < n2; p += blockDim.x) {
    const int64_t r = off + p;
    for (int32_t e = A.rp[r]; e < A.rp[r + 1]; e++) {
      const int64_t c = A.ci[e];
      const double v = A.v[e];
      if (c >= off && c < off + n2) {
        Tdiag[(int64_t)j * n2 * n2 + (c - off) * n2 + p] = v;
      } else if (j + 1 < nifc && c >= ifc_off[j + 1] && c < ifc_off[j + 1] + n2) {
        if (j >= tr.ulo && j < tr.uhi) Tsup[(int64_t)j * n2 * n2 + (c - ifc_off[j + 1]) * n2 + p] = v;
        else atomicOr(&status->flags, ERR_IFC_STRUCTURE);  // interface-interface coupling across shards
      } else if (j > 0 && c >= ifc_off[j - 1] && c < ifc_off[j - 1] + n2) {
        if (j - 1 >= tr.ulo && j - 1 < tr.uhi) Tsub[(int64_t)(j - 1) * n2 * n2 + (c - ifc_off[j - 1]) * n2 + p] = v;
        else atomicOr(&status->flags, ERR_IFC_STRUCTURE);
      } else {
        // must belong to the strip left (j) or right (j+1) of the interface (a non-local strip
        // cannot be checked here; its own shard checks it)
        bool ok = false, unverifiable = false;
        for (int s = j; s <= j + 1 && s < tr.nstrips_global; s++) {
          const int ls = s - tr.sbase;
          if (ls < 0 || ls >= nstrips) {
            unverifiable = true;
            continue;
          }
          const int64_t b0 = (int64_t)strips[ls].col0 * n2, b1 = b0 + (int64_t)strips[ls].w * n2;
          if (c >= b0 && c < b1) ok = true;
        }
        ok = ok || unverifiable;
        if (!ok) atomicOr(&status->flags, ERR_IFC_STRUCTURE);
      }
    }
  }
}

}  // namespace

void assemble_T(cudaStream_t st, int64_t n2, int nifc, int nstrips, const StripDesc* strips,
                const int32_t* sym, const double* gbuf, int64_t sG, double* Tdiag, double* Tsup,
                double* Tsub, CsrDev A, const int64_t* ifc_off, DevStatus* status, const TRanges& tr) {
  const int64_t bsz = n2 * n2 * sizeof(double);
  SLB_CUDA_CHECK(cudaMemsetAsync(Tdiag, 0, bsz * nifc, st));
  if (nifc > 1) {
    SLB_CUDA_CHECK(cudaMemsetAsync(Tsup, 0, bsz * (nifc - 1), st));
    SLB_CUDA_CHECK(cudaMemsetAsync(Tsub, 0, bsz * (nifc - 1), st));
  }
  if (tr.ohi > tr.olo) {
    direct_T_kernel<<<tr.ohi - tr.olo, 256, 0, st>>>(A, n2, nifc, ifc_off, strips, nstrips, Tdiag, Tsup, Tsub,
                                                     status, tr); count_launch();
    SLB_CUDA_CHECK(cudaGetLastError());
  }
  const int nblocks = 3 * nifc - 2;
  dim3 grid((unsigned)cdiv(n2, 32), (unsigned)cdiv(n2, 32), (unsigned)nblocks);
  assemble_T_kernel<<<grid, dim3(32, 8), 0, st>>>(n2, nifc, nstrips, sym, gbuf, sG, Tdiag, Tsup, Tsub, tr); count_launch();
  SLB_CUDA_CHECK(cudaGetLastError());
}

}  // namespace slb
