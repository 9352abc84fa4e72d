// Slab sweeps of the solve phase (reduce_rhs / recover_interiors) on
// thread-block clusters (sm_100a).
//
// Reference: reduce_rhs (proj/include/slablu/stage_one.hpp:415-433) and
// recover_interiors (:438-462), each one dgbtrs with nrhs columns per slab
// (banded.hpp:116-128).  Bandwidth-bound: every level's sweep operators
// (F = [Ainv ; Fbot], H) are read once per pass.  One task = (strip, 8 RHS
// columns) runs on a cluster of G CTAs; CTA r owns a slice of the output rows
// of every level GEMM and streams only its slice of F / H (TMA bulk copies,
// mbarrier ring).  After each level the new vector (z_{l+1} or x_l) is
// all-gathered through distributed shared memory; parity double buffers make
// one cluster barrier per level sufficient.
#include <cooperative_groups.h>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace slb {
namespace {

constexpr int G = 4;                  // CTAs per cluster
constexpr int C = 8;                  // RHS columns per task
constexpr int NCW = 8;                // consumer warps
constexpr int CTHREADS = NCW * 32;    // consumer threads
constexpr int THREADS = CTHREADS + 32;  // + one producer warp
constexpr int STAGES = 20;            // operand ring (k8 slices)
constexpr int LS = 2;                 // level-data ring (perm + b_{l+1}, or y_l rows)

__host__ __device__ __forceinline__ int mtiles_of(int total, int r) {  // m tiles owned by CTA r (contiguous)
  const int base = total / G, rem = total % G;
  return base + (r < rem ? 1 : 0);
}
__host__ __device__ __forceinline__ int mtile0_of(int total, int r) {
  const int base = total / G, rem = total % G;
  return r * base + (r < rem ? r : rem);
}

struct SolveLay {  // shared-memory layout, in doubles unless noted
  int WC, slot_d, ldd;
  int64_t z, tt, xb, stg, lv, u13_byte, bytes;
};
__host__ __device__ inline SolveLay solve_lay(int Wp, int64_t n2) {
  SolveLay L;
  const int MTH = Wp / 8;
  L.WC = Wp * C;
  L.slot_d = 4 * ((MTH + G - 1) / G) * 32;  // one k8 slice: 2 k4 x (top + bottom) tiles of this CTA
  L.ldd = Wp + L.WC;                        // perm (2 Wp int32) + b_{l+1} (Wp x C)
  L.z = 0;
  L.tt = 2 * L.WC;
  L.xb = 3 * L.WC;
  L.stg = 6 * L.WC;
  L.lv = L.stg + (int64_t)STAGES * L.slot_d;
  L.u13_byte = (L.lv + (int64_t)LS * L.ldd) * 8;
  L.bytes = L.u13_byte + round_up(n2, 16);
  return L;
}

// backward level needs the full H (kb slices): U13 != 0 and not representable as <= 8 columns
__device__ __forceinline__ bool bwd_full(uint8_t f, int bsc) { return (f & 1) && !(bsc && !(f & 64) && ((f >> 2) & 15) <= 8); }

__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release;\n" ::: "memory"); }
// Level barrier for shared-memory-only exchange: the CTA-scope fence performs this CTA's shared
// stores before the relaxed arrive, so peers reading them after the wait observe them.
template <bool RELAXED>
__device__ __forceinline__ void cl_arrive_smem() {
  if (RELAXED) {
    __threadfence_block();
    asm volatile("barrier.cluster.arrive.relaxed;\n" ::: "memory");
  } else {
    cl_arrive();
  }
}
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire;\n" ::: "memory"); }
__device__ __forceinline__ void consumer_bar() { asm volatile("bar.sync 1, %0;\n" ::"n"(CTHREADS) : "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;\n" ::: "memory"); }

// b_l of every (task, level) in level-major tile order: ybuf[task][l][i][n] (rows i >= w and columns
// n >= ncols are zero).  Recover mode folds the interface couplings in (stage_one.hpp:447-455).
__global__ void __launch_bounds__(256) rhs_pack_kernel(SchurArgs a) {
  const int task = blockIdx.x;
  const int s = a.tasks[3 * task];
  const int64_t q0 = a.tasks[3 * task + 2];
  const StripDesc sd = a.strips[s];
  const int Wp = a.Wp;
  const int64_t n2 = a.n2;
  const int n = threadIdx.x & 7;
  const int64_t L = (int64_t)blockIdx.y * 32 + (threadIdx.x >> 3);
  if (L >= n2) return;
  const int64_t rem = a.nrhs - q0;
  const bool live = n < (rem < C ? rem : C);
  const int64_t col = q0 + n;
  const double* cpl = a.cpl + s * a.sCPL;
  double ul = 0.0, ur = 0.0;
  if (live && a.mode == SWEEP_RECOVER) {
    if (sd.left >= 0) ul = a.u_ifc[col * a.K + (int64_t)sd.left * n2 + L];
    if (sd.right >= 0) ur = a.u_ifc[col * a.K + (int64_t)sd.right * n2 + L];
  }
  double* out = a.ybuf + (int64_t)task * a.sY + L * Wp * C + n;
  const double* fc = a.f + col * a.N + (int64_t)sd.col0 * n2 + L;
  for (int i = 0; i < Wp; i++) {
    double v = 0.0;
    if (live && i < sd.w) {
      v = fc[(int64_t)i * n2];
      if (a.mode == SWEEP_RECOVER) {
        if (sd.left >= 0) v -= cpl[L * Wp + i] * ul;
        if (sd.right >= 0) v -= cpl[n2 * Wp + L * Wp + i] * ur;
      }
    }
    out[i * C] = v;
  }
}

// One task = (strip, C RHS columns) on a cluster of G CTAs.  Warp NCW is the producer: it streams
// this CTA's m-tile slice of every level operator (F forward, H backward) with bulk copies into an
// mbarrier ring, plus the per-level data (pivot order + b_{l+1} forward, own rows of y_l backward)
// into a second ring.  Consumer warps run the DMMA GEMVs.  The forward reads z_l straight from the
// owning CTA's shared memory (DSMEM); the backward all-gathers x_l after the level's cluster barrier.
// The producer takes part in every cluster barrier with split arrive/wait so that it can run ahead.
template <bool RELAXED>
__global__ void __launch_bounds__(THREADS, 1) strip_solve_kernel(SchurArgs a) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];
  __shared__ __align__(8) uint64_t lfull[LS];
  __shared__ __align__(8) uint64_t lempty[LS];
  __shared__ int owner[64];
  const int Wp = a.Wp;
  const int64_t n2 = a.n2;
  const SolveLay Ly = solve_lay(Wp, n2);
  const int WC = Ly.WC;
  const int MTH = Wp / 8, MTF = 2 * MTH;
  const int bm0 = mtile0_of(MTH, rank), bmn = mtiles_of(MTH, rank);  // backward: rows of H
  const int fm0 = mtile0_of(MTF, rank), fmn = mtiles_of(MTF, rank);  // forward: contiguous [Ainv ; Fbot] tiles
  double* z = sm + Ly.z;  // [2][Wp x C] z_l parity buffers (own rows valid after level 0)
  double* tt = sm + Ly.tt;
  double* xb = sm + Ly.xb;  // [3][Wp x C] x_l, x_{l+1}, x_{l+2}
  double* stg = sm + Ly.stg;
  double* lv = sm + Ly.lv;
  uint8_t* su13 = reinterpret_cast<uint8_t*>(sm) + Ly.u13_byte;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;

  const int task = blockIdx.x / G;
  const int s = a.tasks[3 * task];
  const int q0 = a.tasks[3 * task + 2];
  const StripDesc sd = a.strips[s];
  const double* fac = a.fac + s * a.sF;
  const int32_t* permg = a.perm + s * a.sP;
  const double* cpl = a.cpl + s * a.sCPL;
  const double* toL = cpl + 2 * n2 * Wp;
  const double* toR = cpl + 3 * n2 * Wp;
  const int64_t lvl = 4LL * Wp * Wp;
  const int kf = Wp / 8, kb = Wp / 4;
  const int64_t rem = a.nrhs - q0;
  const int ncols = (int)(rem < C ? rem : C);
  double* ybase = a.ybuf + (int64_t)task * a.sY;  // b_l (packed) in, y_l out: n2 x (Wp x C)

  for (int64_t i = tid; i < n2; i += THREADS) su13[i] = a.u13[s * n2 + i];
  if (tid < MTH) {  // owner of z row tile b = owner of forward tile MTH + b
    int r = 0;
    while (r + 1 < G && mtile0_of(MTF, r + 1) <= MTH + tid) r++;
    owner[tid] = r;
  }
  if (tid == 0) {
    for (int i = 0; i < STAGES; i++) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], NCW);
    }
    for (int i = 0; i < LS; i++) {
      mbar_init(&lfull[i], 1);
      mbar_init(&lempty[i], NCW);
    }
    fence_mbar_init();
  }
  for (int idx = tid; idx < WC; idx += THREADS) z[idx] = ybase[idx];  // z_0 = b_0, full copy
  __syncthreads();
  cluster.sync();

  if (warp == NCW) {
    // ======================= producer warp =======================
    int slot = 0, ls = 0;
    uint32_t eph = 0, lph = 0;
    bool pending = false;
    const int64_t U = 2 * n2;  // units: forward levels 0..n2-1, then backward levels n2-1..0
#ifdef SLB_SOLVE_PROF
    long long Q0 = clock64(), qE = 0, qL = 0, qC = 0, qT0 = Q0;
#define QM(v) { const long long q_ = clock64(); v += q_ - Q0; Q0 = q_; }
#define QS() Q0 = clock64();
#else
#define QM(v)
#define QS()
#endif
    for (int64_t u = 0; u < U; u++) {
      if (u >= 1) {  // cluster barrier u-1 (consumers reach it at the end of unit u-1)
        QS()
        if (pending) cl_wait();
        QM(qC)
        cl_arrive();
        pending = true;
      }
      const bool fwd = u < n2;
      const int64_t l = fwd ? u : U - 1 - u;
      if (u == n2) {  // y_l of the forward must be complete before the backward streams it
        cl_wait();
        pending = false;
        fence_proxy_async_global();
      }
      QS()
      mbar_wait(&lempty[ls], lph ^ 1u);
      QM(qL)
      if (lane == 0) {
        double* dst = lv + ls * Ly.ldd;
        if (fwd) {
          const uint32_t pb = (uint32_t)(2 * Wp * sizeof(int32_t));
          const bool hn = l + 1 < n2;
          const uint32_t bb = hn ? (uint32_t)(WC * 8) : 0u;
          mbar_arrive_expect_tx(&lfull[ls], pb + bb);
          bulk_g2s(dst, permg + l * 2 * Wp, pb, &lfull[ls]);
          if (hn) bulk_g2s(dst + Wp, ybase + (l + 1) * WC, bb, &lfull[ls]);
        } else {
          const uint32_t yb = (uint32_t)bmn * 8 * C * 8;
          mbar_arrive_expect_tx(&lfull[ls], yb);
          if (yb) bulk_g2s(dst, ybase + l * WC + bm0 * 8 * C, yb, &lfull[ls]);
        }
      }
      __syncwarp();
      if (++ls == LS) {
        ls = 0;
        lph ^= 1u;
      }
      const int nsl = fwd ? kf : (bwd_full(su13[l], a.bsc) ? kb : kb / 2);
      const double* base = fac + l * lvl + (fwd ? 0 : 2LL * Wp * Wp);
      for (int j = 0; j < nsl; j++) {
        QS()
        mbar_wait(&empty_bar[slot], eph ^ 1u);
        QM(qE)
        if (lane == 0) {
          double* dst = stg + slot * Ly.slot_d;
          const uint32_t tb = (uint32_t)bmn * 32 * 8;
          if (fwd) {  // one contiguous run of fmn tiles per k4 step
            const uint32_t fb = (uint32_t)fmn * 32 * 8;
            mbar_arrive_expect_tx(&full_bar[slot], 2 * fb);
            if (fb) {
#pragma unroll
              for (int kk = 0; kk < 2; kk++)
                bulk_g2s(dst + kk * fmn * 32, base + ((int64_t)(2 * j + kk) * MTF + fm0) * 32, fb, &full_bar[slot]);
            }
          } else {
            mbar_arrive_expect_tx(&full_bar[slot], 2 * tb);
            if (tb) {
#pragma unroll
              for (int kk = 0; kk < 2; kk++)
                bulk_g2s(dst + kk * bmn * 32, base + ((int64_t)(2 * j + kk) * MTH + bm0) * 32, tb, &full_bar[slot]);
            }
          }
        }
        __syncwarp();
        if (++slot == STAGES) {
          slot = 0;
          eph ^= 1u;
        }
      }
    }
#ifdef SLB_SOLVE_PROF
    if (blockIdx.x < 2 && lane == 0)
      printf("PROD[%d] total %lld emptywait %lld lemptywait %lld clwait %lld\n", blockIdx.x, clock64() - qT0, qE, qL, qC);
#endif
    if (pending) cl_wait();
    cl_arrive();  // barrier U-1
    cl_wait();
    cl_arrive();  // final barrier
    cl_wait();
    return;
  }

  // ======================= consumer warps =======================
  int slot = 0, ls = 0;
  uint32_t fph = 0, lph = 0;
  int zp = 0;
#ifdef SLB_SOLVE_PROF
  long long P0 = clock64(), ph[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#define PROF_MARK(k) { const long long q_ = clock64(); ph[k] += q_ - P0; P0 = q_; }
#else
#define PROF_MARK(k)
#endif
  for (int64_t l = 0; l < n2; l++) {
    const bool hn = l + 1 < n2;
    const int zo = zp * WC;
    double* zn = z + (1 - zp) * WC;
    mbar_wait(&lfull[ls], lph);
    PROF_MARK(0)
    const int* sperm = reinterpret_cast<const int*>(lv + ls * Ly.ldd);
    const double* bn = lv + ls * Ly.ldd + Wp;
    auto vval = [&](int src, int n) -> double {
      if (src < Wp) {
        const int o = owner[src >> 3];
        const double* zs = (l == 0 || o == rank) ? z : cluster.map_shared_rank(z, o);
        return zs[zo + src * C + n];
      }
      return hn ? bn[(src - Wp) * C + n] : 0.0;
    };
    {  // t_top = (perm [z_l ; b_{l+1}])[0:Wp]: issue every (remote) load before the first store
      constexpr int TMAX = 8;  // Wp * C / CTHREADS <= 8 for Wp <= 256
      double v[TMAX];
#pragma unroll
      for (int k = 0; k < TMAX; k++) {
        const int idx = tid + k * CTHREADS;
        v[k] = idx < WC ? vval(sperm[idx >> 3], idx & 7) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < TMAX; k++) {
        const int idx = tid + k * CTHREADS;
        if (idx < WC) tt[idx] = v[k];
      }
    }
    // warp w owns local tiles w, w+8 of this CTA's fmn forward tiles fm0.. (global tile < MTH:
    // a row of y_l, else a row of z_{l+1})
    double acc[2][2];
    int lts[2];
#pragma unroll
    for (int u = 0; u < 2; u++) {
      const int lt = warp + 8 * u;
      lts[u] = lt < fmn ? lt : -1;
      acc[u][0] = acc[u][1] = 0.0;
      if (lts[u] >= 0 && fm0 + lt >= MTH) {  // bottom half: z_{l+1} = t_bot + Fbot t_top
        const int src = sperm[Wp + (fm0 + lt - MTH) * 8 + g];
        acc[u][0] = vval(src, 2 * t);
        acc[u][1] = vval(src, 2 * t + 1);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&lempty[ls]);
    if (++ls == LS) {
      ls = 0;
      lph ^= 1u;
    }
    PROF_MARK(1)
    consumer_bar();
    PROF_MARK(2)
    for (int j = 0; j < kf; j++) {
      mbar_wait(&full_bar[slot], fph);
      const double* A = stg + slot * Ly.slot_d;
#pragma unroll
      for (int kk = 0; kk < 2; kk++) {
        const double bf = tt[(j * 8 + kk * 4 + t) * C + g];
#pragma unroll
        for (int u = 0; u < 2; u++)
          if (lts[u] >= 0) dmma884(acc[u][0], acc[u][1], A[kk * fmn * 32 + lts[u] * 32 + lane], bf);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[slot]);
      if (++slot == STAGES) {
        slot = 0;
        fph ^= 1u;
      }
    }
    PROF_MARK(3)
    double* ylev = ybase + l * (int64_t)WC;
#pragma unroll
    for (int u = 0; u < 2; u++) {
      if (lts[u] < 0) continue;
      const int mt = fm0 + lts[u];
      if (mt < MTH) {
        const int row = mt * 8 + g;
        ylev[row * C + 2 * t] = acc[u][0];
        ylev[row * C + 2 * t + 1] = acc[u][1];
      } else {
        const int row = (mt - MTH) * 8 + g;
        zn[row * C + 2 * t] = acc[u][0];
        zn[row * C + 2 * t + 1] = acc[u][1];
      }
    }
    if (l == n2 - 1) {
      fence_proxy_async_global();  // y is streamed back by the producer's bulk copies
      cl_arrive();
    } else {
      cl_arrive_smem<RELAXED>();
    }
    cl_wait();
    PROF_MARK(4)
    zp ^= 1;
  }

  // ---------------- backward ----------------
  for (int idx = tid; idx < 3 * WC; idx += CTHREADS) xb[idx] = 0.0;
  consumer_bar();
  int i1 = 1, i2 = 2, i0 = 0;  // x_{l+1} in xb[i1], x_{l+2} in xb[i2], x_l written into xb[i0]
  for (int64_t l = n2 - 1; l >= 0; l--) {
    const uint8_t fl = su13[l];
    const int kbl = bwd_full(fl, a.bsc) ? kb : kb / 2;
    const int nhc = ((fl & 1) && !bwd_full(fl, a.bsc)) ? ((fl >> 2) & 15) : 0;
    const double* x1 = xb + i1 * WC;
    const double* x2 = xb + i2 * WC;
    double* x0 = xb + i0 * WC;
    mbar_wait(&lfull[ls], lph);
    PROF_MARK(5)
    const double* yown = lv + ls * Ly.ldd;  // rows bm0*8 .. (bm0+bmn)*8 of y_l
    double acc[2][2];
    int lts[2];
#pragma unroll
    for (int u = 0; u < 2; u++) {
      const int lt = warp + 8 * u;
      lts[u] = lt < bmn ? lt : -1;
      acc[u][0] = acc[u][1] = 0.0;
      if (lts[u] >= 0) {
        acc[u][0] = -yown[(lt * 8 + g) * C + 2 * t];
        acc[u][1] = -yown[(lt * 8 + g) * C + 2 * t + 1];
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&lempty[ls]);
    if (++ls == LS) {
      ls = 0;
      lph ^= 1u;
    }
    PROF_MARK(6)
    for (int j = 0; j < kbl; j++) {
      mbar_wait(&full_bar[slot], fph);
      const double* A = stg + slot * Ly.slot_d;
      const double* xs = (j * 8 < Wp) ? x1 : x2;
      const int kbase = (j * 8 < Wp) ? j * 8 : j * 8 - Wp;
#pragma unroll
      for (int kk = 0; kk < 2; kk++) {
        const double bf = xs[(kbase + kk * 4 + t) * C + g];
#pragma unroll
        for (int u = 0; u < 2; u++)
          if (lts[u] >= 0) dmma884(acc[u][0], acc[u][1], A[kk * bmn * 32 + lts[u] * 32 + lane], bf);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[slot]);
      if (++slot == STAGES) {
        slot = 0;
        fph ^= 1u;
      }
    }
    if (nhc > 0) {  // x_{l+2} half of H: the columns of the rows pivoted up (schur.cu)
      const int64_t li = (int64_t)s * n2 + l;
      for (int e = 0; e < nhc; e++) {
        const int r = a.hidx[li * 8 + e];
        const double* hc = a.hcol + (li * 8 + e) * Wp;
#pragma unroll
        for (int u = 0; u < 2; u++) {
          if (lts[u] < 0) continue;
          const double hv = hc[(bm0 + lts[u]) * 8 + g];
          acc[u][0] = fma(hv, x2[r * C + 2 * t], acc[u][0]);
          acc[u][1] = fma(hv, x2[r * C + 2 * t + 1], acc[u][1]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 2; u++) {
      if (lts[u] < 0) continue;
      const int row = (bm0 + lts[u]) * 8 + g;
      x0[row * C + 2 * t] = -acc[u][0];
      x0[row * C + 2 * t + 1] = -acc[u][1];
    }
    PROF_MARK(7)
    cl_arrive_smem<RELAXED>();
    cl_wait();
    PROF_MARK(8)
    for (int r = 0; r < G; r++) {
      if (r == rank) continue;
      const int m0 = mtile0_of(MTH, r), mn = mtiles_of(MTH, r);
      const double* rx = cluster.map_shared_rank(x0, r);
      for (int idx = tid; idx < mn * 8 * C; idx += CTHREADS) {
        const int e = m0 * 8 * C + idx;
        x0[e] = rx[e];
      }
    }
    consumer_bar();
    if (a.mode == SWEEP_RECOVER) {
      // each CTA writes its own row slice
      const int r0 = bm0 * 8, r1 = min((bm0 + bmn) * 8, sd.w);
      for (int idx = tid; idx < (r1 - r0) * ncols; idx += CTHREADS) {
        const int i = r0 + idx % (r1 - r0), n = idx / (r1 - r0);
        a.out[(q0 + n) * a.N + (int64_t)(sd.col0 + i) * n2 + l] = x0[i * C + n];
      }
    } else if (rank == 0) {
      // contrib[s][X][col][l] = to_X[l] . x_l[:, col]
      const int X = tid / 128, n = (tid / 16) % C, part = tid % 16;
      const double* tv = (X == 0 ? toL : toR) + l * Wp;
      double sum = 0.0;
      for (int i = part; i < Wp; i += 16) sum = fma(tv[i], x0[i * C + n], sum);
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      const bool has = X == 0 ? sd.left >= 0 : sd.right >= 0;
      if (part == 0 && has && n < ncols) a.out[((int64_t)(s * 2 + X) * a.nrhs + q0 + n) * n2 + l] = sum;
    }
    PROF_MARK(9)
    const int tmp = i2;
    i2 = i1;
    i1 = i0;
    i0 = tmp;
  }
#ifdef SLB_SOLVE_PROF
  if (blockIdx.x < 2 && tid == 0)
    printf("SOLVE[%d] n2=%lld fwd: lfull %lld tt %lld bar %lld kloop %lld epi+cl %lld | bwd: lfull %lld init %lld kloop %lld cl %lld gather+out %lld\n",
           blockIdx.x, (long long)n2, ph[0], ph[1], ph[2], ph[3], ph[4], ph[5], ph[6], ph[7], ph[8], ph[9]);
#endif
  cl_arrive();  // no CTA leaves while a peer may still read its shared memory
  cl_wait();
}

}  // namespace

void strip_rhs_pack(cudaStream_t st, const SchurArgs& a, int ntasks) {
  rhs_pack_kernel<<<dim3((unsigned)ntasks, (unsigned)cdiv(a.n2, 32)), 256, 0, st>>>(a); count_launch();
  SLB_CUDA_CHECK(cudaGetLastError());
}

bool strip_solve_fits(int Wp, int64_t n2) {
  const int MTH = Wp / 8;
  if (MTH > 64 || (MTH + G - 1) / G > 8) return false;
  return solve_lay(Wp, n2).bytes <= 227 * 1024 - 1024;
}

void strip_solve(cudaStream_t st, const SchurArgs& a, int ntasks) {
  const int Wp = a.Wp;
  if (!strip_solve_fits(Wp, a.n2))
    throw CudaFailure(cudaErrorInvalidValue, "strip_solve: slab too wide for the cluster split", __FILE__, __LINE__);
  rhs_pack_kernel<<<dim3((unsigned)ntasks, (unsigned)cdiv(a.n2, 32)), 256, 0, st>>>(a); count_launch();
  SLB_CUDA_CHECK(cudaGetLastError());
  const size_t smem = (size_t)solve_lay(Wp, a.n2).bytes;
  static const bool relaxed = [] {
    const char* e = getenv("SLB_SOLVE_BARRIER");
    return !(e && e[0] == 'r' && e[1] == 'e' && e[2] == 'l' && e[3] == 'e');  // "release": full-scope barrier
  }();
  auto kern = relaxed ? strip_solve_kernel<true> : strip_solve_kernel<false>;
  static size_t attr[2] = {0, 0};
  if (smem > attr[relaxed]) {
    SLB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr[relaxed] = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(G * ntasks));
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = G;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  SLB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, a)); count_launch();
}

}  // namespace slb
