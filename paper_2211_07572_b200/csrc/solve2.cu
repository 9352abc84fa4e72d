// Slab sweeps of the solve phase (reduce_rhs / recover_interiors), version 2:
// thread-block clusters fed by TMA tensor copies, with data-driven level
// exchange (st.async into the peers' shared memory, completion counted on the
// peers' mbarriers: no cluster barrier per level).
//
// Reference: reduce_rhs (proj/include/slablu/stage_one.hpp:415-433) and
// recover_interiors (:438-462): one dgbtrs with nrhs columns per slab
// (banded.hpp:116-128).  Here A_ii^{-1} is applied as the level recurrences of
// band_lu.cu's GEMM form:
//   forward   t = perm_l [z_l ; b_{l+1}],  y_l = Ainv_l t_top,
//             z_{l+1} = t_bot + Fbot_l t_top  (= t_bot - d .* y_l on shortcut levels,
//                                               plus <= 8 exceptional rows)
//   backward  x_l = y_l - H_l [x_{l+1} ; x_{l+2}]   (right half of H as <= 8 columns
//                                                     on most levels)
// One task = (strip, C = 8 right-hand-side columns) on a cluster of G CTAs.  CTA r
// owns a contiguous range of the Wp/8 row tiles of every level operator and
// streams only that slice: one 4-D TMA box (32 doubles x own tiles x half the k4
// rows x 1 level) per half level, so a level costs the producer two
// instructions.  The level's output rows are pushed to every CTA of the cluster
// (itself included) with st.async; each CTA waits for the whole vector on its
// own exchange mbarrier.  The level data the recurrence needs (pivot order,
// b_{l+1}, diag(Lsub), exceptional Fbot rows; y_l rows and H columns in the
// backward) arrive through a second ring fed by a second producer warp.
//
// The bandwidth-bound operator stream (B_solve) is the
// roofline; per level the critical path is one exchange (~0.2 us DSMEM) plus a
// k-split DMMA GEMV over 8 warps.
#include <cooperative_groups.h>
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace slb {
namespace {

constexpr int C = 8;                    // RHS columns per task (DMMA n = 8)
constexpr int NCW = 8;                  // consumer warps
constexpr int CTHREADS = NCW * 32;
constexpr int THREADS = CTHREADS + 64;  // + op producer warp + level producer warp
// DFMA variants need at most 6 row-tile warps (G >= 4 at Wp <= 160): 8 warps in all, so two warps
// per SM sub-partition and the full 255-register budget (10 warps cap threads at 168 registers)
constexpr int NCW_DFMA = 6;
template <int NC>
constexpr int ncw_of() { return NC == 0 ? NCW : NCW_DFMA; }
template <int NC>
constexpr int threads_of() { return ncw_of<NC>() * 32 + 64; }
constexpr int STAGES = 4;               // op ring: half-level chunks
constexpr int LS = 3;                   // level-data ring
constexpr int MNMAX = 8;                // row tiles per CTA (G >= 3 for Wp <= 160)

__host__ __device__ __forceinline__ int mt_cnt(int total, int G, int r) {
  const int base = total / G, rem = total % G;
  return base + (r < rem ? 1 : 0);
}
__host__ __device__ __forceinline__ int mt_first(int total, int G, int r) {
  const int base = total / G, rem = total % G;
  return r * base + (r < rem ? r : rem);
}

struct Lay2 {  // shared-memory layout (bytes)
  int MTH, MNB, KH;
  int64_t op_slot, op, lv_slot, lv, xb, part, flags, bytes;
  // offsets inside a level slot
  int64_t o_perm, o_b, o_dsub, o_epos, o_exc;   // forward
  int64_t o_y, o_hidx, o_hcol;                  // backward
};
__host__ __device__ inline Lay2 lay2(int Wp, int G, int64_t n2) {
  Lay2 L;
  L.MTH = Wp / 8;
  L.MNB = (L.MTH + G - 1) / G;
  L.KH = Wp / 8;  // k4 rows per half level
  L.op_slot = (int64_t)L.KH * L.MNB * 32 * 8;
  L.op = 0;
  L.o_perm = 0;
  L.o_b = L.o_perm + 2 * Wp * 4;
  L.o_dsub = L.o_b + (int64_t)Wp * C * 8;
  L.o_epos = L.o_dsub + (int64_t)Wp * 8;
  L.o_exc = L.o_epos + 64;
  L.o_y = 0;
  L.o_hidx = L.o_y + (int64_t)L.MNB * 8 * C * 8;
  L.o_hcol = L.o_hidx + 64;
  const int64_t fwd_slot = L.o_exc + 8LL * Wp * 8;
  const int64_t bwd_slot = L.o_hcol + 8LL * Wp * 8;
  L.lv_slot = fwd_slot > bwd_slot ? fwd_slot : bwd_slot;
  L.lv = L.op + STAGES * L.op_slot;
  L.xb = L.lv + LS * L.lv_slot;
  L.part = L.xb + 3LL * Wp * C * 8;
  // DMMA partial sums, or (DFMA, NC <= 2) one private t_top copy per row-tile warp
  L.flags = L.part + (int64_t)NCW * L.MNB * 32 * 16;  // DMMA partial sums
  L.bytes = L.flags + round_up(n2, 16) + 128;  // + alignment slack of the dynamic window
  return L;
}

struct Solve2Args {
  SchurArgs a;
  int G;
};

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
// 16-byte store into the shared memory of a cluster CTA, counted on that CTA's mbarrier
__device__ __forceinline__ void consumer_bar() { asm volatile("bar.sync 1, %0;\n" ::"n"(CTHREADS) : "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;\n" ::: "memory"); }

__device__ __forceinline__ bool fwd_shortcut(uint8_t f, int fsc) { return fsc && (f & 2) == 0 && (f >> 2) <= 8; }
__device__ __forceinline__ bool bwd_full2(uint8_t f, int bsc) {
  return (f & 1) && !(bsc && !(f & 64) && ((f >> 2) & 15) <= 8);
}

// acc0/acc1 += A rows (fragment order: lane (g, t) holds A[g][4 k4 + t]) times b[k4 * bstride + n],
// two interleaved accumulator sets for ILP (explicit pairs: a runtime parity index would spill).
template <int NC>
__device__ __forceinline__ void gemv_rows(const double* Aop, int MNB, const double* b, int bstride, int KH,
                                          double (&acc0)[NC], double (&acc1)[NC]) {
  int k4 = 0;
#pragma unroll 2
  for (; k4 + 1 < KH; k4 += 2) {
    const double a0 = Aop[(int64_t)k4 * MNB * 32], a1 = Aop[(int64_t)(k4 + 1) * MNB * 32];
#pragma unroll
    for (int n = 0; n < NC; n++) {
      acc0[n] = fma(a0, b[k4 * bstride + n], acc0[n]);
      acc1[n] = fma(a1, b[(k4 + 1) * bstride + n], acc1[n]);
    }
  }
  if (k4 < KH) {
    const double a0 = Aop[(int64_t)k4 * MNB * 32];
#pragma unroll
    for (int n = 0; n < NC; n++) acc0[n] = fma(a0, b[k4 * bstride + n], acc0[n]);
  }
}

// Prefetched form: the right-hand-side values of a chunk sit in registers (gathered before the
// operator slice is waited for), KMAX = 20 k4 rows unrolled with predication (KH <= 20 for Wp <= 160).
constexpr int KMAX = 20;
// k4 rows gathered per batch (register budget: 4 columns take two batches)
template <int NC>
constexpr int kbatch() { return NC >= 4 ? KMAX / 2 : KMAX; }
template <int NC>
__device__ __forceinline__ void gemv_pref(const double* Aop, int MNB, const double (&bv)[kbatch<NC>()][NC], int k0,
                                          int KH, double (&acc0)[NC], double (&acc1)[NC]) {
  constexpr int KB = kbatch<NC>();
  double av[KB];
#pragma unroll
  for (int k = 0; k < KB; k++) av[k] = k0 + k < KH ? Aop[(int64_t)(k0 + k) * MNB * 32] : 0.0;
#pragma unroll
  for (int k = 0; k < KB; k++)
#pragma unroll
    for (int n = 0; n < NC; n++) {
      if (k & 1) acc1[n] = fma(av[k], bv[k][n], acc1[n]);
      else acc0[n] = fma(av[k], bv[k][n], acc0[n]);
    }
}

// Fully unrolled form for a compile-time chunk height K (no predicates): all A and b loads first,
// then two interleaved FMA chains.  Aw = this lane's element of k4 row 0, S = doubles per k4 row;
// b rows at bw[k * BS + n].
template <int NC, int K, int BS>
__device__ __forceinline__ void gemv_fixed(const double* Aw, int S, const double* bw, double (&acc0)[NC],
                                           double (&acc1)[NC]) {
  double av[K], bv[K][NC];
#pragma unroll
  for (int k = 0; k < K; k++) {
    av[k] = Aw[k * S];
#pragma unroll
    for (int n = 0; n < NC; n++) bv[k][n] = bw[k * BS + n];
  }
#pragma unroll
  for (int k = 0; k < K; k++)
#pragma unroll
    for (int n = 0; n < NC; n++) {
      if (k & 1) acc1[n] = fma(av[k], bv[k][n], acc1[n]);
      else acc0[n] = fma(av[k], bv[k][n], acc0[n]);
    }
}
// KH (k4 rows of a chunk, Wp / 8 <= 20) dispatched to its unrolled form (warp-uniform jump)
template <int NC, int BS>
__device__ __forceinline__ void gemv_k(int KH, const double* Aw, int S, const double* bw, double (&acc0)[NC],
                                       double (&acc1)[NC]) {
  switch (KH) {
#define SLB_K(k) \
  case k: gemv_fixed<NC, k, BS>(Aw, S, bw, acc0, acc1); break;
    SLB_K(1) SLB_K(2) SLB_K(3) SLB_K(4) SLB_K(5) SLB_K(6) SLB_K(7) SLB_K(8) SLB_K(9) SLB_K(10)
    SLB_K(11) SLB_K(12) SLB_K(13) SLB_K(14) SLB_K(15) SLB_K(16) SLB_K(17) SLB_K(18) SLB_K(19) SLB_K(20)
#undef SLB_K
    default: break;
  }
}

// DFMA consumer (see strip_solve2_kernel): warp w < mn owns row tile w for the whole k range.
// (Splitting a tile's k range over two warps combined through shared memory measured the same
// time at cfg3 and was dropped.)
template <int NC>
__device__ __forceinline__ void solve2_dfma_consumer(const SchurArgs& a, int G, int rank, int m0, int mn, int w,
                                                     int lane, int Wp, int64_t n2, const Lay2& Ly,
                                                     unsigned char* smraw, double* xbuf, const uint8_t* sfl,
                                                     uint64_t* full_bar, uint64_t* empty_bar, uint64_t* lfull,
                                                     uint64_t* lempty, uint64_t* xbar, uint64_t* fwd_done,
                                                     double* ybase, int ncols, int q0, const StripDesc& sd) {
  const int g = lane >> 2, t = lane & 3;
  const int KH = Ly.KH, MNB = Ly.MNB;
  const int WC = Wp * C;    // packed level-major layout of b / y / x in HBM and the level ring
  const int XW = Wp * NC;   // one exchange vector: [row][NC] (compact: row gathers stay bank-conflict-free)
  const int tile = w;                   // row tile of this warp
  const int row = (m0 + tile) * 8 + g;  // this lane's output row (all 4 t lanes hold the reduced sums)
  const uint32_t xbytes = (uint32_t)(Wp * NC * 8);
  int slot = 0, ls = 0;
  uint32_t fph = 0, lph = 0, xq = 0;
  auto arm = [&]() {
    if (w == 0 && lane == 0) mbar_arrive_expect_tx(&xbar[xq & 1], xbytes);
  };
  auto wait_x = [&]() {
    mbar_wait(&xbar[xq & 1], (xq >> 1) & 1u);
    xq++;
  };
  auto acquire_op = [&]() -> const double* {
    mbar_wait(&full_bar[slot], fph);
    return reinterpret_cast<const double*>(smraw + Ly.op + (int64_t)slot * Ly.op_slot);
  };
  auto next_slot = [&]() {
    if (++slot == STAGES) {
      slot = 0;
      fph ^= 1u;
    }
  };
  auto release_op = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[slot]);
    next_slot();
  };
  auto release_lv = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive(&lempty[ls]);
    if (++ls == LS) {
      ls = 0;
      lph ^= 1u;
    }
  };
  // sum over the 4 t lanes of a row: every lane ends with the row's totals
  auto rowsum = [&](double (&acc)[NC]) {
#pragma unroll
    for (int n = 0; n < NC; n++) {
      acc[n] += __shfl_xor_sync(0xffffffffu, acc[n], 1);
      acc[n] += __shfl_xor_sync(0xffffffffu, acc[n], 2);
    }
  };
  auto pick = [&](const double (&v)[NC]) -> double {  // column t of a row vector (t < NC)
    double r = v[0];
#pragma unroll
    for (int n = 1; n < NC; n++)
      if (t == n) r = v[n];
    return r;
  };
#ifdef SLB_SOLVE_PROF
  long long P0 = clock64(), ph[24] = {0};
#define PN(k) { const long long q_ = clock64(); ph[k] += q_ - P0; P0 = q_; }
#else
#define PN(k)
#endif
  // lane t pushes the row's NC values (gathered from the 4 t lanes) to cluster CTAs t and t + 4: the
  // G pushes of a row go out in parallel, one st.async per lane
  const int tc = t < NC ? t : 0;
  const uint32_t rxa = dsmem_map(xbuf, t < G ? t : 0), rxb = dsmem_map(xbuf, t + 4 < G ? t + 4 : 0);
  const uint32_t rb0a = dsmem_map(&xbar[0], t < G ? t : 0), rb0b = dsmem_map(&xbar[0], t + 4 < G ? t + 4 : 0);
  const uint32_t rb1a = dsmem_map(&xbar[1], t < G ? t : 0), rb1b = dsmem_map(&xbar[1], t + 4 < G ? t + 4 : 0);
  auto push_row = [&](int buf, double v) {
    double vv[NC];
#pragma unroll
    for (int n = 0; n < NC; n++) vv[n] = __shfl_sync(0xffffffffu, v, (lane & ~3) + n);
    const uint32_t off = (uint32_t)(((buf * Wp + row) * NC) * 8);
    const bool b = xq & 1;
#pragma unroll
    for (int rr = 0; rr < 8; rr += 4) {
      if (rr + t >= G) continue;
      const uint32_t dst = (rr ? rxb : rxa) + off, bar = b ? (rr ? rb1b : rb1a) : (rr ? rb0b : rb0a);
      if constexpr (NC == 1) {
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];\n" ::"r"(dst),
                     "d"(vv[0]), "r"(bar)
                     : "memory");
      } else {
#ifdef SLB_NC2_SCALAR
#pragma unroll
        for (int n = 0; n < NC; n++)
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];\n" ::"r"(dst + n * 8),
                       "d"(vv[n]), "r"(bar)
                       : "memory");
#else
#pragma unroll
        for (int n = 0; n < NC; n += 2) st_async_v2(dst + n * 8, vv[n], vv[n + 1], bar);
#endif
      }
    }
  };
  // ---------------- forward ----------------
  double* tt = xbuf + 2 * XW;  // t_top, one shared copy built by all active warps
  for (int64_t l = 0; l < n2; l++) {
    const bool hn = l + 1 < n2;
    const uint8_t fl = sfl[l];
    const bool sc = fwd_shortcut(fl, a.fsc);
    const double* z = xbuf + (int)(l & 1) * XW;
    PN(7)
    if (l > 0) wait_x();
    if (hn) arm();
    PN(0)
    mbar_wait(&lfull[ls], lph);
    PN(1)
    const unsigned char* lv = smraw + Ly.lv + (int64_t)ls * Ly.lv_slot;
    const int* sperm = reinterpret_cast<const int*>(lv + Ly.o_perm);
    const double* bn = reinterpret_cast<const double*>(lv + Ly.o_b);
    auto val = [&](int src, int n) -> double {  // row src, column n of [z_l ; b_{l+1}]
      if (src < Wp) return z[src * NC + n];
      return hn ? bn[(src - Wp) * C + n] : 0.0;
    };
    // t_top = rows perm[0..Wp) of [z_l ; b_{l+1}], compact [k][NC].  Reuse is safe: the next
    // level rewrites it only after its exchange wait, which needs this level's pushes.
    for (int idx = w * 32 + lane; idx < Wp * NC; idx += mn * 32) tt[idx] = val(sperm[idx / NC], idx % NC);
    asm volatile("bar.sync 2, %0;\n" ::"r"(mn * 32) : "memory");
    PN(2)
    // epilogue operands ahead of the GEMV: t_bot, diag(Lsub), and the exceptional rows of this
    // tile (z = t_bot + Fbot[e, :] t_top needs t_top only)
    double tb = 0.0, d = 0.0;
    double exq[NC];
    bool is_exc = false;
#pragma unroll
    for (int n = 0; n < NC; n++) exq[n] = 0.0;
    if (hn) {
      tb = val(sperm[Wp + row], tc);
      if (sc) {
        d = reinterpret_cast<const double*>(lv + Ly.o_dsub)[row];
        const int ncx = (fl >> 2) & 15;
        const int* epos = reinterpret_cast<const int*>(lv + Ly.o_epos);
        const double* exc = reinterpret_cast<const double*>(lv + Ly.o_exc);
        for (int e = 0; e < ncx; e++) {
          const int er = epos[e];
          if (er < (m0 + tile) * 8 || er >= (m0 + tile) * 8 + 8) continue;  // warp-uniform
          double q[NC];
#pragma unroll
          for (int n = 0; n < NC; n++) q[n] = 0.0;
          for (int k = lane; k < Wp; k += 32) {
            const double ev = exc[e * Wp + k];
#pragma unroll
            for (int n = 0; n < NC; n++) q[n] = fma(ev, tt[k * NC + n], q[n]);
          }
#pragma unroll
          for (int n = 0; n < NC; n++) {
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) q[n] += __shfl_xor_sync(0xffffffffu, q[n], o);
            if (row == er) exq[n] = q[n];
          }
          if (row == er) is_exc = true;
        }
      }
    }
    PN(14)
    double acc[2][NC], acc2[2][NC];
#pragma unroll
    for (int n = 0; n < NC; n++) acc[0][n] = acc[1][n] = acc2[0][n] = acc2[1][n] = 0.0;
    const int nch = (sc || !hn) ? 2 : 4;
    for (int c = 0; c < nch; c++) {
      const double* tk = tt + ((c & 1) * KH * 4 + t) * NC;
      const double* Aw = acquire_op() + tile * 32 + lane;
      PN(5)
      if (c < 2) gemv_k<NC, 4 * NC>(KH, Aw, MNB * 32, tk, acc[0], acc[1]);
      else gemv_k<NC, 4 * NC>(KH, Aw, MNB * 32, tk, acc2[0], acc2[1]);
      release_op();
      PN(6)
    }
#pragma unroll
    for (int n = 0; n < NC; n++) {
      acc[0][n] += acc[1][n];
      acc2[0][n] += acc2[1][n];
    }
    {
      rowsum(acc[0]);
      const double yv = pick(acc[0]);
      if (hn) {
        double zv;
        if (sc) {
          zv = is_exc ? tb + pick(exq) : fma(-d, yv, tb);
        } else {
          rowsum(acc2[0]);
          zv = tb + pick(acc2[0]);
        }
        push_row((int)((l + 1) & 1), zv);
      }
      PN(15)
      if (t < NC) ybase[l * WC + row * C + t] = yv;  // y_l -> HBM (read back by the backward sweep)
    }
    PN(4)
    release_lv();
  }
  fence_proxy_async_global();
  __syncwarp();
  if (lane == 0) mbar_arrive(fwd_done);

  // ---------------- backward ----------------
  for (int idx = w * 32 + lane; idx < 3 * XW; idx += mn * 32) xbuf[idx] = 0.0;
  asm volatile("barrier.cluster.arrive.release;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire;\n" ::: "memory");
  for (int64_t l = n2 - 1; l >= 0; l--) {
    const uint8_t fl = sfl[l];
    const bool full = bwd_full2(fl, a.bsc);
    const int nhc = ((fl & 1) && !full) ? ((fl >> 2) & 15) : 0;
    const int b0 = (int)(l % 3);
    const double* x1 = xbuf + (int)((l + 1) % 3) * XW;
    const double* x2 = xbuf + (int)((l + 2) % 3) * XW;
    PN(8)
    if (l < n2 - 1) wait_x();
    arm();
    PN(9)
    mbar_wait(&lfull[ls], lph);
    PN(10)
    const unsigned char* lv = smraw + Ly.lv + (int64_t)ls * Ly.lv_slot;
    // y_l and the x_{l+2} columns of H ahead of the GEMV
    double xv = 0.0;
    {
      xv = reinterpret_cast<const double*>(lv + Ly.o_y)[(tile * 8 + g) * C + tc];
      if (nhc) {  // x_{l+2} half of H: the columns of the rows pivoted up
        const int* hidx = reinterpret_cast<const int*>(lv + Ly.o_hidx);
        const double* hcol = reinterpret_cast<const double*>(lv + Ly.o_hcol);
        for (int e = 0; e < nhc; e++) xv = fma(-hcol[e * Wp + row], x2[hidx[e] * NC + tc], xv);
      }
    }
    PN(17)
    double acc[2][NC];
#pragma unroll
    for (int n = 0; n < NC; n++) acc[0][n] = acc[1][n] = 0.0;
    const int nch = full ? 4 : 2;
    for (int c = 0; c < nch; c++) {
      const double* xs = (c < 2 ? x1 : x2) + ((c & 1) * KH * 4 + t) * NC;
      const double* Aw = acquire_op() + tile * 32 + lane;
      PN(11)
      gemv_k<NC, 4 * NC>(KH, Aw, MNB * 32, xs, acc[0], acc[1]);
      release_op();
      PN(12)
    }
#pragma unroll
    for (int n = 0; n < NC; n++) acc[0][n] += acc[1][n];
    {
      rowsum(acc[0]);
      xv -= pick(acc[0]);
      push_row(b0, xv);
      if (t < NC) {
        if (a.mode == SWEEP_RECOVER) {
          if (row < sd.w && t < ncols) a.out[(int64_t)(q0 + t) * a.N + (int64_t)(sd.col0 + row) * n2 + l] = xv;
        } else {
          ybase[l * WC + row * C + t] = xv;  // x_l over y_l; to_X x_l in strip_contrib_kernel
        }
      }
    }
    PN(13)
    release_lv();
  }
  wait_x();
#ifdef SLB_SOLVE_PROF
  if (blockIdx.x < G && lane == 0 && w < 2)
    printf("SOLVE2S blk %d w %d G %d mn %d | fwd: xwait %lld lfull %lld tt %lld pre %lld acq %lld gemv %lld epi+push %lld ystore %lld | bwd: xwait %lld "
           "lfull %lld pre %lld acq %lld gemv %lld epi %lld\n",
           blockIdx.x, w, G, mn, ph[0], ph[1], ph[2], ph[14], ph[5], ph[6], ph[15], ph[4], ph[9], ph[10], ph[17], ph[11], ph[12], ph[13]);
#endif
#undef PN
}

// NC = 0: 8 columns, k-split DMMA GEMVs over all 8 consumer warps (one CTA barrier pair per level).
// NC = 1, 2, 4: the first NC columns only, on DFMA (the FP64 tensor pipe gains nothing at 1-4
// columns: DMMA 37.1 vs DFMA 34.1 TF/s measured): consumer warp w < mn owns row tile w for the whole
// k range, gathers its own right-hand-side values through the pivot order, and needs no CTA
// barrier at all - a level is one exchange wait plus a per-warp GEMV and epilogue.
// mapA Ainv tiles, mapF Fbot tiles, mapH H tiles (make_map).
template <int NC>
__global__ void __launch_bounds__(threads_of<NC>(), 1)
    strip_solve2_kernel(const __grid_constant__ Solve2Args A2, const __grid_constant__ CUtensorMap mapA,
                        const __grid_constant__ CUtensorMap mapF, const __grid_constant__ CUtensorMap mapH) {
  const SchurArgs& a = A2.a;
  const int G = A2.G;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  extern __shared__ __align__(128) unsigned char smraw_[];
  // TMA destinations need 128-byte alignment: the dynamic window is over-allocated by 128 bytes
  unsigned char* smraw = smraw_ + ((128 - (smem_u32(smraw_) & 127)) & 127);
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES];
  __shared__ __align__(8) uint64_t lfull[LS], lempty[LS];
  __shared__ __align__(8) uint64_t xbar[2];
  __shared__ __align__(8) uint64_t fwd_done;
  __shared__ double excval[8][C];
  const int Wp = a.Wp;
  const int64_t n2 = a.n2;
  const Lay2 Ly = lay2(Wp, G, n2);
  const int MTH = Ly.MTH, MNB = Ly.MNB, KH = Ly.KH;
  const int m0 = mt_first(MTH, G, rank), mn = mt_cnt(MTH, G, rank);
  const int WC = Wp * C;
  double* xbuf = reinterpret_cast<double*>(smraw + Ly.xb);  // [3][Wp][C]
  double2* part = reinterpret_cast<double2*>(smraw + Ly.part);  // [NCW][MNB][32]
  uint8_t* sfl = smraw + Ly.flags;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;

  const int task = blockIdx.x / G;
  const int s = a.tasks[3 * task];
  const int q0 = a.tasks[3 * task + 2];
  const StripDesc sd = a.strips[s];
  const int64_t rem = a.nrhs - q0;
  const int ncols = (int)(rem < C ? rem : C);
  double* ybase = a.ybuf + (int64_t)task * a.sY;  // b_l in (packed [l][Wp][C]), y_l / x_l out
  const int64_t lvl0 = (int64_t)s * n2;           // this strip's first level in the tensor maps
  // exchange bytes per vector: every CTA pushes its rows to every CTA (itself included)
  const uint32_t xbytes = (uint32_t)(Wp * (NC == 0 ? C : NC) * 8);
  // consumer warps that read the operator / level rings
  const int ncw = NC == 0 ? NCW : mn;

  constexpr int NT = threads_of<NC>();
  constexpr int PW = ncw_of<NC>();  // first producer warp
  for (int64_t i = tid; i < n2; i += NT) sfl[i] = a.u13[s * n2 + i];
  if (tid == 0) {
    for (int i = 0; i < STAGES; i++) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], NC == 0 ? NCW / 2 : mn);  // a chunk is consumed by one warp group (DMMA) / tile set
    }
    for (int i = 0; i < LS; i++) {
      mbar_init(&lfull[i], 1);
      mbar_init(&lempty[i], ncw);
    }
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    mbar_init(&fwd_done, ncw);
    fence_mbar_init();
  }
  // z_0 = b_0 (complete, local): exchange buffer 0 ([row][C] DMMA, [row][NC] DFMA)
  if constexpr (NC == 0) {
    for (int idx = tid; idx < WC; idx += NT) xbuf[idx] = ybase[idx];
  } else {
    for (int idx = tid; idx < Wp * NC; idx += NT) xbuf[idx] = ybase[(idx / NC) * C + idx % NC];
  }
  __syncthreads();
  cluster.sync();  // peers' barriers initialised before any st.async targets them

  const bool idle = warp >= ncw;  // producers and (DFMA path) consumer warps without a row tile
  static_assert(NC == 0 || NCW_DFMA >= 1, "");
  if (idle) {
    // they take part in the one cluster barrier of the consumers (forward -> backward) early
    asm volatile("barrier.cluster.arrive.relaxed;\n" ::: "memory");
  }
  if (warp == PW) {
    // ======================= op producer: level operator slices =======================
    if (lane == 0) {
      int slot = 0;
      uint32_t ph = 0;
      const uint32_t box = (uint32_t)Ly.op_slot;
#ifdef SLB_SOLVE_PROF
      const bool notma = a.fsc == 2;  // timing experiment only: operator slices not loaded
#else
      constexpr bool notma = false;
#endif
      auto put = [&](const CUtensorMap* map, int kbeg, int64_t l) {
        mbar_wait(&empty_bar[slot], ph ^ 1u);
        if (notma) {
          mbar_arrive(&full_bar[slot]);
        } else {
          mbar_arrive_expect_tx(&full_bar[slot], box);
          tma_load_4d(smraw + Ly.op + (int64_t)slot * Ly.op_slot, map, 0, m0, kbeg, (int)(lvl0 + l), &full_bar[slot]);
        }
        if (++slot == STAGES) {
          slot = 0;
          ph ^= 1u;
        }
      };
      for (int64_t l = 0; l < n2; l++) {
        put(&mapA, 0, l);
        put(&mapA, KH, l);
        if (!fwd_shortcut(sfl[l], a.fsc) && l + 1 < n2) {
          put(&mapF, 0, l);
          put(&mapF, KH, l);
        }
      }
      for (int64_t l = n2 - 1; l >= 0; l--) {
        put(&mapH, 0, l);
        put(&mapH, KH, l);
        if (bwd_full2(sfl[l], a.bsc)) {
          put(&mapH, 2 * KH, l);
          put(&mapH, 3 * KH, l);
        }
      }
    }
    __syncwarp();
  } else if (warp == PW + 1) {
    // ======================= level producer: per-level data =======================
    if (lane == 0) {
      int ls = 0;
      uint32_t ph = 0;
      const int32_t* permg = a.perm + s * a.sP;
      const double* dsubg = a.dsub + (int64_t)s * n2 * Wp;
      for (int64_t l = 0; l < n2; l++) {
        const uint8_t f = sfl[l];
        const bool hn = l + 1 < n2;
        const int ncx = (fwd_shortcut(f, a.fsc) && hn) ? ((f >> 2) & 15) : 0;
        mbar_wait(&lempty[ls], ph ^ 1u);
        unsigned char* dst = smraw + Ly.lv + (int64_t)ls * Ly.lv_slot;
        const uint32_t bp = (uint32_t)(2 * Wp * 4), bb = hn ? (uint32_t)(WC * 8) : 0u, bd = (uint32_t)(Wp * 8);
        const uint32_t be = ncx ? 32u : 0u, bx = (uint32_t)(ncx * Wp * 8);
        mbar_arrive_expect_tx(&lfull[ls], bp + bb + bd + be + bx);
        bulk_g2s(dst + Ly.o_perm, permg + l * 2 * Wp, bp, &lfull[ls]);
        if (hn) bulk_g2s(dst + Ly.o_b, ybase + (l + 1) * WC, bb, &lfull[ls]);
        bulk_g2s(dst + Ly.o_dsub, dsubg + l * Wp, bd, &lfull[ls]);
        if (ncx) {
          const int64_t li = (int64_t)s * n2 + l;
          bulk_g2s(dst + Ly.o_epos, a.excpos + li * 8, be, &lfull[ls]);
          bulk_g2s(dst + Ly.o_exc, a.exc + li * 8 * Wp, bx, &lfull[ls]);
        }
        if (++ls == LS) {
          ls = 0;
          ph ^= 1u;
        }
      }
      // y_l rows are written by this CTA's consumers during the forward sweep
      mbar_wait(&fwd_done, 0);
      fence_proxy_async_global();
      for (int64_t l = n2 - 1; l >= 0; l--) {
        const uint8_t f = sfl[l];
        const int nhc = ((f & 1) && !bwd_full2(f, a.bsc)) ? ((f >> 2) & 15) : 0;
        mbar_wait(&lempty[ls], ph ^ 1u);
        unsigned char* dst = smraw + Ly.lv + (int64_t)ls * Ly.lv_slot;
        const uint32_t by = (uint32_t)(mn * 8 * C * 8), bi = nhc ? 32u : 0u, bh = (uint32_t)(nhc * Wp * 8);
        mbar_arrive_expect_tx(&lfull[ls], by + bi + bh);
        bulk_g2s(dst + Ly.o_y, ybase + l * WC + m0 * 8 * C, by, &lfull[ls]);
        if (nhc) {
          const int64_t li = (int64_t)s * n2 + l;
          bulk_g2s(dst + Ly.o_hidx, a.hidx + li * 8, bi, &lfull[ls]);
          bulk_g2s(dst + Ly.o_hcol, a.hcol + li * 8 * Wp, bh, &lfull[ls]);
        }
        if (++ls == LS) {
          ls = 0;
          ph ^= 1u;
        }
      }
    }
    __syncwarp();
  } else if (NC > 0) {
    if (!idle) solve2_dfma_consumer<(NC > 0 ? NC : 1)>(a, G, rank, m0, mn, warp, lane, Wp, n2, Ly, smraw, xbuf, sfl, full_bar,
                                        empty_bar, lfull, lempty, xbar, &fwd_done, ybase, ncols, q0, sd);
  } else {
    // ======================= consumer warps =======================
    int slot = 0, ls = 0;
    uint32_t fph = 0, lph = 0;
    uint32_t xq = 0;  // exchange counter: vector q lands on xbar[q & 1], phase parity (q >> 1) & 1
    const int wg = warp >> 2;         // warp group: even (0) / odd (1) half-level chunks
    const int wk = warp & 3;          // k4 rows [wk * KW, ...) of a chunk
    const int KW = (KH + 3) / 4;
    const int k_lo = wk * KW, k_hi = min(KH, k_lo + KW);
    // epilogue thread: (tile et, lane) of this CTA's rows
    const bool epi = tid < mn * 32;
    const int et = tid >> 5;
    const int erow = (m0 + et) * 8 + g;  // row of the level vector
    // remote addresses of the exchange buffers / barriers (this thread's 16-byte element)
    uint32_t rx[8], rb0[8], rb1[8];
#pragma unroll
    for (int r = 0; r < 8; r++) {
      const int rr = r < G ? r : 0;
      rx[r] = dsmem_map(xbuf, rr);
      rb0[r] = dsmem_map(&xbar[0], rr);
      rb1[r] = dsmem_map(&xbar[1], rr);
    }
    auto push = [&](int buf, int row, double v0, double v1) {  // row `row`, cols 2t, 2t+1 of buffer buf
      const uint32_t off = (uint32_t)(((buf * Wp + row) * C + 2 * t) * 8);
      const bool b = xq & 1;
#pragma unroll
      for (int r = 0; r < 8; r++)
        if (r < G) st_async_v2(rx[r] + off, v0, v1, b ? rb1[r] : rb0[r]);
    };
    auto arm = [&]() {  // this CTA expects exchange xq (every row, every CTA's push)
      if (tid == 0) mbar_arrive_expect_tx(&xbar[xq & 1], xbytes);
    };
    auto wait_x = [&]() {
      mbar_wait(&xbar[xq & 1], (xq >> 1) & 1u);
      xq++;
    };
    auto acquire_op = [&]() -> const double* {
      mbar_wait(&full_bar[slot], fph);
      return reinterpret_cast<const double*>(smraw + Ly.op + (int64_t)slot * Ly.op_slot);
    };
    auto release_op = [&]() {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[slot]);
      if (++slot == STAGES) {
        slot = 0;
        fph ^= 1u;
      }
    };
    // chunk c of a level goes to warp group c & 1; a group skips the other group's chunks
    auto skip_op = [&]() {
      if (++slot == STAGES) {
        slot = 0;
        fph ^= 1u;
      }
    };
    // k-split GEMV of one chunk: acc[mt] += A_chunk[own tiles] * B rows [kb*4, ...) of bsrc
    auto gemv_chunk = [&](const double* Aop, const double* bsrc, int kb, double (*acc)[2]) {
      for (int k4 = k_lo; k4 < k_hi; k4++) {
        const double bf = bsrc[((kb + k4) * 4 + t) * C + g];
        const double* Ak = Aop + (int64_t)k4 * MNB * 32 + lane;
#pragma unroll
        for (int mt = 0; mt < MNMAX; mt++) {
          if (mt >= mn) break;
          dmma884(acc[mt][0], acc[mt][1], Ak[mt * 32], bf);
        }
      }
    };
    auto reduce_parts = [&](double (*acc)[2], double& r0, double& r1) {
#pragma unroll
      for (int mt = 0; mt < MNMAX; mt++) {
        if (mt >= mn) break;
        part[(warp * MNB + mt) * 32 + lane] = make_double2(acc[mt][0], acc[mt][1]);
      }
      consumer_bar();
      r0 = r1 = 0.0;
      if (epi) {
#pragma unroll
        for (int w = 0; w < NCW; w++) {
          const double2 v = part[(w * MNB + et) * 32 + lane];
          r0 += v.x;
          r1 += v.y;
        }
      }
    };

#ifdef SLB_SOLVE_PROF
    long long P0 = clock64(), ph[16] = {0};
#define PM(k) { const long long q_ = clock64(); ph[k] += q_ - P0; P0 = q_; }
#else
#define PM(k)
#endif
    // ---------------- forward ----------------
    double* tt = xbuf + 2 * WC;
    for (int64_t l = 0; l < n2; l++) {
      const bool hn = l + 1 < n2;
      const uint8_t fl = sfl[l];
      const bool sc = fwd_shortcut(fl, a.fsc);
      const int zo = (int)(l & 1) * WC;
      PM(7)
      if (l > 0) wait_x();  // z_l complete (all rows, pushed by every CTA)
      if (hn) arm();        // exchange of z_{l+1}
      PM(0)
      mbar_wait(&lfull[ls], lph);
      PM(1)
      const unsigned char* lv = smraw + Ly.lv + (int64_t)ls * Ly.lv_slot;
      const int* sperm = reinterpret_cast<const int*>(lv + Ly.o_perm);
      const double* bn = reinterpret_cast<const double*>(lv + Ly.o_b);
      const double* dsl = reinterpret_cast<const double*>(lv + Ly.o_dsub);
      auto vval2 = [&](int src, int n) -> double2 {  // (row src, cols n, n+1) of [z_l ; b_{l+1}]
        if (src < Wp) return *reinterpret_cast<const double2*>(xbuf + zo + src * C + n);
        if (!hn) return make_double2(0.0, 0.0);
        return *reinterpret_cast<const double2*>(bn + (src - Wp) * C + n);
      };
      // t_top = rows perm[0..Wp) of [z_l ; b_{l+1}]
      for (int idx = tid; idx < WC / 2; idx += CTHREADS) {
        const int r = idx / (C / 2), n = (idx % (C / 2)) * 2;
        *reinterpret_cast<double2*>(tt + r * C + n) = vval2(sperm[r], n);
      }
      // t_bot at this thread's epilogue rows
      double2 tb = make_double2(0.0, 0.0);
      if (epi && hn) tb = vval2(sperm[Wp + erow], 2 * t);
      consumer_bar();
      PM(2)
      const int ncx = (sc && hn) ? ((fl >> 2) & 15) : 0;
      if (warp < ncx) {  // exceptional bottom row e = warp: Fbot[e, :] t_top (all C columns)
        const double* er = reinterpret_cast<const double*>(lv + Ly.o_exc) + warp * Wp;
        const int n = lane & 7, kp = lane >> 3;
        double q = 0.0;
        for (int k = kp; k < Wp; k += 4) q = fma(er[k], tt[k * C + n], q);
        q += __shfl_xor_sync(0xffffffffu, q, 8);
        q += __shfl_xor_sync(0xffffffffu, q, 16);
        if (kp == 0) excval[warp][n] = q;
      }
      PM(3)
      double acc[MNMAX][2], acc2[MNMAX][2];
#pragma unroll
      for (int mt = 0; mt < MNMAX; mt++) acc[mt][0] = acc[mt][1] = acc2[mt][0] = acc2[mt][1] = 0.0;
      const int nch = (sc || !hn) ? 2 : 4;  // Ainv halves (+ Fbot halves)
      for (int c = 0; c < nch; c++) {
        if ((c & 1) != wg) {
          skip_op();
          continue;
        }
        const double* Aop = acquire_op();
        PM(4)
        gemv_chunk(Aop, tt, (c & 1) * KH, c < 2 ? acc : acc2);
        release_op();
        PM(5)
      }
      double y0, y1;
      reduce_parts(acc, y0, y1);
      PM(6)
      double z0 = 0.0, z1 = 0.0;
      if (hn) {
        if (sc) {
          const double d = epi ? dsl[erow] : 0.0;
          z0 = fma(-d, y0, tb.x);
          z1 = fma(-d, y1, tb.y);
          if (ncx && epi) {
            const int* epos = reinterpret_cast<const int*>(lv + Ly.o_epos);
            for (int e = 0; e < ncx; e++)
              if (epos[e] == erow) {
                z0 = tb.x + excval[e][2 * t];
                z1 = tb.y + excval[e][2 * t + 1];
              }
          }
        } else {
          consumer_bar();  // part reused for the Fbot partial sums
          double f0, f1;
          reduce_parts(acc2, f0, f1);
          z0 = tb.x + f0;
          z1 = tb.y + f1;
        }
      }
      if (epi) {
        // y_l rows -> HBM (read back by the backward sweep)
        *reinterpret_cast<double2*>(ybase + l * WC + erow * C + 2 * t) = make_double2(y0, y1);
        if (hn) push((int)((l + 1) & 1), erow, z0, z1);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&lempty[ls]);
      if (++ls == LS) {
        ls = 0;
        lph ^= 1u;
      }
      // no barrier here: tt, part and excval are next written after the next level's t_top barrier
    }
    // forward done: y rows visible to the level producer's bulk copies
    fence_proxy_async_global();
    __syncwarp();
    if (lane == 0) mbar_arrive(&fwd_done);

    // ---------------- backward ----------------
    // x_{n2} = x_{n2+1} = 0; no peer may push x_{n2-1} before every CTA cleared its buffers
    for (int idx = tid; idx < 3 * WC; idx += CTHREADS) xbuf[idx] = 0.0;
    asm volatile("barrier.cluster.arrive.release;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire;\n" ::: "memory");
    for (int64_t l = n2 - 1; l >= 0; l--) {
      const uint8_t fl = sfl[l];
      const bool full = bwd_full2(fl, a.bsc);
      const int nhc = ((fl & 1) && !full) ? ((fl >> 2) & 15) : 0;
      const int b0 = (int)(l % 3), b1 = (int)((l + 1) % 3), b2 = (int)((l + 2) % 3);
      PM(13)
      if (l < n2 - 1) wait_x();  // x_{l+1} complete
      arm();                     // exchange of x_l
      PM(8)
      mbar_wait(&lfull[ls], lph);
      PM(9)
      const unsigned char* lv = smraw + Ly.lv + (int64_t)ls * Ly.lv_slot;
      const double* x1 = xbuf + b1 * WC;
      const double* x2 = xbuf + b2 * WC;
      double acc[MNMAX][2];
#pragma unroll
      for (int mt = 0; mt < MNMAX; mt++) acc[mt][0] = acc[mt][1] = 0.0;
      const int nch = full ? 4 : 2;
      for (int c = 0; c < nch; c++) {
        if ((c & 1) != wg) {
          skip_op();
          continue;
        }
        const double* Aop = acquire_op();
        PM(10)
        gemv_chunk(Aop, c < 2 ? x1 : x2, (c & 1) * KH, acc);
        release_op();
        PM(11)
      }
      double h0, h1;
      reduce_parts(acc, h0, h1);
      PM(12)
      if (epi) {
        const double2 yv = reinterpret_cast<const double2*>(lv + Ly.o_y)[(et * 8 + g) * (C / 2) + t];
        double x0v = yv.x - h0, x1v = yv.y - h1;
        if (nhc) {  // x_{l+2} half of H: the columns of the rows pivoted up (schur.cu)
          const int* hidx = reinterpret_cast<const int*>(lv + Ly.o_hidx);
          const double* hcol = reinterpret_cast<const double*>(lv + Ly.o_hcol);
          for (int e = 0; e < nhc; e++) {
            const double hv = hcol[e * Wp + erow];
            const double2 xr = *reinterpret_cast<const double2*>(x2 + hidx[e] * C + 2 * t);
            x0v = fma(-hv, xr.x, x0v);
            x1v = fma(-hv, xr.y, x1v);
          }
        }
        push(b0, erow, x0v, x1v);
        if (a.mode == SWEEP_RECOVER) {
          if (erow < sd.w) {
            double* o = a.out + (int64_t)(sd.col0 + erow) * n2 + l;
            if (2 * t < ncols) o[(int64_t)(q0 + 2 * t) * a.N] = x0v;
            if (2 * t + 1 < ncols) o[(int64_t)(q0 + 2 * t + 1) * a.N] = x1v;
          }
        } else {  // reduce: x_l rows over y_l (consumed); to_X x_l in strip_contrib_kernel
          *reinterpret_cast<double2*>(ybase + l * WC + erow * C + 2 * t) = make_double2(x0v, x1v);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&lempty[ls]);
      if (++ls == LS) {
        ls = 0;
        lph ^= 1u;
      }
    }
    wait_x();  // x_0 complete everywhere before the cluster exits (peers push into us)
#ifdef SLB_SOLVE_PROF
    if (blockIdx.x < G && (tid == 0 || tid == 160))
      printf("SOLVE2 blk %d tid %d G %d mn %d | fwd: xwait %lld lfull %lld tt %lld exc %lld opwait %lld gemv %lld red %lld epi %lld"
             " | bwd: xwait %lld lfull %lld opwait %lld gemv %lld red %lld epi %lld\n",
             blockIdx.x, tid, G, mn, ph[0], ph[1], ph[2], ph[3], ph[4], ph[5], ph[6], ph[7], ph[8], ph[9], ph[10], ph[11],
             ph[12], ph[13]);
#endif
  }
  if (idle) asm volatile("barrier.cluster.wait;\n" ::: "memory");
  // no CTA leaves while a peer may still push into its shared memory
  __syncthreads();
  cluster.sync();
}

// contrib[s][X][col][l] = to_X[l] . x_l[:, col] (reduce mode), x_l in the task's slab [l][Wp][C]
__global__ void __launch_bounds__(256) strip_contrib_kernel(SchurArgs a) {
  const int task = blockIdx.y;
  const int s = a.tasks[3 * task];
  const int q0 = a.tasks[3 * task + 2];
  const StripDesc sd = a.strips[s];
  const int Wp = a.Wp;
  const int64_t n2 = a.n2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t l = (int64_t)blockIdx.x * 8 + warp;
  if (l >= n2) return;
  const int64_t rem = a.nrhs - q0;
  const int ncols = (int)(rem < C ? rem : C);
  const double* x = a.ybuf + (int64_t)task * a.sY + l * Wp * C;
  const double* cpl = a.cpl + s * a.sCPL;
  const int n = lane & 7, kp = lane >> 3;
  for (int X = 0; X < 2; X++) {
    if ((X == 0 ? sd.left : sd.right) < 0) continue;
    const double* tv = cpl + (2 + X) * n2 * Wp + l * Wp;
    double q = 0.0;
    for (int i = kp; i < Wp; i += 4) q = fma(tv[i], x[i * C + n], q);
    q += __shfl_xor_sync(0xffffffffu, q, 8);
    q += __shfl_xor_sync(0xffffffffu, q, 16);
    if (kp == 0 && n < ncols) a.out[((int64_t)(s * 2 + X) * a.nrhs + q0 + n) * n2 + l] = q;
  }
}

}  // namespace

// ---- tensor maps over the factor storage (driver API entry point resolved at run time) ----
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
    cudaGetLastError();
  });
  return fn;
}

// 4-D map {32 doubles, m tiles, k4 rows, level} over per-level operator blocks stored in DMMA fragment
// order [k4][m8][lane]; base = first tile of the block, tile_stride tiles per k4 row, mt tiles mapped.
CUtensorMap make_map(const double* base, int mt, int tile_stride, int k4rows, int64_t levels, int64_t lvl_doubles,
                     int box_mt, int box_k) {
  CUtensorMap m;
  const cuuint64_t dims[4] = {32, (cuuint64_t)mt, (cuuint64_t)k4rows, (cuuint64_t)levels};
  const cuuint64_t strides[3] = {256, (cuuint64_t)tile_stride * 256, (cuuint64_t)lvl_doubles * 8};
  const cuuint32_t box[4] = {32, (cuuint32_t)box_mt, (cuuint32_t)box_k, 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  EncodeFn fn = encode_fn();
  if (!fn) throw CudaFailure(cudaErrorNotSupported, "cuTensorMapEncodeTiled unavailable", __FILE__, __LINE__);
  const CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaFailure(cudaErrorInvalidValue, "cuTensorMapEncodeTiled failed", __FILE__, __LINE__);
  return m;
}


bool strip_solve2_fits(int Wp, int64_t n2, int G, bool dmma_only) {
  const int MTH = Wp / 8;
  if (G < 1 || G > 8 || G > MTH || (MTH + G - 1) / G > MNMAX) return false;
  if (!dmma_only && (MTH + G - 1) / G > NCW_DFMA) return false;  // the DFMA variants' row-tile warps
  return lay2(Wp, G, n2).bytes <= 227 * 1024 - 1024;
}

// Cluster size for ntasks concurrent tasks: the largest G in {8, 6, 5, 4} whose clusters all fit at
// once (cudaOccupancyMaxActiveClusters), else 4.
int strip_solve2_cluster(int Wp, int64_t n2, int ntasks, bool dmma) {
  static std::mutex mu;
  static std::map<std::pair<int, int64_t>, int> cache;  // (Wp, n2 * 1024 + ntasks) -> G
  const char* e = getenv("SLB_SOLVE_G");
  if (e) return std::min(atoi(e), Wp / 8);
  const char* e2 = getenv("SLB_SOLVE_G_WAVES");  // cluster size when the tasks run in waves (A/B)
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_pair(Wp * 2 + (dmma ? 1 : 0), n2 * 1024 + ntasks);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  const int MTH = Wp / 8;
  // no size fits every task at once (many right-hand sides: tasks run in waves): small clusters,
  // more of them resident per wave (cfg4, 64 RHS on the DMMA variant: 1.31 ms per RHS with 2-CTA
  // clusters, 1.42 with 3, 1.56 with 4)
  int best = (dmma && strip_solve2_fits(Wp, n2, 2, true)) ? 2 : strip_solve2_fits(Wp, n2, 3) ? 3 : std::min(4, MTH);
  if (e2) best = std::min(atoi(e2), MTH);
  for (int G : {8, 6, 5, 4}) {
    if (!strip_solve2_fits(Wp, n2, G)) continue;
    const size_t smem = (size_t)lay2(Wp, G, n2).bytes;
    if (cudaFuncSetAttribute(strip_solve2_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(G * ntasks));
    cfg.blockDim = dim3(threads_of<0>());
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, strip_solve2_kernel<0>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (nc >= ntasks) {
      best = G;
      break;
    }
  }
  cache[key] = best;
  return best;
}

void strip_solve2(cudaStream_t st, const SchurArgs& a, int ntasks) {
  const int Wp = a.Wp;
  const bool dmma = a.nrhs > 4 || getenv("SLB_SOLVE_DMMA") != nullptr;
  const int G = strip_solve2_cluster(Wp, a.n2, ntasks, dmma);
  if (!strip_solve2_fits(Wp, a.n2, G, dmma))
    throw CudaFailure(cudaErrorInvalidValue, "strip_solve2: slab too wide for the cluster split", __FILE__, __LINE__);
  strip_rhs_pack(st, a, ntasks);
  const Lay2 Ly = lay2(Wp, G, a.n2);
  const int64_t levels = (int64_t)a.nstrips * a.n2;
  const int64_t lvl = 4LL * Wp * Wp;
  const int MTH = Wp / 8;
  const CUtensorMap mA = make_map(a.fac, MTH, 2 * MTH, Wp / 4, levels, lvl, Ly.MNB, Ly.KH);
  const CUtensorMap mF = make_map(a.fac + MTH * 32, MTH, 2 * MTH, Wp / 4, levels, lvl, Ly.MNB, Ly.KH);
  const CUtensorMap mH = make_map(a.fac + 2LL * Wp * Wp, MTH, MTH, Wp / 2, levels, lvl, Ly.MNB, Ly.KH);
  const size_t smem = (size_t)Ly.bytes;
  // columns per task: 1, 2, 3-4 on DFMA, 5-8 on DMMA (SLB_SOLVE_DMMA=1 forces DMMA)
  static const bool force_dmma = getenv("SLB_SOLVE_DMMA") != nullptr;
  const int64_t cols = a.nrhs < C ? a.nrhs : C;
  void (*kern)(Solve2Args, CUtensorMap, CUtensorMap, CUtensorMap) =
      (force_dmma || cols > 4) ? strip_solve2_kernel<0>
      : cols == 1             ? strip_solve2_kernel<1>
      : cols == 2             ? strip_solve2_kernel<2>
                              : strip_solve2_kernel<4>;
  SLB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  Solve2Args A2{a, G};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(G * ntasks));
  cfg.blockDim = dim3((force_dmma || cols > 4) ? threads_of<0>()
                      : cols == 1             ? threads_of<1>()
                      : cols == 2             ? threads_of<2>()
                                              : threads_of<4>());
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = G;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  SLB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, A2, mA, mF, mH)); count_launch();
  if (a.mode == SWEEP_REDUCE) {
    strip_contrib_kernel<<<dim3((unsigned)cdiv(a.n2, 8), (unsigned)ntasks), 256, 0, st>>>(a); count_launch();
    SLB_CUDA_CHECK(cudaGetLastError());
  }
}

}  // namespace slb
