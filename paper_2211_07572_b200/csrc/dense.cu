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
#include <algorithm>
#include <map>
#include <mutex>
#include <vector>
#include <climits>
#include <cstdlib>
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace slb {
namespace {

constexpr int PNB = 32;          // panel width
constexpr int PTHREADS = 256;    // threads per CTA of the panel cluster (<= 16 CTAs, 1 or 2 rows each: n <= 8192)

// Factor rows [j, n) x cols [j, j + nb) of A in place.  Thread (rank, tid)
// owns panel row i = rank * PTHREADS + tid in registers.  Per column one
// cluster barrier (relaxed arrive after a CTA fence: the exchange is shared-memory only): every CTA publishes its best candidate (value, row index,
// row data) and, if it owns it, row k, into parity-double-buffered shared
// memory; after the barrier every CTA reads the candidates through DSMEM and
// applies the same swap and rank-1 update.  ipiv[j + k] = global pivot row.
template <bool RELAXED>
__device__ __forceinline__ void panel_cluster_barrier() {
  if (RELAXED) {
    // shared-memory exchange only: perform this CTA's shared stores, then a relaxed arrive
    __threadfence_block();
    asm volatile("barrier.cluster.arrive.relaxed;\n" ::: "memory");
  } else {
    asm volatile("barrier.cluster.arrive.release;\n" ::: "memory");
  }
  asm volatile("barrier.cluster.wait.acquire;\n" ::: "memory");
}

// r[k] for a runtime k without local memory or branches: a select tree on the bits of k
// (depth log2 N instead of a chain of N dependent selects)
template <int N>
__device__ __forceinline__ double pick(const double (&r)[N], int k) {
  static_assert(N == 32, "pick: 32-wide rows");
  double t16[16], t8[8], t4[4], t2[2];
#pragma unroll
  for (int c = 0; c < 16; c++) t16[c] = (k & 16) ? r[c + 16] : r[c];
#pragma unroll
  for (int c = 0; c < 8; c++) t8[c] = (k & 8) ? t16[c + 8] : t16[c];
#pragma unroll
  for (int c = 0; c < 4; c++) t4[c] = (k & 4) ? t8[c + 4] : t8[c];
#pragma unroll
  for (int c = 0; c < 2; c++) t2[c] = (k & 2) ? t4[c + 2] : t4[c];
  return (k & 1) ? t2[1] : t2[0];
}

__device__ __forceinline__ void better(double& v, int& vi, double ov, int oi) {
  if (ov > v || (ov == v && oi < vi)) {
    v = ov;
    vi = oi;
  }
}

// Warp-wide first maximum of (v, vi) with three hardware reductions on the bit pattern of v
// (non-negative doubles order like their bit patterns): the maximum v, ties to the smallest vi.
// Candidates with v < 0 or NaN never win (key 0; a 0.0 maximum is the singular case anyway).
// Returns the lanes holding the winner.
__device__ __forceinline__ unsigned warp_argmax(double& v, int& vi) {
  const unsigned long long key = (v >= 0.0) ? (unsigned long long)__double_as_longlong(v) : 0ull;
  const unsigned khi = (unsigned)(key >> 32), klo = (unsigned)key;
  const unsigned mhi = __reduce_max_sync(0xffffffffu, khi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, khi == mhi ? klo : 0u);
  const bool ismax = khi == mhi && klo == mlo;
  const int mi = (int)__reduce_min_sync(0xffffffffu, ismax ? (unsigned)vi : 0x7fffffffu);
  const unsigned who = __ballot_sync(0xffffffffu, ismax && vi == mi);
  vi = mi;
  v = __longlong_as_double((long long)(((unsigned long long)mhi << 32) | mlo));
  return who;
}

template <bool RELAXED>
__global__ void __launch_bounds__(PTHREADS) panel_getrf_kernel(double* A, int64_t lda, int64_t n, int64_t j, int nb,
                                                               int32_t* ipiv, DevStatus* status, int block_index) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int ncta = (int)cluster.num_blocks();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = PTHREADS / 32;
  const int64_t m = n - j;
  const int64_t i = (int64_t)rank * PTHREADS + tid;
  const bool own = i < m;
  __shared__ double s_wv[NW];
  __shared__ int s_wi[NW];
  __shared__ double s_cv[2];
  __shared__ int s_ci[2];
  __shared__ double s_crow[2][PNB];  // this CTA's candidate row
  __shared__ double s_krow[2][PNB];  // row k (owner CTA only)
  // pushed by every CTA of the cluster before the barrier (so the resolve reads only local memory)
  __shared__ double s_allv[2][16];
  __shared__ int s_alli[2][16];
  __shared__ double s_allrow[2][16][PNB];  // candidate rows of all CTAs
  __shared__ double s_allk[2][PNB];        // row k

  double r[PNB];
#pragma unroll
  for (int c = 0; c < PNB; c++) r[c] = (own && c < nb) ? A[(j + c) * lda + j + i] : 0.0;

#ifdef SLB_PANEL_PROF
  long long P0 = clock64(), ph[5] = {0, 0, 0, 0, 0};
#define PP(k_) { const long long q_ = clock64(); ph[k_] += q_ - P0; P0 = q_; }
#else
#define PP(k_)
#endif
  for (int k = 0; k < nb; k++) {
    const int pb = k & 1;
    // (1) CTA argmax over rows i >= k (first max by row index); every warp reduces the
    //     per-warp winners redundantly, so one CTA barrier suffices
    double v = -1.0;
    int vi = INT_MAX;
    if (own && i >= k) {
      v = fabs(pick(r, k));
      vi = (int)i;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) better(v, vi, __shfl_xor_sync(0xffffffffu, v, o), __shfl_xor_sync(0xffffffffu, vi, o));
    if (lane == 0) {
      s_wv[warp] = v;
      s_wi[warp] = vi;
    }
    __syncthreads();
    v = lane < NW ? s_wv[lane] : -1.0;
    vi = lane < NW ? s_wi[lane] : INT_MAX;
#pragma unroll
    for (int o = NW / 2; o > 0; o >>= 1) better(v, vi, __shfl_xor_sync(0xffffffffu, v, o), __shfl_xor_sync(0xffffffffu, vi, o));
    v = __shfl_sync(0xffffffffu, v, 0);
    vi = __shfl_sync(0xffffffffu, vi, 0);
    PP(0)
    // (2) publish the CTA candidate and row k
    if (tid == 0) {
      s_cv[pb] = v;
      s_ci[pb] = vi;
    }
    if (own && i == vi)
#pragma unroll
      for (int c = 0; c < PNB; c++) s_crow[pb][c] = r[c];
    if (own && i == k)
#pragma unroll
      for (int c = 0; c < PNB; c++) s_krow[pb][c] = r[c];
    __syncthreads();
    // push candidate (value, row index, row) and row k into every CTA of the cluster
    if (warp == 0) {
      const double cr = s_crow[pb][lane];  // PNB == 32 == warp size
      for (int r2 = 0; r2 < ncta; r2++) dsmem_st_f64(dsmem_map(&s_allrow[pb][rank][lane], r2), cr);
      if (lane < ncta) {
        dsmem_st_f64(dsmem_map(&s_allv[pb][rank], lane), s_cv[pb]);
        dsmem_st_s32(dsmem_map(&s_alli[pb][rank], lane), s_ci[pb]);
      }
    } else if (warp == 1 && k / PTHREADS == rank) {
      const double kr = s_krow[pb][lane];
      for (int r2 = 0; r2 < ncta; r2++) dsmem_st_f64(dsmem_map(&s_allk[pb][lane], r2), kr);
    }
    panel_cluster_barrier<false>();  // release / acquire: the pushed data is visible after it
    PP(1)
    // (3) every warp resolves the same pivot from local copies
    double bv = -1.0;
    int bi = INT_MAX, bc = 0;
    if (lane < ncta) {
      bv = s_allv[pb][lane];
      bi = s_alli[pb][lane];
      bc = lane;
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {  // ncta <= 16
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
        bc = oc;
      }
    }
    bv = __shfl_sync(0xffffffffu, bv, 0);
    bi = __shfl_sync(0xffffffffu, bi, 0);
    bc = __shfl_sync(0xffffffffu, bc, 0);
    if (!(bv > 0.0)) {  // exactly singular column: no interchange
      bi = k;
      bc = k / PTHREADS;
      if (tid == 0 && rank == 0) {
        atomicOr(&status->flags, ERR_SINGULAR);
        atomicMin(&status->singular_block, block_index);
      }
    }
    if (tid == 0 && rank == 0) ipiv[j + k] = (int32_t)(j + bi);
    PP(2)
    const int p = bi;
    const double* prow = (bi == k) ? s_allk[pb] : s_allrow[pb][bc];
    if (p != k) {
      const double* src_row = (own && i == k) ? prow : s_allk[pb];
      if (own && (i == k || i == p)) {
#pragma unroll
        for (int c = 0; c < PNB; c++) r[c] = src_row[c];
      }
    }
    // (4) scale + rank-1 update of rows below k, branch-free over the register row
    if (own && i > k) {
      const double pv = prow[k];
      const double inv = pv != 0.0 ? 1.0 / pv : 0.0;
      const double l = pick(r, k) * inv;
#pragma unroll
      for (int c = 0; c < PNB; c++) {
        const double nv = fma(-l, prow[c], r[c]);
        r[c] = c > k ? nv : (c == k ? l : r[c]);
      }
    }
    PP(3)
  }
#ifdef SLB_PANEL_PROF
  if (tid == 0 && (rank == 0 || rank == ncta - 1) && j == 0)
    printf("PANEL rank %d m=%lld: argmax %lld publish+barrier %lld resolve %lld update %lld (cycles)\n", rank,
           (long long)m, ph[0], ph[1], ph[2], ph[3]);
#endif
  cluster.sync();
  if (own)
#pragma unroll
    for (int c = 0; c < PNB; c++)
      if (c < nb) A[(j + c) * lda + j + i] = r[c];
}

// Panel of nb <= PNB columns with the register row SHIFTED one column per step: at step k
// a thread's r[c] holds column k + c of its row, so the pivot column is always r[0] and every
// register index is static inside a rolled loop (no select trees, small code).  L entries are
// stored as they are computed (coalesced across threads); a row retires as U when it becomes
// row k.  The per-column exchange is data driven: every CTA pushes its candidate (|a|, row
// index, row) and CTA 0 row k into every CTA of the cluster (itself included) with st.async,
// counted on the receiver's mbarrier; two barriers and buffers alternate by column parity.  A
// CTA pushes column k+1 only after its own column-k resolve and update (the CTA barrier of k+1
// orders them), and a peer can push column k+2 into buffer k&1 only after it received column
// k+1 from this CTA, so no cluster barrier per column is needed.  The panel's interchanges are
// replayed at the end into a swap list (row pos[s] <- original row org[s]) for
// panel_swaps_list_kernel.
constexpr int PNW = PTHREADS / 32;
// RPT rows per thread (RPT = 2: panels of up to 8192 rows on the 16-CTA cluster): thread tid of
// CTA rank owns rows rank * RPT * PTHREADS + tid + q * PTHREADS, q < RPT.
template <int RPT>
__global__ void __launch_bounds__(PTHREADS) panel32_kernel(double* A, int64_t lda, int64_t n, int64_t j, int nb,
                                                           int32_t* ipiv, DevStatus* status, int block_index,
                                                           int32_t* swl) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int ncta = (int)cluster.num_blocks();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t m = n - j;
  int64_t iq[RPT];
  bool ownq[RPT];
#pragma unroll
  for (int q = 0; q < RPT; q++) {
    iq[q] = (int64_t)rank * RPT * PTHREADS + tid + q * PTHREADS;
    ownq[q] = iq[q] < m;
  }
  __shared__ __align__(16) double s_row[2][16][PNB];  // candidate rows of all CTAs (pushed)
  __shared__ __align__(16) double s_rec[2][16][2];    // {|a|, row index} of all CTAs (pushed)
  __shared__ __align__(16) double s_krow[2][PNB];     // row k (pushed by CTA 0)
  __shared__ __align__(16) double s_wrow[2][PNW][PNB];  // per-warp candidate rows (local staging)
  __shared__ __align__(16) double s_kst[2][PNB];        // row k (local staging, CTA 0)
  __shared__ double s_wv[2][PNW];
  __shared__ int s_wi[2][PNW];
  __shared__ __align__(8) uint64_t s_bar[2];
  __shared__ int s_piv[PNB];
  __shared__ int s_pos[2 * PNB], s_org[2 * PNB];
  __shared__ double s_urow[PNB][PNB + 1];  // retired U rows (CTA 0), shifted: [k][c] = U(k, k + c)

  double rr[RPT][PNB];
#pragma unroll
  for (int q = 0; q < RPT; q++)
#pragma unroll
    for (int c = 0; c < PNB; c++) rr[q][c] = (ownq[q] && c < nb) ? A[(j + c) * lda + j + iq[q]] : 0.0;
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    fence_mbar_init();
  }
  cluster.sync();  // every CTA's barriers initialised before any push targets them
  // warp w pushes to CTAs w and w + PNW
  uint32_t rrow[2], rrec[2], rkrow[2], rbar[2];
#pragma unroll
  for (int q = 0; q < 2; q++) {
    const int d = warp + q * PNW < ncta ? warp + q * PNW : 0;
    rrow[q] = dsmem_map(&s_row[0][rank][0], d);
    rrec[q] = dsmem_map(&s_rec[0][rank][0], d);
    rkrow[q] = dsmem_map(&s_krow[0][0], d);
    rbar[q] = dsmem_map(&s_bar[0], d);
  }
  const uint32_t xbytes = (uint32_t)(ncta * (PNB * 8 + 16) + PNB * 8);
#ifdef SLB_PANEL_PROF
  long long P0 = clock64(), ph[5] = {0, 0, 0, 0, 0};
#endif

#pragma unroll 1
  for (int k = 0; k < nb; k++) {
    const int pb = k & 1;
    bool liveq[RPT];  // rows above k have retired
#pragma unroll
    for (int q = 0; q < RPT; q++) liveq[q] = ownq[q] && iq[q] >= k;
    if (tid == 0) mbar_arrive_expect_tx(&s_bar[pb], xbytes);
    // (1) warp argmax (first max by row index); the warp winner stages its row
    double v = -1.0;
    int vi = INT_MAX;
#pragma unroll
    for (int q = 0; q < RPT; q++)
      if (liveq[q]) better(v, vi, fabs(rr[q][0]), (int)iq[q]);
    warp_argmax(v, vi);
#pragma unroll
    for (int q = 0; q < RPT; q++) {
      if (liveq[q] && iq[q] == vi)
#pragma unroll
        for (int c = 0; c < PNB; c++) s_wrow[pb][warp][c] = rr[q][c];
      if (liveq[q] && iq[q] == k)
#pragma unroll
        for (int c = 0; c < PNB; c++) s_kst[pb][c] = rr[q][c];
    }
    if (lane == 0) {
      s_wv[pb][warp] = v;
      s_wi[pb][warp] = vi;
    }
    __syncthreads();
    PP(0)
    // (2) CTA winner (every warp, redundantly), then push to this warp's two destinations
    v = lane < PNW ? s_wv[pb][lane] : -1.0;
    vi = lane < PNW ? s_wi[pb][lane] : INT_MAX;
    const unsigned wwho = warp_argmax(v, vi) & ((1u << PNW) - 1);
    const int wb = wwho ? __ffs(wwho) - 1 : 0;  // the winning warp (its row is staged)
    {
      const uint32_t boff = (uint32_t)(pb * 8);
      const uint32_t roff = (uint32_t)(pb * 16 * PNB * 8);
      const uint32_t coff = (uint32_t)(pb * 16 * 2 * 8);
      const uint32_t koff = (uint32_t)(pb * PNB * 8);
      const bool lo = lane < 16;
      const int e = 2 * (lane & 15);
      const double a0 = lo ? s_wrow[pb][wb][e] : s_kst[pb][e];
      const double a1 = lo ? s_wrow[pb][wb][e + 1] : s_kst[pb][e + 1];
      const uint32_t dst = (lo ? roff : koff) + (uint32_t)(lane & 15) * 16;
      const bool go = lo || rank == 0;
#pragma unroll
      for (int q = 0; q < 2; q++)
        if (warp + q * PNW < ncta) {
          if (go) st_async_v2((lo ? rrow[q] : rkrow[q]) + dst, a0, a1, rbar[q] + boff);
          if (lane == 0) st_async_v2(rrec[q] + coff, v, (double)vi, rbar[q] + boff);
        }
    }
    PP(1)
    // (3) wait for every CTA's candidate and row k
    mbar_wait(&s_bar[pb], (uint32_t)((k >> 1) & 1));
    PP(2)
    // (4) resolve the pivot from the local copies
    double bv = -1.0;
    int bi = INT_MAX;
    if (lane < ncta) {
      bv = s_rec[pb][lane][0];
      bi = (int)s_rec[pb][lane][1];
    }
    const unsigned cwho = warp_argmax(bv, bi) & (ncta >= 32 ? 0xffffffffu : ((1u << ncta) - 1));
    int bc = cwho ? __ffs(cwho) - 1 : 0;  // the CTA holding the pivot row
    if (!(bv > 0.0)) {  // exactly singular column: no interchange
      bi = k;
      bc = 0;
      if (tid == 0 && rank == 0) {
        atomicOr(&status->flags, ERR_SINGULAR);
        atomicMin(&status->singular_block, block_index);
      }
    }
    const double* prow = (bi == k) ? s_krow[pb] : s_row[pb][bc];
    // bookkeeping on CTA 0's last warp (warp 0 holds the panel's own rows and is the busiest):
    // the pivot index, and row k retiring as the U row = the pivot row (shifted: r[c] = column
    // k + c), one element per lane
    if (rank == 0 && warp == PNW - 1) {
      if (lane == 0) {
        ipiv[j + k] = (int32_t)(j + bi);
        s_piv[k] = bi;
      }
      s_urow[k][lane] = prow[lane];  // PNB == 32
    }
    const double pv = prow[0];
    const double pinv = pv != 0.0 ? __drcp_rn(pv) : 0.0;  // == 1.0 / pv (both correctly rounded)
#pragma unroll
    for (int q = 0; q < RPT; q++) {
      if (!liveq[q]) continue;
      if (iq[q] == k) {  // row k retires (copied to s_urow above)
      } else {
        if (iq[q] == bi && bi != k)
#pragma unroll
          for (int c = 0; c < PNB; c++) rr[q][c] = s_krow[pb][c];
        // (5) scale, store L, rank-1 update shifted down one column
        const double l = rr[q][0] * pinv;
        A[(j + k) * lda + j + iq[q]] = l;
#pragma unroll
        for (int c = 1; c < PNB; c++) rr[q][c - 1] = fma(-l, prow[c], rr[q][c]);
        rr[q][PNB - 1] = 0.0;
      }
    }
    PP(3)
  }
#ifdef SLB_PANEL_PROF
  if (tid == 0 && (rank == 0 || rank == ncta - 1) && j == 0)
    printf("PANEL32 rank %d/%d m=%lld: argmax+stage %lld push %lld wait %lld resolve+update %lld (cycles)\n", rank, ncta,
           (long long)m, ph[0], ph[1], ph[2], ph[3]);
#endif
  if (rank == 0) {  // U rows, coalesced: thread (c, k) for the upper triangle
    __syncthreads();
    for (int e = tid; e < PNB * PNB; e += PTHREADS) {
      const int c = e / PNB, k = e % PNB;  // column c, row k <= c
      if (c < nb && k <= c) A[(j + c) * lda + j + k] = s_urow[k][c - k];
    }
  }
  // swap list: replay the interchanges over the affected rows (slots 0..31 = panel rows,
  // 32.. = rows below the panel that took part)
  if (rank == 0 && warp == 0) {
    __syncwarp();
    s_pos[lane] = lane;
    s_org[lane] = lane;
    int ns = 0;
    for (int q = 0; q < nb; q++) {
      const int p = s_piv[q];
      int slot = p;
      if (p >= nb) {
        const unsigned hit = __ballot_sync(0xffffffffu, lane < ns && s_pos[PNB + lane] == p);
        if (hit) {
          slot = PNB + __ffs(hit) - 1;
        } else {
          slot = PNB + ns;
          if (lane == 0) {
            s_pos[slot] = p;
            s_org[slot] = p;
          }
          ns++;
        }
      }
      __syncwarp();
      if (lane == 0 && slot != q) {
        const int t = s_org[q];
        s_org[q] = s_org[slot];
        s_org[slot] = t;
      }
      __syncwarp();
    }
    const int cnt = PNB + ns;
    if (lane == 0) swl[0] = cnt;
    for (int s2 = lane; s2 < cnt; s2 += 32) {
      swl[1 + s2] = (int32_t)(j + s_pos[s2]);
      swl[1 + 2 * PNB + s2] = (int32_t)(j + s_org[s2]);
    }
  }
  cluster.sync();  // no CTA leaves while a peer may still push into it
}

// The panel's interchanges applied to every column outside it from the swap list: one warp
// per column, every affected row loaded first, then stored (no dependent swap chain).
constexpr int SWL = 1 + 4 * PNB;  // swap-list ints per panel
// Interchanges ipiv[j + q0 + 1 .. j + nb) applied to one column (rows relative to j): one warp
// replays them over the affected rows (ballot search of the side list), then moves the values.
__device__ void panel_column_swaps(double* col, int64_t j, int nb, int q0, const int32_t* ipiv, int lane) {
  int pos0 = lane, org0 = lane;  // slot `lane`: panel row `lane`
  int pos1 = -1, org1 = -1;      // side slot `lane`: a row below the panel
  int ns = 0;
  for (int q = q0 + 1; q < nb; q++) {
    const int p = (int)(ipiv[j + q] - j);
    if (p == q) continue;
    // slot of row p: panel row p, or the side slot holding it (appended if new)
    int side = -1;
    if (p >= nb) {
      const unsigned hit = __ballot_sync(0xffffffffu, lane < ns && pos1 == p);
      if (hit) {
        side = __ffs(hit) - 1;
      } else {
        side = ns;
        if (lane == ns) {
          pos1 = p;
          org1 = p;
        }
        ns++;
      }
    }
    // swap the contents (org) of slot q and the slot of p
    const int oq = __shfl_sync(0xffffffffu, org0, q);
    const int op = side < 0 ? __shfl_sync(0xffffffffu, org0, p) : __shfl_sync(0xffffffffu, org1, side);
    if (lane == q) org0 = op;
    if (side < 0 && lane == p) org0 = oq;
    if (side >= 0 && lane == side) org1 = oq;
  }
  const bool a0 = lane < nb && pos0 != org0;
  const bool a1 = lane < ns && pos1 != org1;
  const double v0 = a0 ? col[j + org0] : 0.0;
  const double v1 = a1 ? col[j + org1] : 0.0;
  __syncwarp();
  if (a0) col[j + pos0] = v0;
  if (a1) col[j + pos1] = v1;
}

__global__ void __launch_bounds__(256) panel_swaps_list_kernel(double* A, int64_t lda, int64_t n, int64_t j, int nb,
                                                              const int32_t* swl, const int32_t* ipiv, int64_t cmax) {
  __shared__ int s_cnt;
  __shared__ int s_pos[2 * PNB], s_org[2 * PNB];
  if (threadIdx.x == 0) s_cnt = swl[0];
  if (threadIdx.x < 2 * PNB) {
    s_pos[threadIdx.x] = swl[1 + threadIdx.x];
    s_org[threadIdx.x] = swl[1 + 2 * PNB + threadIdx.x];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (c >= n) return;
  if (c >= n - nb) {  // the panel's own column q: its L entries take the interchanges of steps > q
    const int q0 = (int)(c - (n - nb));
    panel_column_swaps(A + (j + q0) * lda, j, nb, q0, ipiv, lane);
    return;
  }
  if (c >= j) c += nb;
  if (c >= cmax) return;  // columns at or beyond cmax take these interchanges later (laswp)
  double* col = A + c * lda;
  const int cnt = s_cnt;
  const bool a0 = lane < cnt && s_pos[lane] != s_org[lane];
  const bool a1 = lane + 32 < cnt && s_pos[lane + 32] != s_org[lane + 32];
  const double v0 = a0 ? col[s_org[lane]] : 0.0;
  const double v1 = a1 ? col[s_org[lane + 32]] : 0.0;
  __syncwarp();
  if (a0) col[s_pos[lane]] = v0;
  if (a1) col[s_pos[lane + 32]] = v1;
}

// The same interchanges restricted to column ranges (the look-ahead LU splits them between its
// two streams): warps [0, own) fix the panel's own L columns, the next ones take the columns
// [a0, a1) and then [b0, b1).
__global__ void __launch_bounds__(256) panel_swaps_range_kernel(double* A, int64_t lda, int64_t j, int nb,
                                                               const int32_t* swl, const int32_t* ipiv, int own,
                                                               int64_t a0, int64_t a1, int64_t b0, int64_t b1) {
  __shared__ int s_cnt;
  __shared__ int s_pos[2 * PNB], s_org[2 * PNB];
  if (threadIdx.x == 0) s_cnt = swl[0];
  if (threadIdx.x < 2 * PNB) {
    s_pos[threadIdx.x] = swl[1 + threadIdx.x];
    s_org[threadIdx.x] = swl[1 + 2 * PNB + threadIdx.x];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (w < own) {
    panel_column_swaps(A + (j + w) * lda, j, nb, (int)w, ipiv, lane);
    return;
  }
  w -= own;
  int64_t c;
  if (w < a1 - a0) {
    c = a0 + w;
  } else {
    w -= a1 - a0;
    if (w >= b1 - b0) return;
    c = b0 + w;
  }
  double* col = A + c * lda;
  const int cnt = s_cnt;
  const bool f0 = lane < cnt && s_pos[lane] != s_org[lane];
  const bool f1 = lane + 32 < cnt && s_pos[lane + 32] != s_org[lane + 32];
  const double v0 = f0 ? col[s_org[lane]] : 0.0;
  const double v1 = f1 ? col[s_org[lane + 32]] : 0.0;
  __syncwarp();
  if (f0) col[s_pos[lane]] = v0;
  if (f1) col[s_pos[lane + 32]] = v1;
}

// The interchanges of nl consecutive panels (their swap lists, in order) on the columns
// [a0, a1) and [b0, b1): one warp per column replays the lists one after the other.
constexpr int MAXL = 8;  // panels per look-ahead block (<= 256 columns)
__global__ void __launch_bounds__(256) swaps_multi_kernel(double* A, int64_t lda, const int32_t* lists, int nl,
                                                         int64_t a0, int64_t a1, int64_t b0, int64_t b1) {
  __shared__ int s_cnt[MAXL];
  __shared__ int s_pos[MAXL][2 * PNB], s_org[MAXL][2 * PNB];
  for (int i = threadIdx.x; i < nl * 2 * PNB; i += blockDim.x) {
    const int l = i / (2 * PNB), e = i % (2 * PNB);
    const int32_t* sl = lists + l * SWL;
    s_pos[l][e] = sl[1 + e];
    s_org[l][e] = sl[1 + 2 * PNB + e];
    if (e == 0) s_cnt[l] = sl[0];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  int64_t c;
  if (w < a1 - a0) {
    c = a0 + w;
  } else {
    w -= a1 - a0;
    if (w >= b1 - b0) return;
    c = b0 + w;
  }
  double* col = A + c * lda;
  for (int l = 0; l < nl; l++) {
    const int cnt = s_cnt[l];
    const bool f0 = lane < cnt && s_pos[l][lane] != s_org[l][lane];
    const bool f1 = lane + 32 < cnt && s_pos[l][lane + 32] != s_org[l][lane + 32];
    const double v0 = f0 ? col[s_org[l][lane]] : 0.0;
    const double v1 = f1 ? col[s_org[l][lane + 32]] : 0.0;
    __syncwarp();
    if (f0) col[s_pos[l][lane]] = v0;
    if (f1) col[s_pos[l][lane + 32]] = v1;
    __syncwarp();
  }
}

void swaps_multi(cudaStream_t st, double* A, int64_t lda, const int32_t* lists, int nl, int64_t a0, int64_t a1,
                 int64_t b0, int64_t b1) {
  const int64_t tot = std::max<int64_t>(0, a1 - a0) + std::max<int64_t>(0, b1 - b0);
  if (tot <= 0 || nl <= 0) return;
  swaps_multi_kernel<<<(unsigned)cdiv(tot, (int64_t)8), 256, 0, st>>>(A, lda, lists, nl, a0, std::max(a0, a1), b0,
                                                                     std::max(b0, b1));
  count_launch();
  SLB_CUDA_CHECK(cudaGetLastError());
}

// Row interchanges ipiv[k1..k2) (LAPACK order) as one permutation of rows
// [k1, n): idx[r - k1] = source row of row r.  One CTA, swaps replayed in
// shared memory by one thread (n - k1 <= 8192).
__global__ void swap_perm_kernel(const int32_t* ipiv, int64_t n, int64_t k1, int64_t k2, int32_t* idx) {
  // rows and pivots as int16 in shared memory (n - k1 <= 8192): the serial replay touches
  // shared memory only
  extern __shared__ int16_t sidx[];
  int16_t* spiv = sidx + (n - k1);
  const int64_t m = n - k1;
  for (int64_t r = threadIdx.x; r < m; r += blockDim.x) sidx[r] = (int16_t)r;
  for (int64_t k = k1 + threadIdx.x; k < k2; k += blockDim.x) spiv[k - k1] = (int16_t)(ipiv[k] - k1);
  __syncthreads();
  if (threadIdx.x == 0)
    for (int64_t k = 0; k < k2 - k1; k++) {
      const int p = spiv[k];
      const int16_t t = sidx[k];
      sidx[k] = sidx[p];
      sidx[p] = t;
    }
  __syncthreads();
  for (int64_t r = threadIdx.x; r < m; r += blockDim.x) idx[r] = (int32_t)(k1 + sidx[r]);
}
// tmp[c][r] = A[c][idx[r]] for rows [k1, n) of columns [c0, c1)
__global__ void gather_rows_kernel(const double* A, int64_t lda, int64_t c0, int64_t c1, int64_t k1, int64_t m,
                                   const int32_t* idx, double* tmp) {
  const int64_t c = c0 + blockIdx.y;
  const double* col = A + c * lda;
  double* t = tmp + (int64_t)blockIdx.y * m;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x)
    t[r] = col[idx[r]];
}
__global__ void scatter_rows_kernel(double* A, int64_t lda, int64_t c0, int64_t k1, int64_t m, const double* tmp) {
  const int64_t c = c0 + blockIdx.y;
  double* col = A + c * lda + k1;
  const double* t = tmp + (int64_t)blockIdx.y * m;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x)
    col[r] = t[r];
}

// The panel's interchanges ipiv[j, j+nb) applied, in order, to every column outside the panel
// (LAPACK dlaswp on both sides at once): one thread per column, rows swapped in registers-free
// place.  Applying them when the panel finishes is equivalent to the recursion's deferred laswp
// calls (row interchanges commute with the updates of columns not yet touched).
__global__ void panel_swaps_kernel(double* A, int64_t lda, int64_t n, int64_t j, int nb, const int32_t* ipiv,
                                   int64_t cmax) {
  __shared__ int32_t sp[PNB];
  if (threadIdx.x < nb) sp[threadIdx.x] = ipiv[j + threadIdx.x];
  __syncthreads();
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= j) c += nb;  // skip the panel's own columns
  if (c >= n || c >= cmax) return;
  double* col = A + c * lda;
  for (int q = 0; q < nb; q++) {
    const int64_t r = j + q, p = sp[q];
    if (p != r) {
      const double t = col[r];
      col[r] = col[p];
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
  static const bool relaxed = [] {
    const char* e = getenv("SLB_PANEL_BARRIER");
    return !(e && e[0] == 'r' && e[1] == 'e' && e[2] == 'l' && e[3] == 'e');  // "release": full-scope barrier
  }();
  auto kern = relaxed ? panel_getrf_kernel<true> : panel_getrf_kernel<false>;
  static bool attr[2] = {false, false};
  if (!attr[relaxed]) {
    SLB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr[relaxed] = true;
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
  SLB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, A, lda, n, j, nb, ipiv, status, block_index)); count_launch();
}

bool panel_v1() {
  static const bool v1 = [] {
    const char* e = getenv("SLB_PANEL_V1");
    return e && e[0] == '1';
  }();
  return v1;
}

void panel32(cudaStream_t st, double* A, int64_t lda, int64_t n, int64_t j, int nb, int32_t* ipiv,
             DevStatus* status, int block_index, int32_t* swl) {
  const int64_t m = n - j;
  const int rpt = m > 16 * PTHREADS ? 2 : 1;
  const int ncta = (int)cdiv(m, (int64_t)PTHREADS * rpt);
  if (ncta > 16)
    throw CudaFailure(cudaErrorInvalidValue, "dgetrf: block dimension > 8192 unsupported", __FILE__, __LINE__);
  static bool attr = false;
  if (!attr) {
    SLB_CUDA_CHECK(cudaFuncSetAttribute(panel32_kernel<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    SLB_CUDA_CHECK(cudaFuncSetAttribute(panel32_kernel<2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
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
  SLB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, rpt == 2 ? panel32_kernel<2> : panel32_kernel<1>, A, lda, n, j, nb, ipiv,
                                    status, block_index, swl));
  count_launch();
}

// laswp scratch comes from the device's stream-ordered pool (cudaMallocAsync): stage two runs
// laswp on two streams at once, and a pool kept warm (release threshold) makes it cheap.
void* pool_alloc(size_t bytes, cudaStream_t st) {
  static bool init[64] = {};
  int dev = 0;
  SLB_CUDA_CHECK(cudaGetDevice(&dev));
  if (dev < 64 && !init[dev]) {
    cudaMemPool_t pool;
    SLB_CUDA_CHECK(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t thr = 1ull << 30;  // keep up to 1 GiB of freed blocks for reuse
    SLB_CUDA_CHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    init[dev] = true;
  }
  void* p = nullptr;
  SLB_CUDA_CHECK(cudaMallocAsync(&p, bytes, st));
  return p;
}

// Apply ipiv[k1..k2) to columns [c0, c1) of the n-row matrix A: replay the
// interchanges once as a row permutation, then a coalesced permuted copy.
void laswp(cudaStream_t st, double* A, int64_t lda, int64_t c0, int64_t c1, const int32_t* ipiv, int64_t k1,
           int64_t k2, int64_t n) {
  if (c1 <= c0 || k2 <= k1) return;
  const int64_t m = n - k1, nc = c1 - c0;
  int32_t* idx = static_cast<int32_t*>(pool_alloc(m * sizeof(int32_t), st));
  double* tmp = static_cast<double*>(pool_alloc(m * nc * sizeof(double), st));
  swap_perm_kernel<<<1, 1024, (m + (k2 - k1)) * sizeof(int16_t), st>>>(ipiv, n, k1, k2, idx); count_launch();
  SLB_CUDA_CHECK(cudaGetLastError());
  for (int64_t cb = 0; cb < nc; cb += 65535) {
    const int64_t ncb = std::min<int64_t>(65535, nc - cb);
    dim3 grid((unsigned)std::min<int64_t>(cdiv(m, 256), 16), (unsigned)ncb);
    gather_rows_kernel<<<grid, 256, 0, st>>>(A, lda, c0 + cb, c0 + cb + ncb, k1, m, idx, tmp + cb * m); count_launch();
    scatter_rows_kernel<<<grid, 256, 0, st>>>(A, lda, c0 + cb, k1, m, tmp + cb * m); count_launch();
  }
  SLB_CUDA_CHECK(cudaGetLastError());
  SLB_CUDA_CHECK(cudaFreeAsync(idx, st));
  SLB_CUDA_CHECK(cudaFreeAsync(tmp, st));
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
// cmax: columns >= cmax are not touched (their interchanges are applied later by laswp).
void getrf_rec(cudaStream_t st, double* A, int64_t n, int64_t c0, int64_t c1, int32_t* ipiv,
               DevStatus* status, int block_index, int32_t* swl, int64_t cmax) {
  const int64_t w = c1 - c0;
  if (w <= PNB) {
    if (swl && !panel_v1()) {
      panel32(st, A, n, n, c0, (int)w, ipiv, status, block_index, swl);
      // interchanges on every other column now (so the recursion needs no laswp) and the later
      // steps' interchanges on the panel's own L columns
      panel_swaps_list_kernel<<<(unsigned)cdiv(n, 8), 256, 0, st>>>(A, n, n, c0, (int)w, swl, ipiv, cmax);
      count_launch();
      SLB_CUDA_CHECK(cudaGetLastError());
      return;
    }
    panel(st, A, n, n, c0, (int)w, ipiv, status, block_index);
    if (n - w > 0) {  // interchanges on every other column now, so the recursion needs no laswp
      panel_swaps_kernel<<<(unsigned)cdiv(n - w, 128), 128, 0, st>>>(A, n, n, c0, (int)w, ipiv, cmax); count_launch();
      SLB_CUDA_CHECK(cudaGetLastError());
    }
    return;
  }
  int64_t h = round_up(w / 2, PNB);
  if (h >= w) h = w - PNB;
  getrf_rec(st, A, n, c0, c0 + h, ipiv, status, block_index, swl, cmax);
  trsm(st, true, A + c0 * n + c0, n, h, A + (c0 + h) * n + c0, n, w - h);
  dgemm_batched(st, n - c0 - h, w - h, h, -1.0, A + c0 * n + c0 + h, n, 0, A + (c0 + h) * n + c0, n, 0, 1.0,
                A + (c0 + h) * n + c0 + h, n, 0, 1);
  getrf_rec(st, A, n, c0 + h, c1, ipiv, status, block_index, swl, cmax);
}

// Streams of the look-ahead LU (per host thread and device): the panel chain on a
// greatest-priority stream, the trailing updates on a least-priority one.
struct LaStreams {
  cudaStream_t hi = nullptr, lo = nullptr;
  cudaEvent_t ev[4] = {};
};
LaStreams& la_streams() {
  thread_local std::map<int, LaStreams> per_dev;
  int dev = 0;
  SLB_CUDA_CHECK(cudaGetDevice(&dev));
  LaStreams& s = per_dev[dev];
  if (!s.hi) {
    int least = 0, greatest = 0;
    SLB_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    SLB_CUDA_CHECK(cudaStreamCreateWithPriority(&s.hi, cudaStreamNonBlocking, greatest));
    SLB_CUDA_CHECK(cudaStreamCreateWithPriority(&s.lo, cudaStreamNonBlocking, least));
    for (auto& e : s.ev) SLB_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  return s;
}

bool getrf_rec_only() {
  static const bool v = [] {
    const char* e = getenv("SLB_GETRF_REC");
    return e && e[0] == '1';
  }();
  return v;
}

// Recursive LU of the block [c0, c1) inside the look-ahead LU: like getrf_rec, but the
// interchanges touch only the block's own columns (the caller applies them elsewhere from the
// swap lists, kept one per 32-column panel at lists + ((j - cb) / 32) * SWL).
void getrf_blk(cudaStream_t st, double* A, int64_t n, int64_t c0, int64_t c1, int64_t cb, int64_t ce,
               int32_t* ipiv, DevStatus* status, int block_index, int32_t* lists) {
  const int64_t w = c1 - c0;
  if (w <= PNB) {
    int32_t* sw = lists + ((c0 - cb) / PNB) * SWL;
    panel32(st, A, n, n, c0, (int)w, ipiv, status, block_index, sw);
    const int64_t tot = w + (c0 - cb) + (ce - c1);
    panel_swaps_range_kernel<<<(unsigned)cdiv(tot, (int64_t)8), 256, 0, st>>>(A, n, c0, (int)w, sw, ipiv, (int)w, cb,
                                                                             c0, c1, ce);
    count_launch();
    SLB_CUDA_CHECK(cudaGetLastError());
    return;
  }
  int64_t h = round_up(w / 2, PNB);
  if (h >= w) h = w - PNB;
  getrf_blk(st, A, n, c0, c0 + h, cb, ce, ipiv, status, block_index, lists);
  trsm(st, true, A + c0 * n + c0, n, h, A + (c0 + h) * n + c0, n, w - h);
  dgemm_batched(st, n - c0 - h, w - h, h, -1.0, A + c0 * n + c0 + h, n, 0, A + (c0 + h) * n + c0, n, 0, 1.0,
                A + (c0 + h) * n + c0 + h, n, 0, 1);
  getrf_blk(st, A, n, c0 + h, c1, cb, ce, ipiv, status, block_index, lists);
}

// LU of columns [c0, c1) (rows c0..n) of the n x n matrix A with look-ahead: blocks of NBW
// columns, each factored recursively (getrf_blk) on a greatest-priority stream; then the same
// stream applies the block's interchanges, TRSM and update to the NEXT block only, so that
// block's factorization starts at once, while a least-priority stream applies the interchanges
// to the columns left of the block and right of the next one and the rank-NBW update to the
// trailing columns [p + 2 NBW, c1) (cmax as in getrf_rec).  The trailing GEMM of one block
// (K = NBW) hides behind the next block's latency-bound panels.
//   panel stream:    LU block k | wait T(k-1) | swaps+TRSM+GEMM on block k+1
//   trailing stream: wait | swaps on [0, p) and [p + 2 NBW, cmax) | TRSM+GEMM on [p + 2 NBW, c1)
// T(k-1) is waited for before block k+1 is touched: it wrote those columns.  The swap lists
// alternate between two sets (T(k) reads set k while block k + 1 writes the other).
void getrf_la(cudaStream_t st, double* A, int64_t n, int64_t c0, int64_t c1, int32_t* ipiv, DevStatus* status,
              int block_index, int64_t cmax) {
  if (c1 <= c0) return;
  static const int64_t NBW = [] {
    const char* e = getenv("SLB_GETRF_NBW");
    const int v = e ? atoi(e) : 64;  // cfg3 stage two: 64 0.677 s, 128 0.685, 256 0.695 (recursive 0.720)
    return (int64_t)std::min(std::max(PNB, v / PNB * PNB), MAXL * PNB);
  }();
  LaStreams& S = la_streams();
  cudaStream_t sa = S.hi, sb = S.lo;
  cudaEvent_t evP = S.ev[0], evB[2] = {S.ev[1], S.ev[2]}, evJ = S.ev[3];
  SLB_CUDA_CHECK(cudaEventRecord(evJ, st));
  SLB_CUDA_CHECK(cudaStreamWaitEvent(sa, evJ, 0));
  SLB_CUDA_CHECK(cudaStreamWaitEvent(sb, evJ, 0));
  const int64_t lset = (NBW / PNB) * SWL;
  int32_t* swl = nullptr;
  SLB_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&swl), 2 * lset * sizeof(int32_t), sa));
  const int64_t nbk = cdiv(c1 - c0, NBW);
  // SLB_GETRF_TRACE=1 (measurement): timed events per block, printed for a few blocks
  static const bool trace = getenv("SLB_GETRF_TRACE") != nullptr;
  std::vector<cudaEvent_t> tev;
  auto mark = [&](cudaStream_t s) {
    if (!trace) return;
    cudaEvent_t e;
    SLB_CUDA_CHECK(cudaEventCreate(&e));
    SLB_CUDA_CHECK(cudaEventRecord(e, s));
    tev.push_back(e);
  };
  mark(sa);
  for (int64_t k = 0; k < nbk; k++) {
    const int64_t p = c0 + k * NBW;
    const int64_t w = std::min(NBW, c1 - p);
    const int nl = (int)cdiv(w, (int64_t)PNB);
    const int64_t q = p + w;                                      // next block [q, q + wn)
    const int64_t wn = std::max<int64_t>(0, std::min(NBW, c1 - q));
    const int64_t r = q + wn;                                     // trailing columns [r, c1)
    int32_t* ls = swl + (k & 1) * lset;
    getrf_blk(sa, A, n, p, q, p, q, ipiv, status, block_index, ls);
    mark(sa);
    if (k > 0) SLB_CUDA_CHECK(cudaStreamWaitEvent(sa, evB[(k - 1) & 1], 0));
    mark(sa);
    SLB_CUDA_CHECK(cudaEventRecord(evP, sa));
    SLB_CUDA_CHECK(cudaStreamWaitEvent(sb, evP, 0));
    if (wn > 0) {
      swaps_multi(sa, A, n, ls, nl, q, q + wn, 0, 0);
      trsm(sa, true, A + p * n + p, n, w, A + q * n + p, n, wn);
      dgemm_batched(sa, n - q, wn, w, -1.0, A + p * n + q, n, 0, A + q * n + p, n, 0, 1.0, A + q * n + q, n, 0, 1);
    }
    mark(sa);
    swaps_multi(sb, A, n, ls, nl, 0, p, std::min(r, cmax), cmax);
    if (r < c1) {
      trsm(sb, true, A + p * n + p, n, w, A + r * n + p, n, c1 - r);
      dgemm_batched(sb, n - q, c1 - r, w, -1.0, A + p * n + q, n, 0, A + r * n + p, n, 0, 1.0, A + r * n + q, n, 0, 1);
    }
    mark(sb);
    SLB_CUDA_CHECK(cudaEventRecord(evB[k & 1], sb));
  }
  SLB_CUDA_CHECK(cudaStreamWaitEvent(sa, evB[(nbk - 1) & 1], 0));
  SLB_CUDA_CHECK(cudaFreeAsync(swl, sa));
  SLB_CUDA_CHECK(cudaEventRecord(evJ, sa));
  SLB_CUDA_CHECK(cudaStreamWaitEvent(st, evJ, 0));
  if (trace) {
    // per block: LU end, T(k-1) wait end, next-block update end (sa), T(k) end (sb); us from the block start
    SLB_CUDA_CHECK(cudaStreamSynchronize(st));
    double sum[3] = {0, 0, 0};
    for (int64_t k = 0; k < nbk; k++) {
      float t[4];
      cudaEvent_t e0 = tev[k == 0 ? 0 : 4 * k - 1];
      for (int i = 0; i < 4; i++) SLB_CUDA_CHECK(cudaEventElapsedTime(&t[i], e0, tev[4 * k + 1 + i]));
      sum[0] += t[0];
      sum[1] += t[1] - t[0];
      sum[2] += t[2] - t[1];
      if (k % 8 == 0 || k == nbk - 1)
        fprintf(stderr, "[getrf_la] block %lld: LU %.1f us, wait %.1f us, next-block update %.1f us; trailing done at %.1f us\n",
                (long long)k, 1e3 * t[0], 1e3 * (t[1] - t[0]), 1e3 * (t[2] - t[1]), 1e3 * t[3]);
    }
    fprintf(stderr, "[getrf_la] n=%lld cols [%lld,%lld) NBW %lld: block LU %.2f ms, wait %.2f ms, next-block %.2f ms\n",
            (long long)n, (long long)c0, (long long)c1, (long long)NBW, sum[0], sum[1], sum[2]);
    for (auto e : tev) cudaEventDestroy(e);
  }
}

}  // namespace

void dgetrf(cudaStream_t st, int64_t n, double* a, int32_t* ipiv, double* /*work*/, DevStatus* status,
            int block_index) {
  if (!panel_v1() && !getrf_rec_only()) {
    getrf_la(st, a, n, 0, n, ipiv, status, block_index, n);
    return;
  }
  int32_t* swl = nullptr;  // swap list of the current panel (stream ordered, reused by every panel)
  SLB_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&swl), SWL * sizeof(int32_t), st));
  getrf_rec(st, a, n, 0, n, ipiv, status, block_index, swl, n);
  SLB_CUDA_CHECK(cudaFreeAsync(swl, st));
}

// The same LU with columns [h, n) not ready yet: columns [0, h) are factored first (their
// interchanges kept off the right part), then the stream waits for right_ready, applies the
// left part's interchanges to columns [h, n) (LAPACK's deferred laswp), and finishes with the
// triangular solve, the trailing update and the LU of the right part.
void dgetrf_split(cudaStream_t st, int64_t n, double* a, int32_t* ipiv, DevStatus* status, int block_index,
                  int64_t h, cudaEvent_t right_ready) {
  h = std::min<int64_t>(round_up(std::max<int64_t>(h, PNB), PNB), n);
  if (!panel_v1() && !getrf_rec_only()) {
    getrf_la(st, a, n, 0, h, ipiv, status, block_index, h);
    SLB_CUDA_CHECK(cudaStreamWaitEvent(st, right_ready, 0));
    if (h < n) {
      laswp(st, a, n, h, n, ipiv, 0, h, n);
      trsm(st, true, a, n, h, a + h * n, n, n - h);
      dgemm_batched(st, n - h, n - h, h, -1.0, a + h, n, 0, a + h * n, n, 0, 1.0, a + h * n + h, n, 0, 1);
      getrf_la(st, a, n, h, n, ipiv, status, block_index, n);
    }
    return;
  }
  int32_t* swl = nullptr;
  SLB_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&swl), SWL * sizeof(int32_t), st));
  getrf_rec(st, a, n, 0, h, ipiv, status, block_index, swl, h);
  SLB_CUDA_CHECK(cudaStreamWaitEvent(st, right_ready, 0));
  if (h < n) {
    laswp(st, a, n, h, n, ipiv, 0, h, n);
    trsm(st, true, a, n, h, a + h * n, n, n - h);
    dgemm_batched(st, n - h, n - h, h, -1.0, a + h, n, 0, a + h * n, n, 0, 1.0, a + h * n + h, n, 0, 1);
    getrf_rec(st, a, n, h, n, ipiv, status, block_index, swl, n);
  }
  SLB_CUDA_CHECK(cudaFreeAsync(swl, st));
}

void dgetrs(cudaStream_t st, int64_t n, int64_t nrhs, const double* lu, const int32_t* ipiv, double* b,
            int64_t ldb, double* /*work*/) {
  laswp(st, b, ldb, 0, nrhs, ipiv, 0, n, n);
  trsm(st, true, lu, n, n, b, ldb, nrhs);
  trsm(st, false, lu, n, n, b, ldb, nrhs);
}

void dset_identity(cudaStream_t st, double* a, int64_t n) {
  identity_kernel<<<(unsigned)std::min<int64_t>(cdiv(n * n, 256), 8192), 256, 0, st>>>(a, n); count_launch();
  SLB_CUDA_CHECK(cudaGetLastError());
}

void check_finite(cudaStream_t st, const double* a, int64_t count, DevStatus* status) {
  if (count <= 0) return;
  finite_kernel<<<(unsigned)std::min<int64_t>(cdiv(count, 256), 4096), 256, 0, st>>>(a, count, status); count_launch();
  SLB_CUDA_CHECK(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// y = beta*y + alpha*A*x for small nrhs (deterministic split-K).
namespace {
constexpr int GV_ROWS = 64;   // rows per CTA (lane -> 2 rows)
constexpr int GV_SPLIT = 8;   // K splits
__global__ void __launch_bounds__(256) gemv_partial_kernel(int64_t m, int64_t n, int64_t nrhs, const double* A,
                                                           int64_t lda, const double* x, int64_t ldx, double* part) {
  // CTA: 64 rows (lane -> 2 consecutive rows as one 16-byte load), 8 warps split the K range,
  // each warp keeps 4 columns in flight.
  const int64_t r0 = (int64_t)blockIdx.x * GV_ROWS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t kc = cdiv(n, GV_SPLIT);
  const int64_t k0 = blockIdx.y * kc, k1 = min(n, k0 + kc);
  __shared__ double red[8][GV_ROWS];
  const int64_t ra = r0 + 2 * lane;
  const bool full = ra + 1 < m && ((lda & 1) == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
  for (int64_t c = 0; c < nrhs; c++) {
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
    const double* xc = x + c * ldx;
    int64_t k = k0 + warp;
    for (; k + 24 < k1; k += 32) {  // 4 columns per iteration (stride 8 warps)
      double2 v[4];
      double xv[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const double* col = A + (k + 8 * u) * lda;
        xv[u] = xc[k + 8 * u];
        if (full) v[u] = *reinterpret_cast<const double2*>(col + ra);
        else v[u] = make_double2(ra < m ? col[ra] : 0.0, ra + 1 < m ? col[ra + 1] : 0.0);
      }
#pragma unroll
      for (int u = 0; u < 4; u += 2) {
        a0 = fma(v[u].x, xv[u], a0);
        a1 = fma(v[u].y, xv[u], a1);
        b0 = fma(v[u + 1].x, xv[u + 1], b0);
        b1 = fma(v[u + 1].y, xv[u + 1], b1);
      }
    }
    for (; k < k1; k += 8) {
      const double* col = A + k * lda;
      const double xv = xc[k];
      if (ra < m) a0 = fma(col[ra], xv, a0);
      if (ra + 1 < m) a1 = fma(col[ra + 1], xv, a1);
    }
    red[warp][2 * lane] = a0 + b0;
    red[warp][2 * lane + 1] = a1 + b1;
    __syncthreads();
    if (threadIdx.x < GV_ROWS) {
      double s = 0.0;
      for (int w = 0; w < 8; w++) s += red[w][threadIdx.x];
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
  gemv_partial_kernel<<<grid, 256, 0, st>>>(m, n, nrhs, A, lda, x, ldx, part); count_launch();
  SLB_CUDA_CHECK(cudaGetLastError());
  gemv_reduce_kernel<<<(unsigned)cdiv(m * nrhs, 256), 256, 0, st>>>(m, nrhs, alpha, part, beta, y, ldy); count_launch();
  SLB_CUDA_CHECK(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// dgetrs for the stage-two sweep solve (stage_two.hpp:176-186: S_j^{-1} r is
// applied from the LU factors of S_j, as DenseLU::solve does, dense.hpp:48-61).
// One launch runs both triangular solves as a chain of 64-row blocks per
// 8-column group of right-hand sides: CTA i of the first half solves block i
// of L y = P b, CTA i of the second half block i of U z = y (bottom block
// first).  Each CTA streams its off-diagonal row of 64x64 tiles two at a time
// as the blocks they multiply are published, so the critical path per block
// is one L2 hop plus two 64x64 GEMVs: the diagonal blocks are applied through
// their inverses (computed once at factorization by getrs_prepare from the LU
// factors, as MAGMA's trsv does).  There are no flags: a published block is
// its data, and a consumer polls the values themselves against a sentinel NaN
// pattern that no computation can produce (NaN results are canonicalised).
// The y/z scratch holds two sets used on alternating calls; each CTA resets
// its own block of the other set to the sentinel, ready for the next call.
// Polls only ever wait on lower CTA indices of the same chain.  That is
// deadlock-free when every CTA of a launch is resident at once, which the
// launcher guarantees by sizing each launch to the occupancy limit (CTAs are
// not guaranteed to be dispatched in blockIdx order, so a launch larger than
// the resident capacity could park waiting CTAs ahead of the ones they wait
// on).  Polls are bounded: an expired spin raises ERR_CHAIN_TIMEOUT in the
// status word, which the solve reports as an error instead of returning data.
namespace {
constexpr int CT = 64;
constexpr unsigned long long kSentinel = 0xFFFFFFFFFFFFFFFFull;
constexpr unsigned long long kCanonNaN = 0x7FF8000000000000ull;
constexpr int kSpinLimit = 1 << 22;
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const double* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_f64(double* p, double v) {
  unsigned long long u = (unsigned long long)__double_as_longlong(v);
  if ((u & 0x7FF0000000000000ull) == 0x7FF0000000000000ull && (u & 0x000FFFFFFFFFFFFFull)) u = kCanonNaN;
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(u) : "memory");
}

// perm[r] = source row of row r after the interchanges ipiv[0..n); one CTA per call.
// dinv: per 64-row block b, [inv(L_bb) | inv(U_bb)] (64x64 col-major each, padded with identity).
__global__ void __launch_bounds__(64) diag_inverse_kernel(int n, const double* __restrict__ lu, double* dinv) {
  __shared__ double T[CT][CT + 1];
  const int blk = blockIdx.x, upper = blockIdx.y, c = threadIdx.x;
  const int r0 = blk * CT, m = min(CT, n - r0);
  for (int k = 0; k < CT; k++)
    T[c][k] = (c < m && k < m) ? lu[(int64_t)(r0 + k) * n + r0 + c] : (c == k ? 1.0 : 0.0);
  __syncthreads();
  double X[CT];  // thread c solves for column c of the inverse (fully unrolled: registers)
#pragma unroll
  for (int r = 0; r < CT; r++) X[r] = (r == c) ? 1.0 : 0.0;
  if (!upper) {
#pragma unroll
    for (int k = 0; k < CT; k++) {
#pragma unroll
      for (int r = k + 1; r < CT; r++) X[r] -= T[r][k] * X[k];
    }
  } else {
#pragma unroll
    for (int k = CT - 1; k >= 0; k--) {
      X[k] = X[k] / T[k][k];
#pragma unroll
      for (int r = 0; r < k; r++) X[r] -= T[r][k] * X[k];
    }
  }
  double* out = dinv + ((int64_t)blk * 2 + upper) * CT * CT;
#pragma unroll
  for (int r = 0; r < CT; r++) out[(int64_t)c * CT + r] = X[r];
}

// MINB = 2 (two CTAs per SM, registers capped at 128, a few spills) only for blocks beyond
// 4096 rows, whose chains (2 * n / 64 CTAs) need more than one resident CTA per SM.
template <int NR, int MINB>
__global__ void __launch_bounds__(256, MINB) getrs_chain_kernel(int n, int nb, const double* __restrict__ lu,
                                                          const double* __restrict__ dinv,
                                                          const int32_t* __restrict__ perm, const double* b,
                                                          int64_t ldb, double* x, int64_t ldx, double alpha,
                                                          double beta, double* cur, double* nxt,
                                                          DevStatus* status) {
  {  // chain = 8-column group: its own columns and scratch (y at +0, z at +8n)
    const int chain = (int)blockIdx.x / (2 * nb);
    b += (int64_t)chain * NR * ldb;
    x += (int64_t)chain * NR * ldx;
    cur += (int64_t)chain * 16 * n;
    nxt += (int64_t)chain * 16 * n;
  }
  const int cta = (int)blockIdx.x % (2 * nb);
  // row / k index innermost: lanes touch consecutive words (no bank conflicts)
  __shared__ double red[4][NR][CT];
  __shared__ double vt[2][NR][CT];
  __shared__ double vs[NR][CT];
  const int t = threadIdx.x, r = t & (CT - 1), kq = t >> 6;
  const bool lower = cta < nb;
  const int i = lower ? cta : nb - 1 - (cta - nb);
  const int r0 = i * CT, mrow = min(CT, n - r0);
  double* y = cur;
  double* z = cur + (int64_t)8 * n;
  const double* src = lower ? y : z;  // published blocks this CTA multiplies
  double* own = lower ? y : z;
  const bool row_owner = t < CT && r < mrow;
  if (row_owner) {  // the next call's copy of this block starts unpublished
    double* o = lower ? nxt : nxt + (int64_t)8 * n;
#pragma unroll
    for (int c = 0; c < NR; c++) o[(int64_t)c * n + r0 + r] = __longlong_as_double((long long)kSentinel);
  }
  double d[16];  // the diagonal block's inverse, prefetched
  {
    const double* D = dinv + ((int64_t)i * 2 + (lower ? 0 : 1)) * CT * CT;
#pragma unroll
    for (int u = 0; u < 16; u++) d[u] = D[(int64_t)(kq * 16 + u) * CT + r];
  }
  double rhs[NR];
  if (lower && row_owner) {
    const int32_t pr = perm[r0 + r];
#pragma unroll
    for (int c = 0; c < NR; c++) rhs[c] = b[(int64_t)c * ldb + pr];
  }
  double acc[NR];
#pragma unroll
  for (int c = 0; c < NR; c++) acc[c] = 0.0;
  const int ntiles = lower ? i : nb - 1 - i;
  constexpr int PER = (2 * CT * NR + 255) / 256;  // staged values per thread (two tiles)
  for (int q = 0; q < ntiles; q += 2) {
    const int j0 = lower ? q : nb - 1 - q, j1 = lower ? q + 1 : nb - 2 - q;
    const int c00 = j0 * CT, nc0 = min(CT, n - c00);
    const int c01 = j1 * CT, nc1 = q + 1 < ntiles ? min(CT, n - c01) : 0;
    double a0[16], a1[16];
#pragma unroll
    for (int u = 0; u < 16; u++) {
      const int k = kq * 16 + u;
      a0[u] = (r < mrow && k < nc0) ? __ldg(&lu[(int64_t)(c00 + k) * n + r0 + r]) : 0.0;
      a1[u] = (r < mrow && k < nc1) ? __ldg(&lu[(int64_t)(c01 + k) * n + r0 + r]) : 0.0;
    }
    unsigned long long v[PER];
    const double* vp[PER];
#pragma unroll
    for (int m = 0; m < PER; m++) {
      const int e = t + 256 * m, tile = e / (CT * NR), rem = e % (CT * NR), c = rem / CT, k = rem % CT;
      const bool valid = e < 2 * CT * NR && k < (tile ? nc1 : nc0);
      vp[m] = valid ? src + (int64_t)c * n + (tile ? c01 : c00) + k : nullptr;
      v[m] = valid ? ld_relaxed_u64(vp[m]) : 0ull;
    }
    for (int spin = 0;; spin++) {  // re-poll the values not yet published
      bool miss = false;
#pragma unroll
      for (int m = 0; m < PER; m++)
        if (v[m] == kSentinel) {
          v[m] = ld_relaxed_u64(vp[m]);
          miss = true;
        }
      if (!miss) break;
      if (spin == kSpinLimit) {
        if (status) atomicOr(&status->flags, ERR_CHAIN_TIMEOUT);
        break;
      }
    }
    __syncthreads();  // the previous pair's FMAs are done with vt
#pragma unroll
    for (int m = 0; m < PER; m++) {
      const int e = t + 256 * m, tile = e / (CT * NR), rem = e % (CT * NR), c = rem / CT, k = rem % CT;
      if (e < 2 * CT * NR) vt[tile][c][k] = __longlong_as_double((long long)v[m]);
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 16; u++) {
      const int k = kq * 16 + u;
#pragma unroll
      for (int c = 0; c < NR; c++) acc[c] = fma(a1[u], vt[1][c][k], fma(a0[u], vt[0][c][k], acc[c]));
    }
  }
  if (!lower && row_owner) {  // upper: this block's right-hand side is y_i from lower CTA i
#pragma unroll
    for (int c = 0; c < NR; c++) {
      unsigned long long u = ld_relaxed_u64(&y[(int64_t)c * n + r0 + r]);
      for (int spin = 0; u == kSentinel; spin++) {
        if (spin == kSpinLimit) {
          if (status) atomicOr(&status->flags, ERR_CHAIN_TIMEOUT);
          break;
        }
        u = ld_relaxed_u64(&y[(int64_t)c * n + r0 + r]);
      }
      rhs[c] = __longlong_as_double((long long)u);
    }
  }
#pragma unroll
  for (int c = 0; c < NR; c++) red[kq][c][r] = acc[c];
  __syncthreads();
  if (t < CT) {
#pragma unroll
    for (int c = 0; c < NR; c++)
      vs[c][r] = r < mrow ? rhs[c] - (red[0][c][r] + red[1][c][r] + red[2][c][r] + red[3][c][r]) : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < NR; c++) {  // out = Dinv_i * (rhs - off-diagonal sum)
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < 16; u++) s = fma(d[u], vs[c][kq * 16 + u], s);
    red[kq][c][r] = s;
  }
  __syncthreads();
  if (row_owner) {
#pragma unroll
    for (int c = 0; c < NR; c++) {
      const double o = red[0][c][r] + red[1][c][r] + red[2][c][r] + red[3][c][r];
      st_relaxed_f64(&own[(int64_t)c * n + r0 + r], o);  // publishes the value
      if (!lower) {
        double* xo = x + (int64_t)c * ldx + r0 + r;
        *xo = beta == 0.0 ? alpha * o : fma(alpha, o, beta * *xo);
      }
    }
  }
}
}  // namespace

void getrs_prepare(cudaStream_t st, int64_t n, const double* lu, const int32_t* ipiv, int32_t* perm,
                   double* dinv) {
  if (n <= 0) return;
  if (n > 8192) throw CudaFailure(cudaErrorInvalidValue, "getrs_prepare: n must be <= 8192", __FILE__, __LINE__);
  swap_perm_kernel<<<1, 1024, 2 * n * sizeof(int16_t), st>>>(ipiv, n, 0, n, perm); count_launch();
  SLB_CUDA_CHECK(cudaGetLastError());
  diag_inverse_kernel<<<dim3((unsigned)cdiv(n, CT), 2), CT, 0, st>>>((int)n, lu, dinv); count_launch();
  SLB_CUDA_CHECK(cudaGetLastError());
}

void getrs_chain(cudaStream_t st, int64_t n, int64_t nrhs, const double* lu, const double* dinv,
                 const int32_t* perm, const double* b, int64_t ldb, double* x, int64_t ldx, double alpha,
                 double beta, double* yz, int epoch, DevStatus* status) {
  if (n <= 0 || nrhs <= 0) return;
  const int nb = (int)cdiv(n, CT);
  // chains of 8 columns, the remainder (< 8 columns) as one more chain; each launch holds at
  // most as many chains as can be resident at once (a chain's CTAs wait on each other)
  const int64_t full = nrhs / 8, rem = nrhs % 8;
  const int64_t set = 16 * n * cdiv(nrhs, 8);
  double* cur = yz + (epoch & 1) * set;
  double* nxt = yz + ((epoch + 1) & 1) * set;
  static int resident1 = 0, resident2 = 0;  // CTAs of getrs_chain_kernel<8, MINB> resident at once
  if (resident1 == 0) {
    int dev = 0, sms = 0, per = 0;
    SLB_CUDA_CHECK(cudaGetDevice(&dev));
    SLB_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    SLB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, getrs_chain_kernel<8, 1>, 256, 0));
    resident1 = std::max(1, sms * per);
    SLB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, getrs_chain_kernel<8, 2>, 256, 0));
    resident2 = std::max(1, sms * per);
  }
  const bool two = 2 * nb > resident1;
  const int resident = two ? resident2 : resident1;
  if (2 * nb > resident)
    throw CudaFailure(cudaErrorInvalidValue, "getrs_chain: block too large for one resident chain", __FILE__, __LINE__);
  const int64_t per_launch = std::max<int64_t>(1, resident / (2 * nb));
#define SLB_CHAIN(NR, NCH, OFF)                                                                          \
  (two ? getrs_chain_kernel<NR, 2> : getrs_chain_kernel<NR, 1>)<<<(unsigned)(2 * nb * (NCH)), 256, 0, st>>>( \
      (int)n, nb, lu, dinv, perm, b + (OFF) * 8 * ldb, ldb, x + (OFF) * 8 * ldx, ldx, alpha, beta,       \
      cur + (OFF) * 16 * n, nxt + (OFF) * 16 * n, status);                                               \
  count_launch()
  for (int64_t c0 = 0; c0 < full; c0 += per_launch) SLB_CHAIN(8, std::min(per_launch, full - c0), c0);
  switch (rem) {
    case 0: break;
    case 1: SLB_CHAIN(1, 1, full); break;
    case 2: SLB_CHAIN(2, 1, full); break;
    case 3: SLB_CHAIN(3, 1, full); break;
    case 4: SLB_CHAIN(4, 1, full); break;
    case 5: SLB_CHAIN(5, 1, full); break;
    case 6: SLB_CHAIN(6, 1, full); break;
    case 7: SLB_CHAIN(7, 1, full); break;
  }
#undef SLB_CHAIN
  SLB_CUDA_CHECK(cudaGetLastError());
}

void getrs_chain_init(cudaStream_t st, int64_t n, int64_t nrhs, double* yz) {
  SLB_CUDA_CHECK(cudaMemsetAsync(yz, 0xFF, getrs_chain_scratch(n, nrhs) * sizeof(double), st));
}

}  // namespace slb
