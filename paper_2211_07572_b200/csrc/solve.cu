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

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace slb {
namespace {

constexpr int G = 4;          // CTAs per cluster
constexpr int C = 8;          // RHS columns per task
constexpr int THREADS = 256;  // 8 warps
constexpr int STAGES = 24;

struct SolveSmem {
  // sizes in doubles, computed at runtime from Wp
  int zb, tb, xb, stage_slot, total;
};

__device__ __forceinline__ int mtiles_of(int total, int r) {  // m tiles owned by CTA r (contiguous)
  const int base = total / G, rem = total % G;
  return base + (r < rem ? 1 : 0);
}
__device__ __forceinline__ int mtile0_of(int total, int r) {
  const int base = total / G, rem = total % G;
  return r * base + min(r, rem);
}

__global__ void __launch_bounds__(THREADS, 1) strip_solve_kernel(SchurArgs a) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  extern __shared__ double sm[];
  const int Wp = a.Wp;
  const int64_t n2 = a.n2;
  const int MTH = Wp / 8;                    // m tiles per Wp rows
  const int MTF = 2 * MTH;                   // forward m tiles (rows of [Ainv ; Fbot])
  const int fm0 = mtile0_of(MTF, rank), fmn = mtiles_of(MTF, rank);
  const int bm0 = mtile0_of(MTH, rank), bmn = mtiles_of(MTH, rank);
  const int slot_d = 2 * ((MTF + G - 1) / G) * 32;  // doubles per staged k8 slice (max over CTAs)
  // shared layout
  double* z = sm;                          // [2][Wp * C]  z_l (full, parity buffers)
  double* tt = z + 2 * Wp * C;             // [Wp * C]     t_top
  double* xb = tt + Wp * C;                // [3][Wp * C]  x_{l}, x_{l+1}, x_{l+2} rotating (backward)
  double* stg = xb + 3 * Wp * C;           // [STAGES][slot_d]
  int* sperm = reinterpret_cast<int*>(stg + STAGES * slot_d);  // [2 Wp]
  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;

  const int task = blockIdx.x / G;
  const int s = a.tasks[3 * task];
  const int q0 = a.tasks[3 * task + 2];
  const StripDesc sd = a.strips[s];
  const double* fac = a.fac + s * a.sF;
  const int32_t* permg = a.perm + s * a.sP;
  const uint8_t* u13 = a.u13 + s * n2;
  const double* cpl = a.cpl + s * a.sCPL;
  const double* toL = cpl + 2 * n2 * Wp;
  const double* toR = cpl + 3 * n2 * Wp;
  const int64_t lvl = 4LL * Wp * Wp;
  const int kf = Wp / 8, kb = Wp / 4;
  const int64_t rem = a.nrhs - q0;
  const int ncols = (int)(rem < C ? rem : C);
  double* ybase = a.ybuf + (int64_t)task * a.sY;  // y slab of this task: n2 x (Wp x C), tile-ordered rows

  if (tid == 0) {
    for (int i = 0; i < STAGES; i++) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], THREADS / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();

  auto rhs_val = [&](int64_t L, int i, int n) -> double {
    if (i >= sd.w || n >= ncols) return 0.0;
    const int64_t col = q0 + n;
    double v = a.f[col * a.N + (int64_t)(sd.col0 + i) * n2 + L];
    if (a.mode == SWEEP_RECOVER) {
      if (sd.left >= 0) v -= cpl[L * Wp + i] * a.u_ifc[col * a.K + (int64_t)sd.left * n2 + L];
      if (sd.right >= 0) v -= cpl[n2 * Wp + L * Wp + i] * a.u_ifc[col * a.K + (int64_t)sd.right * n2 + L];
    }
    return v;
  };

  // ---- operand stream: this CTA's m-tile slice of every k4 step ----
  int prod_slot = 0, cons_slot = 0;  // ring positions (no 64-bit div/mod in the loop)
  int64_t p_lvl = 0;
  int p_j = 0;
  bool p_fwd = true, p_done = false;
  auto issue = [&]() {
    if (p_done) {
      cp_async_commit();
      return;
    }
    const double* base;
    int mt0, mtn, mtot;
    if (p_fwd) {
      base = fac + p_lvl * lvl;
      mt0 = fm0; mtn = fmn; mtot = MTF;
    } else {
      base = fac + p_lvl * lvl + 2LL * Wp * Wp;
      mt0 = bm0; mtn = bmn; mtot = MTH;
    }
    const int sl = prod_slot;
    const int half = mtn * 32;  // doubles per k4 sub-slice
#pragma unroll
    for (int kk = 0; kk < 2; kk++) {
      const double* src = base + (int64_t)(2 * p_j + kk) * mtot * 32 + mt0 * 32;
      double* dst = stg + sl * slot_d + kk * half;
      for (int c = tid; c < half / 2; c += THREADS) cp_async16(dst + 2 * c, src + 2 * c, true);
    }
    cp_async_commit();
    if (++prod_slot == STAGES) prod_slot = 0;
    if (p_fwd) {
      if (++p_j == kf) {
        p_j = 0;
        if (++p_lvl == n2) {
          p_fwd = false;
          p_lvl = n2 - 1;
        }
      }
    } else {
      const int kbl = u13[p_lvl] ? kb : kb / 2;
      if (++p_j == kbl) {
        p_j = 0;
        if (--p_lvl < 0) p_done = true;
      }
    }
  };
  // consumer: slice g_cons is complete once at most STAGES-2 newer groups are pending
  auto acquire = [&]() -> const double* {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    return stg + cons_slot * slot_d;
  };
  auto release = [&]() {
    if (++cons_slot == STAGES) cons_slot = 0;
  };
  for (int i = 0; i < STAGES - 1; i++) issue();

  // ---------------- forward ----------------
  // z_0 = b_0 (full copy in every CTA)
  for (int idx = tid; idx < Wp * C; idx += THREADS) {
    const int r = idx / C, n = idx % C;
    z[idx] = rhs_val(0, r, n);
  }
  int zp = 0;
  long long P0 = clock64(), pa = 0, pb = 0, pc = 0, pd = 0, pq;
  for (int64_t l = 0; l < n2; l++) {
    const bool has_next = l + 1 < n2;
    const double* zc = z + zp * Wp * C;
    double* zn = z + (1 - zp) * Wp * C;
    for (int i = tid; i < 2 * Wp; i += THREADS) sperm[i] = permg[l * 2 * Wp + i];
    __syncthreads();
    auto vval = [&](int src, int n) -> double {
      if (src < Wp) return zc[src * C + n];
      return has_next ? rhs_val(l + 1, src - Wp, n) : 0.0;
    };
    for (int idx = tid; idx < Wp * C; idx += THREADS) {
      const int r = idx / C, n = idx % C;
      tt[idx] = vval(sperm[r], n);
    }
    // warp w owns local m tiles w, w+8, ... of this CTA's slice (fmn <= 10)
    double acc[2][2];
    int mts[2];
#pragma unroll
    for (int u = 0; u < 2; u++) {
      const int lm = warp + 8 * u;
      mts[u] = lm < fmn ? fm0 + lm : -1;
      acc[u][0] = acc[u][1] = 0.0;
      if (mts[u] >= MTH) {  // bottom half: z_{l+1} = t_bot + Fbot t_top
        const int row = (mts[u] - MTH) * 8 + g;
        const int src = sperm[Wp + row];
        acc[u][0] = vval(src, 2 * t);
        acc[u][1] = vval(src, 2 * t + 1);
      }
    }
    __syncthreads();
    pq = clock64(); pa += pq - P0; P0 = pq;
    for (int j = 0; j < kf; j++) {
      const double* A = acquire();
      issue();
#pragma unroll
      for (int kk = 0; kk < 2; kk++) {
        const double bf = tt[(j * 8 + kk * 4 + t) * C + g];
#pragma unroll
        for (int u = 0; u < 2; u++)
          if (mts[u] >= 0) dmma884(acc[u][0], acc[u][1], A[kk * fmn * 32 + (warp + 8 * u) * 32 + lane], bf);
      }
      release();
    }
    pq = clock64(); pb += pq - P0; P0 = pq;
    double* ylev = ybase + l * (int64_t)Wp * C;
#pragma unroll
    for (int u = 0; u < 2; u++) {
      if (mts[u] < 0) continue;
      if (mts[u] < MTH) {
        const int row = mts[u] * 8 + g;
        ylev[row * C + 2 * t] = acc[u][0];
        ylev[row * C + 2 * t + 1] = acc[u][1];
      } else {
        const int row = (mts[u] - MTH) * 8 + g;
        zn[row * C + 2 * t] = acc[u][0];
        zn[row * C + 2 * t + 1] = acc[u][1];
      }
    }
    cluster.sync();
    pq = clock64(); pc += pq - P0; P0 = pq;
    // all-gather z_{l+1}: rows of the bottom m tiles owned by other CTAs
    for (int r = 0; r < G; r++) {
      if (r == rank) continue;
      const int m0 = mtile0_of(MTF, r), mn = mtiles_of(MTF, r);
      const int lo = max(m0, MTH) - MTH, hi = m0 + mn - MTH;  // bottom tiles [lo, hi)
      if (hi <= lo) continue;
      const double* rz = cluster.map_shared_rank(zn, r);
      for (int idx = tid; idx < (hi - lo) * 8 * C; idx += THREADS) {
        const int e = lo * 8 * C + idx;
        zn[e] = rz[e];
      }
    }
    zp = 1 - zp;
    pq = clock64(); pd += pq - P0; P0 = pq;
  }
  if (task == 0 && rank == 0 && tid == 0)
    printf("SOLVE fwd phases (cycles, %lld levels): prologue %lld  kloop %lld  store+sync %lld  gather %lld\n",
           (long long)n2, pa, pb, pc, pd);
  cluster.sync();

  // ---------------- backward ----------------
  for (int idx = tid; idx < 3 * Wp * C; idx += THREADS) xb[idx] = 0.0;
  __syncthreads();
  int i1 = 1, i2 = 2, i0 = 0;  // x_{l+1} in xb[i1], x_{l+2} in xb[i2], x_l written into xb[i0]
  for (int64_t l = n2 - 1; l >= 0; l--) {
    const int kbl = u13[l] ? kb : kb / 2;
    const double* ylev = ybase + l * (int64_t)Wp * C;
    const double* x1 = xb + i1 * Wp * C;
    const double* x2 = xb + i2 * Wp * C;
    double* x0 = xb + i0 * Wp * C;
    double acc[2][2];
    int mts[2];
#pragma unroll
    for (int u = 0; u < 2; u++) {
      const int lm = warp + 8 * u;
      mts[u] = lm < bmn ? bm0 + lm : -1;
      acc[u][0] = acc[u][1] = 0.0;
      if (mts[u] >= 0) {
        const int row = mts[u] * 8 + g;
        acc[u][0] = -ylev[row * C + 2 * t];
        acc[u][1] = -ylev[row * C + 2 * t + 1];
      }
    }
    for (int j = 0; j < kbl; j++) {
      const double* A = acquire();
      issue();
      const double* xs = (j * 8 < Wp) ? x1 : x2;
      const int kbase = (j * 8 < Wp) ? j * 8 : j * 8 - Wp;
#pragma unroll
      for (int kk = 0; kk < 2; kk++) {
        const double bf = xs[(kbase + kk * 4 + t) * C + g];
#pragma unroll
        for (int u = 0; u < 2; u++)
          if (mts[u] >= 0) dmma884(acc[u][0], acc[u][1], A[kk * bmn * 32 + (warp + 8 * u) * 32 + lane], bf);
      }
      release();
    }
#pragma unroll
    for (int u = 0; u < 2; u++) {
      if (mts[u] < 0) continue;
      const int row = mts[u] * 8 + g;
      x0[row * C + 2 * t] = -acc[u][0];
      x0[row * C + 2 * t + 1] = -acc[u][1];
    }
    cluster.sync();
    for (int r = 0; r < G; r++) {
      if (r == rank) continue;
      const int m0 = mtile0_of(MTH, r), mn = mtiles_of(MTH, r);
      if (mn <= 0) continue;
      const double* rx = cluster.map_shared_rank(x0, r);
      for (int idx = tid; idx < mn * 8 * C; idx += THREADS) {
        const int e = m0 * 8 * C + idx;
        x0[e] = rx[e];
      }
    }
    __syncthreads();
    if (a.mode == SWEEP_RECOVER) {
      // each CTA writes its own row slice
      const int r0 = bm0 * 8, r1 = min((bm0 + bmn) * 8, sd.w);
      for (int idx = tid; idx < (r1 - r0) * ncols; idx += THREADS) {
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
    const int tmp = i2;
    i2 = i1;
    i1 = i0;
    i0 = tmp;
  }
  cluster.sync();
}

}  // namespace

void strip_solve(cudaStream_t st, const SchurArgs& a, int ntasks) {
  const int Wp = a.Wp;
  const int MTF = 2 * (Wp / 8);
  const int slot_d = 2 * ((MTF + G - 1) / G) * 32;
  const size_t smem = (size_t)(2 * Wp * C + Wp * C + 3 * Wp * C + STAGES * slot_d) * sizeof(double) + 2 * Wp * sizeof(int);
  static size_t attr = 0;
  if (smem > attr) {
    SLB_CUDA_CHECK(cudaFuncSetAttribute(strip_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  if ((MTF + G - 1) / G > 16 || (Wp / 8 + G - 1) / G > 16)
    throw CudaFailure(cudaErrorInvalidValue, "strip_solve: slab too wide for the cluster split", __FILE__, __LINE__);
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
  SLB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, strip_solve_kernel, a));
}

}  // namespace slb
