// Randomized HBS compression of the reduced interface blocks (sm_100a).
//
// Reference: hbs_compress_adaptive / hbs_compress (proj/include/slablu/hbs_compress.hpp:
// 90-311) on the telescoping HBS format of hbs.hpp:100-154 over the cluster tree of
// cluster_tree.hpp:42-111, dispatched from build_reduced (stage_one.hpp:379-397) as the
// reference's default for n2 >= 512 (driver.hpp:125-130).  The reference samples each block
// matrix-free (one dgbtrs per column); on the GPU the dense Schur sweep forms every block at
// ~0.68 of the FP64 tensor peak and a random column costs as much as a dense one there (the
// forward sweep of a random column starts at level 0, an identity column at its own level),
// so the engine samples the dense blocks with DMMA GEMMs (Y = T Omega, Z = T^T Psi: the same
// operator the reference's sampler applies) and runs the reference's recovery on the samples.
//
// Recovery (build_from_samples, hbs_compress.hpp:90-158) per tree level, bottom up, one CTA
// per (block, node): with ym/omm/zm/psm the node's stacked samples (leaf rows of the pools, or
// the children's projected samples),
//   omm^T = Q1 R (Householder)         -> nullspace of omm = complement of Q1, pinv via R
//   E = ym (I - Q1 Q1^T) = ym N N^T    -> same left singular vectors as ym N
//   E^T = Q_E R_E, one-sided Jacobi on R_E^T -> left singular vectors + values of ym N
//   u = those with sigma > trunc_rel * scale, at most min(r, rows) (orth_columns_floor)
//   f = (I - u u^T) ym pinv(omm), g likewise, d = f + u (u^T g^T); projected samples for the
//   parent exactly as hbs_compress.hpp:146-153.  The root keeps d = ym pinv(omm).
// Numerically the Householder/Jacobi route replaces Eigen's BDCSVD + complete orthogonal
// decomposition: the same subspaces and singular values to round-off (singular vectors are
// defined up to sign and rotation inside degenerate clusters, which the represented operator
// does not see).
//
// Probe and densify: the HBS operator is applied level by level (hbs.hpp:100-147) to the
// probe columns (residual estimate, hbs_compress.hpp:161-183) and finally to the identity
// (to_dense); the dense approximation overwrites the block for the sweep stage.
//
// Random numbers: Philox-4x32-10 counter-based normals keyed by the reference's per-task
// seeds (mix_seed(seed, ordinal) then mix_seed(., 1 | 2 | 100), common.hpp:64-69); the
// streams differ from libstdc++'s mt19937_64 + normal_distribution, so samples are not
// bit-identical to the reference's; the compressed blocks agree with it to the compression
// tolerance, which is the reference's own contract (test_stage_one.cpp:347-369).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "host.h"
#include "kernels.h"

namespace slb {
namespace {

constexpr int HT = 256;  // threads per node CTA
constexpr int HW = HT / 32;

// ---------------------------------------------------------------------------
// Philox-4x32-10 normals
__host__ __device__ inline uint64_t mix_seed_dev(uint64_t seed, uint64_t salt) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__device__ inline void philox(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; r++) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = (uint32_t)p1;
    c[2] = n2;
    c[3] = (uint32_t)p0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// out[r + c * ld] = N(0, 1) for rows [0, rows), columns [0, cols); the value depends only on
// (key, row, col0 + c).
__global__ void gauss_fill_kernel(double* out, int64_t ld, int64_t rows, int64_t cols, int64_t col0, uint64_t key) {
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % rows, c = e / rows;
    uint32_t ctr[4] = {(uint32_t)r, (uint32_t)(r >> 32), (uint32_t)(col0 + c), (uint32_t)((col0 + c) >> 32)};
    philox(ctr, (uint32_t)key, (uint32_t)(key >> 32));
    const uint64_t a = ((uint64_t)ctr[0] << 32) | ctr[1], b = ((uint64_t)ctr[2] << 32) | ctr[3];
    const double u1 = ((double)(a >> 11) + 0.5) * 0x1.0p-53;  // (0, 1)
    const double u2 = (double)(b >> 11) * 0x1.0p-53;
    out[r + c * ld] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
  }
}

// ---------------------------------------------------------------------------
// CTA-level dense helpers (column major, global memory; sm = dynamic shared scratch)
__device__ inline double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = lane < HW ? red[lane] : 0.0;
  t = warp_sum(t);
  return t;  // every thread holds the sum
}

// C (M x N, ldc) = alpha * op(A) * op(B) + beta * C; op(A) is M x K, op(B) is K x N.
// 64 x 64 output tiles, 16-deep K slices staged in shared memory, 4 x 4 outputs per thread.
template <bool TA, bool TB>
__device__ void cta_gemm(int M, int N, int K, double alpha, const double* A, int64_t lda, const double* B,
                         int64_t ldb, double beta, double* C, int64_t ldc, double* sm) {
  double* As = sm;              // [16][65]
  double* Bs = sm + 16 * 65;    // [16][65]
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  for (int m0 = 0; m0 < M; m0 += 64)
    for (int n0 = 0; n0 < N; n0 += 64) {
      double acc[4][4];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = 0.0;
      for (int k0 = 0; k0 < K; k0 += 16) {
        __syncthreads();
        for (int e = tid; e < 16 * 64; e += HT) {
          int m, k;
          if (TA) { k = e & 15; m = e >> 4; } else { m = e & 63; k = e >> 6; }
          const int gm = m0 + m, gk = k0 + k;
          As[k * 65 + m] = (gm < M && gk < K) ? (TA ? A[gk + (int64_t)gm * lda] : A[gm + (int64_t)gk * lda]) : 0.0;
        }
        for (int e = tid; e < 16 * 64; e += HT) {
          int n, k;
          if (TB) { n = e & 63; k = e >> 6; } else { k = e & 15; n = e >> 4; }
          const int gn = n0 + n, gk = k0 + k;
          Bs[k * 65 + n] = (gn < N && gk < K) ? (TB ? B[gn + (int64_t)gk * ldb] : B[gk + (int64_t)gn * ldb]) : 0.0;
        }
        __syncthreads();
#pragma unroll 4
        for (int k = 0; k < 16; k++) {
          double a[4], b[4];
#pragma unroll
          for (int i = 0; i < 4; i++) a[i] = As[k * 65 + tx + 16 * i];
#pragma unroll
          for (int j = 0; j < 4; j++) b[j] = Bs[k * 65 + ty + 16 * j];
#pragma unroll
          for (int i = 0; i < 4; i++)
#pragma unroll
            for (int j = 0; j < 4; j++) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const int gm = m0 + tx + 16 * i, gn = n0 + ty + 16 * j;
          if (gm < M && gn < N) {
            double* c = C + gm + (int64_t)gn * ldc;
            *c = alpha * acc[i][j] + (beta != 0.0 ? beta * *c : 0.0);
          }
        }
    }
  __syncthreads();
}

// dst (rows x cols, ldd) = src (rows x cols, lds)
__device__ void cta_copy(double* dst, int64_t ldd, const double* src, int64_t lds, int rows, int cols) {
  for (int64_t e = threadIdx.x; e < (int64_t)rows * cols; e += HT) {
    const int r = (int)(e % rows), c = (int)(e / rows);
    dst[r + c * ldd] = src[r + c * lds];
  }
  __syncthreads();
}

// Householder QR in place (LAPACK dgeqr2 conventions): A (S x m, S >= m) -> R in the upper
// triangle, reflector tails below the diagonal (v_i(i) = 1 implicit), tau[i].
__device__ void cta_qr(double* A, int64_t lda, int S, int m, double* tau, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = 0; i < m; i++) {
    double* col = A + (int64_t)i * lda;
    double s2 = 0.0;
    for (int r = i + 1 + threadIdx.x; r < S; r += HT) s2 += col[r] * col[r];
    s2 = block_sum(s2, red);
    const double alpha = col[i];
    double t = 0.0, beta = alpha;
    if (s2 > 0.0) {
      beta = -copysign(sqrt(alpha * alpha + s2), alpha);
      t = (beta - alpha) / beta;
      const double sc = 1.0 / (alpha - beta);
      for (int r = i + 1 + threadIdx.x; r < S; r += HT) col[r] *= sc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      col[i] = beta;
      tau[i] = t;
    }
    if (t != 0.0)
      for (int c = i + 1 + w; c < m; c += HW) {
        double* cc = A + (int64_t)c * lda;
        double acc = lane == 0 ? cc[i] : 0.0;
        for (int r = i + 1 + lane; r < S; r += 32) acc += col[r] * cc[r];
        acc = warp_sum(acc) * t;
        if (lane == 0) cc[i] -= acc;
        for (int r = i + 1 + lane; r < S; r += 32) cc[r] -= acc * col[r];
      }
    __syncthreads();
  }
}

// Q (S x m, ldq) = the first m columns of H_0 ... H_{m-1} from cta_qr's reflectors.
__device__ void cta_form_q(const double* A, int64_t lda, int S, int m, const double* tau, double* Q, int64_t ldq) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t e = threadIdx.x; e < (int64_t)S * m; e += HT) {
    const int r = (int)(e % S), c = (int)(e / S);
    Q[r + c * ldq] = r == c ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int i = m - 1; i >= 0; i--) {
    const double t = tau[i];
    const double* v = A + (int64_t)i * lda;
    if (t != 0.0)
      for (int c = i + w; c < m; c += HW) {
        double* qc = Q + (int64_t)c * ldq;
        double acc = lane == 0 ? qc[i] : 0.0;
        for (int r = i + 1 + lane; r < S; r += 32) acc += v[r] * qc[r];
        acc = warp_sum(acc) * t;
        if (lane == 0) qc[i] -= acc;
        for (int r = i + 1 + lane; r < S; r += 32) qc[r] -= acc * v[r];
      }
    __syncthreads();
  }
}

// X (mb x n, ldx) <- X R^{-T}, R upper triangular n x n (ldr): row by row back substitution of
// R x^T = b^T.  A zero diagonal (rank-deficient sample block) zeroes that component.
__device__ void cta_trsm_rt(double* X, int64_t ldx, int mb, const double* R, int64_t ldr, int n) {
  for (int row = threadIdx.x; row < mb; row += HT) {
    for (int j = n - 1; j >= 0; j--) {
      double s = X[row + (int64_t)j * ldx];
      for (int k = j + 1; k < n; k++) s -= R[j + (int64_t)k * ldr] * X[row + (int64_t)k * ldx];
      const double dj = R[j + (int64_t)j * ldr];
      X[row + (int64_t)j * ldx] = dj != 0.0 ? s / dj : 0.0;
    }
  }
  __syncthreads();
}

// One-sided (Hestenes) Jacobi on the columns of M (m x m, ldm): afterwards the columns are
// mutually orthogonal, M = W V^T with W = U Sigma.  Then the columns are ranked by norm and the
// leading ones above floor_tol (at most cap) are written normalised to U (m x ru, ldu): the
// left singular vectors of the original M.  Returns ru.  Parallel round-robin ordering: each
// step rotates m/2 disjoint pairs, one warp per pair.
__device__ int cta_jacobi_basis(double* M, int64_t ldm, int m, double floor_tol, int cap, double* U, int64_t ldu,
                                double* sig, int* sflag) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int mp = m + (m & 1);
  for (int sweep = 0; sweep < 60 && m > 1; sweep++) {
    if (threadIdx.x == 0) *sflag = 0;
    __syncthreads();
    for (int s = 0; s < mp - 1; s++) {
      // two pairs per warp at a time (their reductions and rotation arithmetic interleave)
      for (int k0 = w; k0 < mp / 2; k0 += 2 * HW) {
        double* cp[2];
        double* cq[2];
        bool ok[2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int k = k0 + h * HW;
          int p = 0, q = 0;
          if (k == 0) {
            p = mp - 1;
            q = s;
          } else {
            p = (s + k) % (mp - 1);
            q = (s - k + mp - 1) % (mp - 1);
          }
          ok[h] = k < mp / 2 && p < m && q < m;
          cp[h] = M + (int64_t)(ok[h] ? p : 0) * ldm;
          cq[h] = M + (int64_t)(ok[h] ? q : 0) * ldm;
        }
        double a[2] = {0.0, 0.0}, b[2] = {0.0, 0.0}, c[2] = {0.0, 0.0};
        for (int r = lane; r < m; r += 32) {
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const double x = cp[h][r], y = cq[h][r];
            a[h] += x * x;
            b[h] += y * y;
            c[h] += x * y;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int h = 0; h < 2; h++) {
            a[h] += __shfl_xor_sync(0xffffffffu, a[h], o);
            b[h] += __shfl_xor_sync(0xffffffffu, b[h], o);
            c[h] += __shfl_xor_sync(0xffffffffu, c[h], o);
          }
        double cs[2], sn[2];
        bool rot[2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
          rot[h] = ok[h] && c[h] != 0.0 && c[h] * c[h] > 1e-30 * a[h] * b[h];
          const double zeta = rot[h] ? (b[h] - a[h]) / (2.0 * c[h]) : 0.0;
          const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          cs[h] = rsqrt(1.0 + t * t);
          sn[h] = cs[h] * t;
        }
        if (rot[0] || rot[1]) {
          for (int r = lane; r < m; r += 32) {
#pragma unroll
            for (int h = 0; h < 2; h++) {
              if (!rot[h]) continue;
              const double x = cp[h][r], y = cq[h][r];
              cp[h][r] = cs[h] * x - sn[h] * y;
              cq[h][r] = sn[h] * x + cs[h] * y;
            }
          }
          if (lane == 0) *sflag = 1;
        }
      }
      __syncthreads();
    }
    const int rotated = *sflag;
    __syncthreads();
    if (!rotated) break;
  }
  // column norms
  for (int c = w; c < m; c += HW) {
    const double* cc = M + (int64_t)c * ldm;
    double a = 0.0;
    for (int r = lane; r < m; r += 32) a += cc[r] * cc[r];
    a = warp_sum(a);
    if (lane == 0) sig[c] = sqrt(a);
  }
  __syncthreads();
  // rank of each column (descending norm, ties by index); count above the floor
  int above = 0;
  for (int c = 0; c < m; c++) above += sig[c] > floor_tol ? 1 : 0;
  const int ru = min(above, cap);
  for (int c = threadIdx.x; c < m; c += HT) {
    int rk = 0;
    for (int o = 0; o < m; o++) rk += (sig[o] > sig[c] || (sig[o] == sig[c] && o < c)) ? 1 : 0;
    if (rk < ru) {
      const double inv = 1.0 / sig[c];
      for (int r = 0; r < m; r++) U[r + (int64_t)rk * ldu] = M[r + (int64_t)c * ldm] * inv;
    }
  }
  __syncthreads();
  return ru;
}

// ---------------------------------------------------------------------------
// Per-node layout.  Offsets (doubles) into the block's arenas; ranks live in `rk`.
struct NodeDesc {
  int begin, size, left, right, parent, leaf;
  int mcap, rcap;        // stacked-sample rows capacity, generator width capacity
  int64_t o_u, o_v, o_d;                 // persistent: u (mcap x rcap), v, d (mcap x mcap); ld mcap
  int64_t o_w;                            // level work area (see build kernel)
  int64_t o_hy, o_hz, o_hom, o_hps;       // projected samples (S x rcap each, ld S) in the hat arena
};
// rk[4 * node]: mu, mv, ru, rv

struct BuildArgs {
  const NodeDesc* nodes;
  const int* level_nodes;  // node ids of this level
  int n;                   // operator dimension
  int S;                   // sample columns
  int r;                   // working rank
  double* const* pools;    // per block: OM | Y | PS | Z (n x S each, ld n)
  int64_t pool_ld;         // n
  int64_t pool_stride;     // doubles between OM, Y, PS, Z inside one block's pool
  double* const* persist;  // per block
  double* const* work;     // per block
  double* const* hats_cur; // per block: hat arena written by this level
  double* const* hats_kid; // per block: hat arena of the children's level
  int* const* rk;          // per block: 4 ints per node
  const double* floor_tol; // per block
};

// Work area of a node (doubles, offsets relative to o_w): 6 x S x mcap + small squares.
__host__ __device__ inline int64_t work_doubles(int64_t S, int64_t mcap) {
  return 6 * S * mcap + 8 * mcap * mcap + 2 * mcap + 64;
}

__global__ void __launch_bounds__(HT) hbs_build_level_kernel(BuildArgs a) {
  extern __shared__ double sm[];
  double* red = sm + 2 * 16 * 65;
  int* sflag = reinterpret_cast<int*>(red + 32);
  const int id = a.level_nodes[blockIdx.x];
  const int b = blockIdx.y;
  const NodeDesc nd = a.nodes[id];
  const int S = a.S;
  double* pools = a.pools[b];
  const double* OM = pools;
  const double* Y = pools + a.pool_stride;
  const double* PS = pools + 2 * a.pool_stride;
  const double* Z = pools + 3 * a.pool_stride;
  double* P = a.persist[b];
  double* W = a.work[b] + nd.o_w;
  int* rk = a.rk[b];
  const int64_t mc = nd.mcap;
  double* yT = W;
  double* omT = yT + S * mc;
  double* zT = omT + S * mc;
  double* psT = zT + S * mc;
  double* W1 = psT + S * mc;
  double* W2 = W1 + S * mc;
  double* Rom = W2 + S * mc;
  double* Rps = Rom + mc * mc;
  double* B1 = Rps + mc * mc;
  double* C1 = B1 + mc * mc;
  double* Mj = C1 + mc * mc;
  double* T1 = Mj + mc * mc;
  double* T2 = T1 + mc * mc;
  double* G = T2 + mc * mc;
  double* tau = G + mc * mc;
  double* sig = tau + mc;
  double* u = P + nd.o_u;
  double* v = P + nd.o_v;
  double* d = P + nd.o_d;

  // stacked samples, transposed (column c of yT = row c of ym)
  int mu, mv;
  if (nd.leaf) {
    mu = mv = nd.size;
    for (int64_t e = threadIdx.x; e < (int64_t)S * nd.size; e += HT) {
      const int s = (int)(e % S), t = (int)(e / S);
      const int64_t src = nd.begin + t + (int64_t)s * a.pool_ld;
      yT[s + t * S] = Y[src];
      omT[s + t * S] = OM[src];
      zT[s + t * S] = Z[src];
      psT[s + t * S] = PS[src];
    }
    __syncthreads();
  } else {
    const NodeDesc L = a.nodes[nd.left], R = a.nodes[nd.right];
    const int rul = rk[4 * nd.left + 2], rvl = rk[4 * nd.left + 3];
    const int rur = rk[4 * nd.right + 2], rvr = rk[4 * nd.right + 3];
    mu = rul + rur;
    mv = rvl + rvr;
    const double* H = a.hats_kid[b];
    cta_copy(yT, S, H + L.o_hy, S, S, rul);
    cta_copy(yT + (int64_t)rul * S, S, H + R.o_hy, S, S, rur);
    cta_copy(psT, S, H + L.o_hps, S, S, rul);
    cta_copy(psT + (int64_t)rul * S, S, H + R.o_hps, S, S, rur);
    cta_copy(omT, S, H + L.o_hom, S, S, rvl);
    cta_copy(omT + (int64_t)rvl * S, S, H + R.o_hom, S, S, rvr);
    cta_copy(zT, S, H + L.o_hz, S, S, rvl);
    cta_copy(zT + (int64_t)rvl * S, S, H + R.o_hz, S, S, rvr);
  }
  const bool root = nd.parent < 0;

  // u side: omm^T = Q1 Rom; B1 = ym Q1 (mu x mv)
  cta_copy(W1, S, omT, S, S, mv);
  cta_qr(W1, S, S, mv, tau, red);
  for (int64_t e = threadIdx.x; e < (int64_t)mv * mv; e += HT) {
    const int i = (int)(e % mv), j = (int)(e / mv);
    Rom[i + j * mc] = i <= j ? W1[i + (int64_t)j * S] : 0.0;
  }
  cta_form_q(W1, S, S, mv, tau, W2, S);
  cta_gemm<true, false>(mu, mv, S, 1.0, yT, S, W2, S, 0.0, B1, mc, sm);
  if (root) {  // d = ym pinv(omm) = B1 Rom^{-T}
    cta_trsm_rt(B1, mc, mu, Rom, mc, mv);
    cta_copy(d, mc, B1, mc, mu, mv);
    if (threadIdx.x == 0) {
      rk[4 * id + 0] = mu;
      rk[4 * id + 1] = mv;
      rk[4 * id + 2] = 0;
      rk[4 * id + 3] = 0;
    }
    return;
  }
  const int cap = min(a.r, min(mu, mv));
  const double ftol = a.floor_tol[b];
  // E^T = ym^T - Q1 B1^T (S x mu); R_E; Jacobi on R_E^T
  cta_copy(W1, S, yT, S, S, mu);
  cta_gemm<false, true>(S, mu, mv, -1.0, W2, S, B1, mc, 1.0, W1, S, sm);
  cta_qr(W1, S, S, mu, tau, red);
  for (int64_t e = threadIdx.x; e < (int64_t)mu * mu; e += HT) {
    const int i = (int)(e % mu), j = (int)(e / mu);  // Mj = R_E^T
    Mj[i + j * mc] = j <= i ? W1[j + (int64_t)i * S] : 0.0;
  }
  __syncthreads();
  const int ru = cta_jacobi_basis(Mj, mc, mu, ftol, cap, u, mc, sig, sflag);

  // v side: psm^T = Q1' Rps; C1 = zm Q1' (mv x mu)
  cta_copy(W1, S, psT, S, S, mu);
  cta_qr(W1, S, S, mu, tau, red);
  for (int64_t e = threadIdx.x; e < (int64_t)mu * mu; e += HT) {
    const int i = (int)(e % mu), j = (int)(e / mu);
    Rps[i + j * mc] = i <= j ? W1[i + (int64_t)j * S] : 0.0;
  }
  cta_form_q(W1, S, S, mu, tau, W2, S);
  cta_gemm<true, false>(mv, mu, S, 1.0, zT, S, W2, S, 0.0, C1, mc, sm);
  cta_copy(W1, S, zT, S, S, mv);
  cta_gemm<false, true>(S, mv, mu, -1.0, W2, S, C1, mc, 1.0, W1, S, sm);
  cta_qr(W1, S, S, mv, tau, red);
  for (int64_t e = threadIdx.x; e < (int64_t)mv * mv; e += HT) {
    const int i = (int)(e % mv), j = (int)(e / mv);
    Mj[i + j * mc] = j <= i ? W1[j + (int64_t)i * S] : 0.0;
  }
  __syncthreads();
  const int rv = cta_jacobi_basis(Mj, mc, mv, ftol, cap, v, mc, sig, sflag);

  // f = (I - u u^T) B1 Rom^{-T} -> d;  g = (I - v v^T) C1 Rps^{-T} -> G;  d += u (g u)^T
  cta_trsm_rt(B1, mc, mu, Rom, mc, mv);
  cta_copy(d, mc, B1, mc, mu, mv);
  cta_gemm<true, false>(ru, mv, mu, 1.0, u, mc, B1, mc, 0.0, T1, mc, sm);   // T1 = u^T X
  cta_gemm<false, false>(mu, mv, ru, -1.0, u, mc, T1, mc, 1.0, d, mc, sm);  // d = X - u T1
  cta_trsm_rt(C1, mc, mv, Rps, mc, mu);
  cta_copy(G, mc, C1, mc, mv, mu);
  cta_gemm<true, false>(rv, mu, mv, 1.0, v, mc, C1, mc, 0.0, T1, mc, sm);
  cta_gemm<false, false>(mv, mu, rv, -1.0, v, mc, T1, mc, 1.0, G, mc, sm);
  cta_gemm<false, false>(mv, ru, mu, 1.0, G, mc, u, mc, 0.0, T2, mc, sm);   // T2 = g u (mv x ru)
  cta_gemm<false, true>(mu, mv, ru, 1.0, u, mc, T2, mc, 1.0, d, mc, sm);    // d += u T2^T

  // projected samples for the parent (hbs_compress.hpp:146-153), transposed
  double* Hc = a.hats_cur[b];
  double* yh = Hc + nd.o_hy;
  double* zh = Hc + nd.o_hz;
  double* omh = Hc + nd.o_hom;
  double* psh = Hc + nd.o_hps;
  cta_gemm<true, false>(mv, ru, mu, 1.0, d, mc, u, mc, 0.0, T1, mc, sm);    // T1 = d^T u (mv x ru)
  cta_gemm<false, false>(S, ru, mu, 1.0, yT, S, u, mc, 0.0, yh, S, sm);
  cta_gemm<false, false>(S, ru, mv, -1.0, omT, S, T1, mc, 1.0, yh, S, sm);
  cta_gemm<false, false>(mu, rv, mv, 1.0, d, mc, v, mc, 0.0, T2, mc, sm);   // T2 = d v (mu x rv)
  cta_gemm<false, false>(S, rv, mv, 1.0, zT, S, v, mc, 0.0, zh, S, sm);
  cta_gemm<false, false>(S, rv, mu, -1.0, psT, S, T2, mc, 1.0, zh, S, sm);
  cta_gemm<false, false>(S, rv, mv, 1.0, omT, S, v, mc, 0.0, omh, S, sm);
  cta_gemm<false, false>(S, ru, mu, 1.0, psT, S, u, mc, 0.0, psh, S, sm);
  if (threadIdx.x == 0) {
    rk[4 * id + 0] = mu;
    rk[4 * id + 1] = mv;
    rk[4 * id + 2] = ru;
    rk[4 * id + 3] = rv;
  }
}

// ---------------------------------------------------------------------------
// Apply (hbs.hpp:100-147): Y = H X or H^T X for nc columns, level by level.  xh / yh of a
// node: (rcap x nc, ld rcap) at o_x[node] in per-block apply arenas; one CTA per (node, block,
// 64-column chunk).
struct ApplyArgs {
  const NodeDesc* nodes;
  const int* level_nodes;
  int nc;
  int adj;
  double* const* persist;
  int* const* rk;
  const double* const* X;  // per block, n x nc (ld ldx)
  double* const* Yout;     // per block, n x nc (ld ldy)
  int64_t ldx, ldy;
  double* const* xh;       // per block arena
  double* const* yh;
  const int64_t* o_x;      // per node offset in the xh / yh arenas
};

__global__ void __launch_bounds__(HT) hbs_apply_up_kernel(ApplyArgs a) {
  extern __shared__ double sm[];
  const int id = a.level_nodes[blockIdx.x];
  const int b = blockIdx.y;
  const int c0 = blockIdx.z * 64, nc = min(64, a.nc - c0);
  const NodeDesc nd = a.nodes[id];
  if (nd.parent < 0) return;
  const int* rk = a.rk[b];
  const double* P = a.persist[b];
  const double* G = P + (a.adj ? nd.o_u : nd.o_v);
  const int w = rk[4 * id + (a.adj ? 2 : 3)];
  double* out = a.xh[b] + a.o_x[id] + (int64_t)c0 * nd.rcap;
  if (nd.leaf) {
    cta_gemm<true, false>(w, nc, nd.size, 1.0, G, nd.mcap, a.X[b] + nd.begin + c0 * a.ldx, a.ldx, 0.0, out,
                          nd.rcap, sm);
  } else {
    const NodeDesc L = a.nodes[nd.left], R = a.nodes[nd.right];
    const int kl = rk[4 * nd.left + (a.adj ? 2 : 3)], kr = rk[4 * nd.right + (a.adj ? 2 : 3)];
    cta_gemm<true, false>(w, nc, kl, 1.0, G, nd.mcap, a.xh[b] + a.o_x[nd.left] + (int64_t)c0 * L.rcap, L.rcap, 0.0,
                          out, nd.rcap, sm);
    cta_gemm<true, false>(w, nc, kr, 1.0, G + kl, nd.mcap, a.xh[b] + a.o_x[nd.right] + (int64_t)c0 * R.rcap, R.rcap,
                          1.0, out, nd.rcap, sm);
  }
}

__global__ void __launch_bounds__(HT) hbs_apply_down_kernel(ApplyArgs a) {
  extern __shared__ double sm[];
  const int id = a.level_nodes[blockIdx.x];
  const int b = blockIdx.y;
  const int c0 = blockIdx.z * 64, nc = min(64, a.nc - c0);
  const NodeDesc nd = a.nodes[id];
  const int* rk = a.rk[b];
  const double* P = a.persist[b];
  const double* d = P + nd.o_d;
  const double* H = P + (a.adj ? nd.o_v : nd.o_u);  // expansion generator
  const bool root = nd.parent < 0;
  const int hw = root ? 0 : rk[4 * id + (a.adj ? 3 : 2)];
  const double* yhp = root ? nullptr : a.yh[b] + a.o_x[id] + (int64_t)c0 * nd.rcap;
  const int64_t ldd = nd.mcap;
  if (nd.leaf) {
    double* y = a.Yout[b] + nd.begin + c0 * a.ldy;
    const double* x = a.X[b] + nd.begin + c0 * a.ldx;
    if (a.adj)
      cta_gemm<true, false>(nd.size, nc, nd.size, 1.0, d, ldd, x, a.ldx, 0.0, y, a.ldy, sm);
    else
      cta_gemm<false, false>(nd.size, nc, nd.size, 1.0, d, ldd, x, a.ldx, 0.0, y, a.ldy, sm);
    if (hw > 0) cta_gemm<false, false>(nd.size, nc, hw, 1.0, H, ldd, yhp, nd.rcap, 1.0, y, a.ldy, sm);
    return;
  }
  const NodeDesc L = a.nodes[nd.left], R = a.nodes[nd.right];
  // x side widths of the children (stacked input) and y side widths (outputs)
  const int xl = rk[4 * nd.left + (a.adj ? 2 : 3)], xr = rk[4 * nd.right + (a.adj ? 2 : 3)];
  const int yl = rk[4 * nd.left + (a.adj ? 3 : 2)], yr = rk[4 * nd.right + (a.adj ? 3 : 2)];
  const double* xhl = a.xh[b] + a.o_x[nd.left] + (int64_t)c0 * L.rcap;
  const double* xhr = a.xh[b] + a.o_x[nd.right] + (int64_t)c0 * R.rcap;
  double* yhl = a.yh[b] + a.o_x[nd.left] + (int64_t)c0 * L.rcap;
  double* yhr = a.yh[b] + a.o_x[nd.right] + (int64_t)c0 * R.rcap;
  // core(i, j) = adj ? d(j, i) : d(i, j); rows split (yl | yr), columns split (xl | xr)
  for (int half = 0; half < 2; half++) {
    const int r0 = half ? yl : 0, nr = half ? yr : yl;
    double* out = half ? yhr : yhl;
    const int64_t ldo = half ? R.rcap : L.rcap;
    if (nr == 0) continue;
    if (a.adj) {
      cta_gemm<true, false>(nr, nc, xl, 1.0, d + (int64_t)r0 * ldd, ldd, xhl, L.rcap, 0.0, out, ldo, sm);
      cta_gemm<true, false>(nr, nc, xr, 1.0, d + xl + (int64_t)r0 * ldd, ldd, xhr, R.rcap, 1.0, out, ldo, sm);
    } else {
      cta_gemm<false, false>(nr, nc, xl, 1.0, d + r0, ldd, xhl, L.rcap, 0.0, out, ldo, sm);
      cta_gemm<false, false>(nr, nc, xr, 1.0, d + r0 + (int64_t)xl * ldd, ldd, xhr, R.rcap, 1.0, out, ldo, sm);
    }
    if (hw > 0) cta_gemm<false, false>(nr, nc, hw, 1.0, H + r0, ldd, yhp, nd.rcap, 1.0, out, ldo, sm);
  }
}

// ---------------------------------------------------------------------------
// ||A||_F^2 for up to 4 matrices per block (n x cols, ld n): out[4 * b + q]
constexpr int NB_NORM = 32;  // blocks per norms launch (kernel-parameter size)
struct NormArgs {
  const double* p[NB_NORM][4];
  int64_t rows;
  int64_t cols[4];
  int64_t ld;
  const double* sub[NB_NORM][4];  // optional: norm of (p - sub)
  double* out;
};
__global__ void norms_kernel(NormArgs a) {
  __shared__ double red[32];
  const int b = blockIdx.y, q = blockIdx.x;
  const double* p = a.p[b][q];
  const double* s = a.sub[b][q];
  double acc = 0.0;
  if (p)
    for (int64_t e = threadIdx.x; e < a.rows * a.cols[q]; e += blockDim.x) {
      const int64_t r = e % a.rows, c = e / a.rows;
      const double x = p[r + c * a.ld] - (s ? s[r + c * a.ld] : 0.0);
      acc += x * x;
    }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (int)(blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) a.out[4 * b + q] = t;
  }
}

__global__ void set_identity_kernel(double* a, int64_t n) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x)
    a[e] = (e % n == e / n) ? 1.0 : 0.0;
}

// ---------------------------------------------------------------------------
// Host side
struct Tree {
  std::vector<NodeDesc> nodes;
  std::vector<std::vector<int>> levels;  // node ids per level, root level 0
};

// cluster_tree.hpp:42-66: breadth-first halving until a range fits the leaf size.
Tree build_tree(int n, int leaf) {
  Tree t;
  t.nodes.push_back(NodeDesc{0, n, -1, -1, -1, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0});
  std::vector<int> level = {0};
  for (size_t k = 0; k < t.nodes.size(); k++) {
    if (t.nodes[k].size <= leaf) continue;
    const int mid = t.nodes[k].begin + t.nodes[k].size / 2;
    const int id = (int)k;
    NodeDesc l{t.nodes[k].begin, mid - t.nodes[k].begin, -1, -1, id, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    NodeDesc r{mid, t.nodes[k].begin + t.nodes[k].size - mid, -1, -1, id, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    t.nodes[k].leaf = 0;
    t.nodes[k].left = (int)t.nodes.size();
    t.nodes.push_back(l);
    t.nodes[k].right = (int)t.nodes.size();
    t.nodes.push_back(r);
  }
  std::vector<int> depth(t.nodes.size(), 0);
  for (size_t k = 1; k < t.nodes.size(); k++) depth[k] = depth[t.nodes[k].parent] + 1;
  const int maxd = *std::max_element(depth.begin(), depth.end());
  t.levels.assign(maxd + 1, {});
  for (size_t k = 0; k < t.nodes.size(); k++) t.levels[depth[k]].push_back((int)k);
  return t;
}

struct Layout {
  int64_t persist = 0, work = 0, hats[2] = {0, 0}, xh = 0;
};

// Capacities and arena offsets for working rank r and S sample columns.
Layout plan_layout(Tree& t, int r, int S) {
  Layout L;
  // capacities bottom up
  for (int lv = (int)t.levels.size() - 1; lv >= 0; lv--)
    for (int id : t.levels[lv]) {
      NodeDesc& nd = t.nodes[id];
      nd.mcap = nd.leaf ? nd.size : t.nodes[nd.left].rcap + t.nodes[nd.right].rcap;
      nd.rcap = std::max(1, std::min(r, nd.mcap));
    }
  for (int lv = (int)t.levels.size() - 1; lv >= 0; lv--) {
    int64_t w = 0, h = 0;
    const int par = lv & 1;
    for (int id : t.levels[lv]) {
      NodeDesc& nd = t.nodes[id];
      const int64_t mc = nd.mcap, rc = nd.rcap;
      nd.o_u = L.persist;
      L.persist += mc * rc;
      nd.o_v = L.persist;
      L.persist += mc * rc;
      nd.o_d = L.persist;
      L.persist += mc * mc;
      nd.o_w = w;
      w += work_doubles(S, mc);
      nd.o_hy = h;
      nd.o_hz = h + (int64_t)S * rc;
      nd.o_hom = h + 2 * (int64_t)S * rc;
      nd.o_hps = h + 3 * (int64_t)S * rc;
      h += 4 * (int64_t)S * rc;
    }
    L.work = std::max(L.work, w);
    L.hats[par] = std::max(L.hats[par], h);
  }
  return L;
}

struct DevMem {
  cudaStream_t st;
  std::vector<void*> ptrs;
  template <class T>
  T* alloc(size_t n) {
    void* p = nullptr;
    SLB_CUDA_CHECK(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), st));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  ~DevMem() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
};

int64_t sample_count(int64_t r) { return 3 * r + 10; }
bool rank_feasible(const Tree& t, int64_t r) {
  if (t.nodes[0].leaf) return sample_count(r) >= t.nodes[0].size;
  int mx = 0;
  for (const NodeDesc& nd : t.nodes)
    if (nd.leaf) mx = std::max(mx, nd.size);
  return sample_count(r) >= mx + r;
}

const size_t kSmemBytes = (2 * 16 * 65 + 32 + 8) * sizeof(double);

}  // namespace

// Device bytes one block needs at the largest round (pools + arenas), and the densify temporaries.
HbsFootprint hbs_footprint(int64_t n, const HbsOptions& o) {
  Tree tt = build_tree((int)n, std::max(1, std::min<int>(o.leaf, (int)n)));
  const int64_t r_top = o.fixed_rank ? o.r_max : std::max<int64_t>(o.r_max, 2);
  const int64_t S_top = sample_count(r_top) + 4 * 64;
  const Layout Lt = plan_layout(tt, (int)r_top, (int)S_top);
  HbsFootprint f;
  f.per_block = 8.0 * (double)(4 * n * S_top + Lt.persist + Lt.work + Lt.hats[0] + Lt.hats[1] + 24 * n);
  int64_t sum_rcap = 0;
  for (const NodeDesc& nd : tt.nodes) sum_rcap += nd.rcap;
  f.densify = 8.0 * (double)(n * n + 2 * sum_rcap * n);
  return f;
}

// Compress nb dense n x n blocks (device, column major, ld n) in place: each becomes the dense
// materialization of its HBS approximation.  seeds[i] is the block's CompressOptions.seed.
// fixed_rank: hbs_compress with rank bound r_max (one round); else hbs_compress_adaptive.
// Blocks are processed in groups that fit the device's free memory.
void hbs_compress_blocks(cudaStream_t st, int64_t n, int nb, double* const* blocks, const uint64_t* seeds,
                         const HbsOptions& o, HbsStats* stats) {
  for (int i = 0; i < nb; i++) stats[i] = HbsStats{};
  if (nb == 0) return;
  if (o.leaf < 1 || o.leaf > n) throw HbsError("ClusterTree: need 1 <= leaf_size <= n", 0.0, true);
  Tree tree = build_tree((int)n, o.leaf);
  if (o.fixed_rank) {
    if (o.r_max < 0) throw HbsError("hbs_compress: negative rank bound", 0.0, true);
    if (!rank_feasible(tree, o.r_max))
      throw HbsError("hbs_compress: rank bound leaves no sketch nullspace at the widest leaf", INFINITY, false);
  } else if (o.r_start > o.r_max) {
    throw HbsError("hbs_compress_adaptive: r_start must be <= r_max", 0.0, true);
  }
  static bool attr = false;
  if (!attr) {
    SLB_CUDA_CHECK(cudaFuncSetAttribute(hbs_build_level_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)kSmemBytes));
    attr = true;
  }
  // blocks per group from the largest round's footprint (pools + arenas + the densify temporaries)
  {
    const HbsFootprint fp = hbs_footprint(n, o);
    size_t fr = 0, tot = 0;
    SLB_CUDA_CHECK(cudaMemGetInfo(&fr, &tot));
    const double budget = 0.6 * (double)fr - fp.densify;
    const int group = (int)std::max<double>(1.0, std::min<double>(256.0, budget / fp.per_block));
    if (group < nb) {
      for (int g0 = 0; g0 < nb; g0 += group) {
        const int ng = std::min(group, nb - g0);
        hbs_compress_blocks(st, n, ng, blocks + g0, seeds + g0, o, stats + g0);
      }
      return;
    }
  }
  const int64_t r_top = o.fixed_rank ? o.r_max : std::max<int64_t>(o.r_max, 2);
  const int64_t S_top = sample_count(r_top) + 4 * 64;
  // the rounds allocate and free their arenas stream-ordered: keep the pool's memory mapped across
  // rounds (a release threshold of 0 would unmap and remap gigabytes at every synchronization)
  // and hand it back to the device once the compression is done
  struct PoolKeep {
    cudaMemPool_t pool = nullptr;
    uint64_t old = 0;
    cudaStream_t st;
    explicit PoolKeep(cudaStream_t s) : st(s) {
      int dev = 0;
      if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) {
        cudaGetLastError();
        pool = nullptr;
        return;
      }
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &old);
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    ~PoolKeep() {
      if (!pool) return;
      cudaStreamSynchronize(st);
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &old);
      cudaMemPoolTrimTo(pool, (size_t)old);
      cudaGetLastError();
    }
  } keep_pool(st);
  DevMem mem{st, {}};
  const int B = nb;
  // per block pools (OM | Y | PS | Z), n x Smax each
  std::vector<int64_t> Scur(B, 0), drawn(B, 0);  // pool columns; columns drawn from the om / ps streams
  int64_t Smax = S_top;
  double* pool = mem.alloc<double>((size_t)B * 4 * n * Smax);
  const int64_t pstride = n * Smax;
  auto OMp = [&](int b) { return pool + (size_t)b * 4 * pstride; };
  auto Yp = [&](int b) { return OMp(b) + pstride; };
  auto PSp = [&](int b) { return OMp(b) + 2 * pstride; };
  auto Zp = [&](int b) { return OMp(b) + 3 * pstride; };
  double* probe = mem.alloc<double>((size_t)B * 8 * n);  // W | MW | Q | MQ | HW | HQ (4 cols each) + spare
  double* probe2 = mem.alloc<double>((size_t)B * 16 * n);
  double* dnorm = mem.alloc<double>((size_t)B * 4);
  std::vector<double> hnorm(4 * (size_t)B);
  std::vector<int> active(B, 1), passed(B, 0);
  std::vector<double> floor_h(B, 0.0);
  int64_t r = o.fixed_rank ? o.r_max : std::max<int64_t>(o.r_start, 2);

  auto fill = [&](double* out, int64_t ld, int64_t rows, int64_t cols, int64_t col0, uint64_t key) {
    if (rows * cols == 0) return;
    gauss_fill_kernel<<<(unsigned)std::min<int64_t>(cdiv(rows * cols, 256), 4096), 256, 0, st>>>(out, ld, rows, cols,
                                                                                                    col0, key);
    count_launch();
    SLB_CUDA_CHECK(cudaGetLastError());
  };
  auto sample = [&](int b, const double* X, double* Yo, int64_t cols, bool adjoint) {
    if (cols == 0) return;
    dgemm_batched(st, n, cols, n, 1.0, blocks[b], n, 0, X, n, 0, 0.0, Yo, n, 0, 1, adjoint ? 1 : 0);
  };
  std::vector<int> probe_col(B, 0);  // probe columns drawn so far (the probe stream)

  for (;;) {
    bool any = false;
    for (int b = 0; b < B; b++) any |= active[b] != 0;
    if (!any) break;
    if (rank_feasible(tree, r)) {
      const int64_t s = sample_count(r);
      for (int b = 0; b < B; b++) {
        if (!active[b] || Scur[b] >= s) continue;
        const int64_t add = s - Scur[b];
        if (Scur[b] + add > Smax) throw HbsError("hbs: sample pool overflow", 0.0, false);
        const uint64_t ks = seeds[b];
        fill(OMp(b) + Scur[b] * n, n, n, add, drawn[b], mix_seed_dev(ks, 1));
        fill(PSp(b) + Scur[b] * n, n, n, add, drawn[b], mix_seed_dev(ks, 2));
        drawn[b] += add;
        sample(b, OMp(b) + Scur[b] * n, Yp(b) + Scur[b] * n, add, false);
        sample(b, PSp(b) + Scur[b] * n, Zp(b) + Scur[b] * n, add, true);
        stats[b].products_normal += add;
        stats[b].products_adjoint += add;
        Scur[b] += add;
      }
      // all active blocks share S (they started together and failed the same rounds)
      int64_t S = 0;
      std::vector<int> act;
      for (int b = 0; b < B; b++)
        if (active[b]) {
          S = Scur[b];
          act.push_back(b);
        }
      const int A = (int)act.size();
      Tree t = tree;
      const Layout L = plan_layout(t, (int)r, (int)S);
      DevMem rmem{st, {}};  // this round's arenas (released stream ordered at the end of the round)
      double* persist = rmem.alloc<double>((size_t)A * L.persist);
      double* work = rmem.alloc<double>((size_t)A * L.work);
      double* hats0 = rmem.alloc<double>((size_t)A * L.hats[0]);
      double* hats1 = rmem.alloc<double>((size_t)A * L.hats[1]);
      int* rk = rmem.alloc<int>((size_t)A * 4 * t.nodes.size());
      NodeDesc* dnodes = rmem.alloc<NodeDesc>(t.nodes.size());
      int* dlev = rmem.alloc<int>(t.nodes.size());
      double** dptr = rmem.alloc<double*>((size_t)8 * A);
      int** drk = rmem.alloc<int*>((size_t)A);
      double* dfloor = rmem.alloc<double>((size_t)A);
      SLB_CUDA_CHECK(cudaMemcpyAsync(dnodes, t.nodes.data(), t.nodes.size() * sizeof(NodeDesc), cudaMemcpyHostToDevice, st));
      std::vector<int> lev_flat;
      std::vector<int> lev_off;
      for (auto& lv : t.levels) {
        lev_off.push_back((int)lev_flat.size());
        lev_flat.insert(lev_flat.end(), lv.begin(), lv.end());
      }
      SLB_CUDA_CHECK(cudaMemcpyAsync(dlev, lev_flat.data(), lev_flat.size() * sizeof(int), cudaMemcpyHostToDevice, st));
      // floor tolerance: trunc_rel * max(||Y||, ||Z||) / sqrt(S)  (hbs_compress.hpp:98-101)
      {
        for (int i0 = 0; i0 < A; i0 += NB_NORM) {
          NormArgs na{};
          const int nA = std::min(NB_NORM, A - i0);
          for (int i = 0; i < nA; i++) {
            na.p[i][0] = Yp(act[i0 + i]);
            na.p[i][1] = Zp(act[i0 + i]);
          }
          na.rows = n;
          na.cols[0] = na.cols[1] = S;
          na.ld = n;
          na.out = dnorm + 4 * i0;
          norms_kernel<<<dim3(2, nA), 256, 0, st>>>(na);
          count_launch();
        }
        SLB_CUDA_CHECK(cudaMemcpyAsync(hnorm.data(), dnorm, 4 * (size_t)A * sizeof(double), cudaMemcpyDeviceToHost, st));
        SLB_CUDA_CHECK(cudaStreamSynchronize(st));
        std::vector<double> fl(A);
        for (int i = 0; i < A; i++)
          fl[i] = o.trunc_rel * std::max(std::sqrt(hnorm[4 * i]), std::sqrt(hnorm[4 * i + 1])) /
                  std::sqrt((double)std::max<int64_t>(S, 1));
        SLB_CUDA_CHECK(cudaMemcpyAsync(dfloor, fl.data(), A * sizeof(double), cudaMemcpyHostToDevice, st));
      }
      std::vector<double*> hp(8 * (size_t)A);
      std::vector<int*> hrk(A);
      for (int i = 0; i < A; i++) {
        hp[0 * A + i] = OMp(act[i]);
        hp[1 * A + i] = persist + (size_t)i * L.persist;
        hp[2 * A + i] = work + (size_t)i * L.work;
        hp[3 * A + i] = hats0 + (size_t)i * L.hats[0];
        hp[4 * A + i] = hats1 + (size_t)i * L.hats[1];
        hrk[i] = rk + (size_t)i * 4 * t.nodes.size();
      }
      SLB_CUDA_CHECK(cudaMemcpyAsync(dptr, hp.data(), hp.size() * sizeof(double*), cudaMemcpyHostToDevice, st));
      SLB_CUDA_CHECK(cudaMemcpyAsync(drk, hrk.data(), hrk.size() * sizeof(int*), cudaMemcpyHostToDevice, st));
      // build, bottom up
      for (int lv = (int)t.levels.size() - 1; lv >= 0; lv--) {
        BuildArgs ba{};
        ba.nodes = dnodes;
        ba.level_nodes = dlev + lev_off[lv];
        ba.n = (int)n;
        ba.S = (int)S;
        ba.r = (int)r;
        ba.pools = dptr + 0 * A;
        ba.pool_ld = n;
        ba.pool_stride = pstride;
        ba.persist = dptr + 1 * A;
        ba.work = dptr + 2 * A;
        ba.hats_cur = dptr + ((lv & 1) ? 4 : 3) * A;
        ba.hats_kid = dptr + ((lv & 1) ? 3 : 4) * A;
        ba.rk = drk;
        ba.floor_tol = dfloor;
        hbs_build_level_kernel<<<dim3((unsigned)t.levels[lv].size(), (unsigned)A), HT, kSmemBytes, st>>>(ba);
        count_launch();
        SLB_CUDA_CHECK(cudaGetLastError());
      }
      // apply machinery
      std::vector<int64_t> ox(t.nodes.size());
      int64_t xh_per_col = 0;
      for (size_t k = 0; k < t.nodes.size(); k++) {
        ox[k] = xh_per_col;
        xh_per_col += t.nodes[k].rcap;
      }
      auto apply = [&](int nc, bool adj, const std::vector<const double*>& X, int64_t ldx,
                       const std::vector<double*>& Yo, int64_t ldy, const std::vector<int>& which) {
        // which: indices into act
        const int Aw = (int)which.size();
        if (Aw == 0 || nc == 0) return;
        DevMem amem{st, {}};
        double* xh = amem.alloc<double>((size_t)Aw * xh_per_col * nc);
        double* yh = amem.alloc<double>((size_t)Aw * xh_per_col * nc);
        std::vector<const void*> hv(6 * (size_t)Aw);
        for (int i = 0; i < Aw; i++) {
          hv[0 * Aw + i] = hp[1 * A + which[i]];
          hv[1 * Aw + i] = hrk[which[i]];
          hv[2 * Aw + i] = X[i];
          hv[3 * Aw + i] = Yo[i];
          hv[4 * Aw + i] = xh + (size_t)i * xh_per_col * nc;
          hv[5 * Aw + i] = yh + (size_t)i * xh_per_col * nc;
        }
        void** dv = amem.alloc<void*>(hv.size());
        int64_t* dox_nc = amem.alloc<int64_t>(t.nodes.size());
        std::vector<int64_t> oxn(t.nodes.size());
        for (size_t k = 0; k < t.nodes.size(); k++) oxn[k] = ox[k] * nc;
        SLB_CUDA_CHECK(cudaMemcpyAsync(dv, hv.data(), hv.size() * sizeof(void*), cudaMemcpyHostToDevice, st));
        SLB_CUDA_CHECK(cudaMemcpyAsync(dox_nc, oxn.data(), oxn.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        ApplyArgs aa{};
        aa.nodes = dnodes;
        aa.nc = nc;
        aa.adj = adj ? 1 : 0;
        aa.persist = reinterpret_cast<double* const*>(dv + 0 * Aw);
        aa.rk = reinterpret_cast<int* const*>(dv + 1 * Aw);
        aa.X = reinterpret_cast<const double* const*>(dv + 2 * Aw);
        aa.Yout = reinterpret_cast<double* const*>(dv + 3 * Aw);
        aa.ldx = ldx;
        aa.ldy = ldy;
        aa.xh = reinterpret_cast<double* const*>(dv + 4 * Aw);
        aa.yh = reinterpret_cast<double* const*>(dv + 5 * Aw);
        aa.o_x = dox_nc;
        const unsigned chunks = (unsigned)cdiv(nc, 64);
        for (int lv = (int)t.levels.size() - 1; lv >= 1; lv--) {
          aa.level_nodes = dlev + lev_off[lv];
          hbs_apply_up_kernel<<<dim3((unsigned)t.levels[lv].size(), (unsigned)Aw, chunks), HT, kSmemBytes, st>>>(aa);
          count_launch();
        }
        for (int lv = 0; lv < (int)t.levels.size(); lv++) {
          aa.level_nodes = dlev + lev_off[lv];
          hbs_apply_down_kernel<<<dim3((unsigned)t.levels[lv].size(), (unsigned)Aw, chunks), HT, kSmemBytes, st>>>(aa);
          count_launch();
        }
        SLB_CUDA_CHECK(cudaGetLastError());
      };
      // probe (hbs_compress.hpp:161-183): W, Q fresh from the probe stream
      std::vector<int> all(A);
      std::vector<const double*> Xw(A), Xq(A);
      std::vector<double*> Yw(A), Yq(A);
      for (int i = 0; i < A; i++) {
        const int b = act[i];
        all[i] = i;
        double* pb = probe + (size_t)b * 8 * n;
        double* qb = probe2 + (size_t)b * 16 * n;
        const uint64_t kp = mix_seed_dev(seeds[b], 100);
        fill(pb, n, n, 4, probe_col[b], kp);                 // W
        fill(pb + 4 * n, n, n, 4, probe_col[b] + 4, kp);     // Q
        probe_col[b] += 8;
        sample(b, pb, qb, 4, false);                         // MW
        sample(b, pb + 4 * n, qb + 4 * n, 4, true);          // MQ
        stats[b].products_normal += 4;
        stats[b].products_adjoint += 4;
        Xw[i] = pb;
        Xq[i] = pb + 4 * n;
        Yw[i] = qb + 8 * n;   // HW
        Yq[i] = qb + 12 * n;  // H^T Q
      }
      apply(4, false, Xw, n, Yw, n, all);
      apply(4, true, Xq, n, Yq, n, all);
      for (int i0 = 0; i0 < A; i0 += NB_NORM) {
        NormArgs na{};
        const int nA = std::min(NB_NORM, A - i0);
        for (int i = 0; i < nA; i++) {
          const int b = act[i0 + i];
          double* qb = probe2 + (size_t)b * 16 * n;
          na.p[i][0] = qb;           // ||MW||
          na.p[i][1] = qb + 4 * n;   // ||MQ||
          na.p[i][2] = qb;           // ||MW - HW||
          na.sub[i][2] = qb + 8 * n;
          na.p[i][3] = qb + 4 * n;   // ||MQ - HQ||
          na.sub[i][3] = qb + 12 * n;
        }
        na.rows = n;
        na.cols[0] = na.cols[1] = na.cols[2] = na.cols[3] = 4;
        na.ld = n;
        na.out = dnorm + 4 * i0;
        norms_kernel<<<dim3(4, nA), 256, 0, st>>>(na);
        count_launch();
      }
      SLB_CUDA_CHECK(cudaMemcpyAsync(hnorm.data(), dnorm, 4 * (size_t)A * sizeof(double), cudaMemcpyDeviceToHost, st));
      std::vector<int> hrk_all((size_t)A * 4 * t.nodes.size());
      SLB_CUDA_CHECK(cudaMemcpyAsync(hrk_all.data(), rk, hrk_all.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
      SLB_CUDA_CHECK(cudaStreamSynchronize(st));
      std::vector<int> pass_idx;
      for (int i = 0; i < A; i++) {
        const int b = act[i];
        const double nn = std::sqrt(hnorm[4 * i]), na_ = std::sqrt(hnorm[4 * i + 1]);
        const double dn = std::sqrt(hnorm[4 * i + 2]), da = std::sqrt(hnorm[4 * i + 3]);
        const double rel = std::max(nn > 0 ? dn / nn : dn, na_ > 0 ? da / na_ : da);
        stats[b].rounds++;
        stats[b].residual = rel;
        int64_t fr = 0;
        for (size_t k = 0; k < t.nodes.size(); k++)
          fr = std::max<int64_t>(fr, std::max(hrk_all[(size_t)i * 4 * t.nodes.size() + 4 * k + 2],
                                              hrk_all[(size_t)i * 4 * t.nodes.size() + 4 * k + 3]));
        stats[b].final_rank = fr;
        if (rel <= o.tol) {
          pass_idx.push_back(i);
        } else if (!o.fixed_rank) {
          // failed probes are samples: fold them into the pool (hbs_compress.hpp:299-304)
          double* pb = probe + (size_t)b * 8 * n;
          double* qb = probe2 + (size_t)b * 16 * n;
          if (Scur[b] + 4 > Smax) throw HbsError("hbs: sample pool overflow", rel, false);
          SLB_CUDA_CHECK(cudaMemcpyAsync(OMp(b) + Scur[b] * n, pb, 4 * n * sizeof(double), cudaMemcpyDeviceToDevice, st));
          SLB_CUDA_CHECK(cudaMemcpyAsync(Yp(b) + Scur[b] * n, qb, 4 * n * sizeof(double), cudaMemcpyDeviceToDevice, st));
          SLB_CUDA_CHECK(cudaMemcpyAsync(PSp(b) + Scur[b] * n, pb + 4 * n, 4 * n * sizeof(double), cudaMemcpyDeviceToDevice, st));
          SLB_CUDA_CHECK(cudaMemcpyAsync(Zp(b) + Scur[b] * n, qb + 4 * n, 4 * n * sizeof(double), cudaMemcpyDeviceToDevice, st));
          Scur[b] += 4;
        }
      }
      // densify the passed blocks (to_dense as H applied to the identity), one at a time
      if (!pass_idx.empty()) {
        double* I = rmem.alloc<double>((size_t)n * n);
        set_identity_kernel<<<(unsigned)std::min<int64_t>(cdiv(n * n, 256), 8192), 256, 0, st>>>(I, n);
        count_launch();
        for (int i : pass_idx) {
          apply((int)n, false, {I}, n, {blocks[act[i]]}, n, {i});
          passed[act[i]] = 1;
          active[act[i]] = 0;
        }
      }
      if (o.fixed_rank) {
        for (int b = 0; b < B; b++)
          if (active[b])
            throw HbsError("hbs_compress: probe residual exceeds tolerance (rank bound too small)", stats[b].residual,
                           false, b);
        break;
      }
      // round arenas are released with the DevMem at the end (stream ordered)
    }
    bool left = false;
    for (int b = 0; b < B; b++) left |= active[b] != 0;
    if (!left) break;
    if (r >= o.r_max) {
      for (int b = 0; b < B; b++)
        if (active[b])
          throw HbsError("hbs_compress_adaptive: rank ceiling reached without passing the probe",
                         stats[b].rounds ? stats[b].residual : INFINITY, false, b);
    }
    r = std::min<int64_t>(2 * r, o.r_max);
  }
  SLB_CUDA_CHECK(cudaStreamSynchronize(st));
}

}  // namespace slb
