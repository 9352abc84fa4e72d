// Batched FP64 GEMM on the DMMA pipe (sm_100a):
//   C[b] = alpha * A[b] * B[b] + beta * C[b]     (column major, strided batch)
// A may be stored transposed (transA: element (m, k) at A[m * lda + k]),
// which is how the band-LU chain keeps its row-major L factors.
//
// Tiling: 128x128x16 CTA tile, 8 warps each owning 64x32 (8x4 m8n8 DMMA
// tiles), 3-stage cp.async pipeline, padded smem (stride = 4 mod 16 doubles).
#include "common.cuh"
#include "kernels.h"

namespace slb {
namespace {

constexpr int BK = 16, STAGES = 3;
constexpr int SB = BK + 4;  // sB[n][k]
template <int BM, int BN>
constexpr int smem_doubles() { return STAGES * (BK * (BM + 4) + BN * SB); }

struct GemmArgs {
  int64_t M, N, K;
  double alpha, beta;
  const double* A;
  int64_t lda, sA;
  const double* B;
  int64_t ldb, sB;
  double* C;
  int64_t ldc, sC;
  int transA;
};

// BM x BN CTA tile, WM x WN warps, each warp (BM/WM) x (BN/WN).
template <int BM, int BN, int WM, int WN>
__global__ void __launch_bounds__(WM * WN * 32) dgemm_kernel(GemmArgs p) {
  constexpr int THREADS = WM * WN * 32;
  constexpr int SA = BM + 4;  // sA[k][m]
  constexpr int MI = BM / WM / 8, NJ = BN / WN / 8;
  extern __shared__ double smem[];
  double* sA = smem;
  double* sB = smem + STAGES * BK * SA;
  const int64_t bz = blockIdx.z;
  const double* A = p.A + bz * p.sA;
  const double* B = p.B + bz * p.sB;
  double* C = p.C + bz * p.sC;
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % WM, wn = warp / WM;

  auto load_stage = [&](int stage, int64_t k0) {
    double* a = sA + stage * BK * SA;
    double* b = sB + stage * BN * SB;
    if (!p.transA) {
#pragma unroll
      for (int r = 0; r < (BM * BK) / THREADS; r++) {
        const int idx = tid + r * THREADS;
        const int k = idx / BM, m = idx % BM;
        const int64_t gm = m0 + m, gk = k0 + k;
        const bool ok = gm < p.M && gk < p.K;
        cp_async8(a + k * SA + m, ok ? A + gk * p.lda + gm : A, ok);
      }
    } else {
#pragma unroll
      for (int r = 0; r < (BM * BK) / THREADS; r++) {
        const int idx = tid + r * THREADS;
        const int m = idx / BK, k = idx % BK;
        const int64_t gm = m0 + m, gk = k0 + k;
        const bool ok = gm < p.M && gk < p.K;
        cp_async8(a + k * SA + m, ok ? A + gm * p.lda + gk : A, ok);
      }
    }
#pragma unroll
    for (int r = 0; r < (BN * BK) / THREADS; r++) {
      const int idx = tid + r * THREADS;
      const int n = idx / BK, k = idx % BK;
      const int64_t gn = n0 + n, gk = k0 + k;
      const bool ok = gn < p.N && gk < p.K;
      cp_async8(b + n * SB + k, ok ? B + gn * p.ldb + gk : B, ok);
    }
  };

  double acc[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; i++)
#pragma unroll
    for (int j = 0; j < NJ; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int64_t nk = cdiv(p.K, BK);
#pragma unroll
  for (int s = 0; s < STAGES - 1; s++) {
    if (s < nk) load_stage(s, s * BK);
    cp_async_commit();
  }
  for (int64_t kt = 0; kt < nk; kt++) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int64_t nxt = kt + STAGES - 1;
    if (nxt < nk) load_stage(nxt % STAGES, nxt * BK);
    cp_async_commit();
    const double* a = sA + (kt % STAGES) * BK * SA + wm * (MI * 8) + g;
    const double* b = sB + (kt % STAGES) * BN * SB + (wn * (NJ * 8) + g) * SB + t;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[MI], bf[NJ];
#pragma unroll
      for (int i = 0; i < MI; i++) af[i] = a[(kk + t) * SA + i * 8];
#pragma unroll
      for (int j = 0; j < NJ; j++) bf[j] = b[j * 8 * SB + kk];
#pragma unroll
      for (int i = 0; i < MI; i++)
#pragma unroll
        for (int j = 0; j < NJ; j++) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

#pragma unroll
  for (int i = 0; i < MI; i++) {
    const int64_t row = m0 + wm * (MI * 8) + i * 8 + g;
    if (row >= p.M) continue;
#pragma unroll
    for (int j = 0; j < NJ; j++)
#pragma unroll
      for (int e = 0; e < 2; e++) {
        const int64_t col = n0 + wn * (NJ * 8) + j * 8 + 2 * t + e;
        if (col >= p.N) continue;
        double* c = C + col * p.ldc + row;
        const double v = p.alpha * acc[i][j][e];
        *c = p.beta == 0.0 ? v : v + p.beta * *c;
      }
  }
}

}  // namespace

void dgemm_batched(cudaStream_t st, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                   int64_t lda, int64_t sA, const double* B, int64_t ldb, int64_t sB, double beta,
                   double* C, int64_t ldc, int64_t sC, int64_t batch, bool transA) {
  if (M <= 0 || N <= 0 || batch <= 0) return;
  static bool attr = false;
  const size_t smem_big = smem_doubles<128, 128>() * sizeof(double);
  const size_t smem_small = smem_doubles<64, 64>() * sizeof(double);
  if (!attr) {
    SLB_CUDA_CHECK(cudaFuncSetAttribute(dgemm_kernel<128, 128, 2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_big));
    SLB_CUDA_CHECK(cudaFuncSetAttribute(dgemm_kernel<64, 64, 2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_small));
    attr = true;
  }
  if (K <= 0) {  // C = beta * C
    dscale_batched(st, M, N, beta, C, ldc, sC, batch);
    return;
  }
  // small tiles when the big-tile grid would not fill the GPU twice, or when big tiles would
  // mostly compute padding (e.g. the 152 x 152 level blocks of the conversion)
  const double pad_big = (double)round_up(M, 128) * round_up(N, 128), pad_small = (double)round_up(M, 64) * round_up(N, 64);
  const bool small = cdiv(M, 128) * cdiv(N, 128) * batch < 296 || pad_big > 1.3 * pad_small;
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
    const int64_t nb = std::min<int64_t>(65535, batch - b0);
    GemmArgs p{M, N, K, alpha, beta, A + b0 * sA, lda, sA, B + b0 * sB, ldb, sB, C + b0 * sC, ldc, sC,
               transA ? 1 : 0};
    if (small) {
      dim3 grid((unsigned)cdiv(M, 64), (unsigned)cdiv(N, 64), (unsigned)nb);
      dgemm_kernel<64, 64, 2, 2><<<grid, 128, smem_small, st>>>(p); count_launch();
    } else {
      dim3 grid((unsigned)cdiv(M, 128), (unsigned)cdiv(N, 128), (unsigned)nb);
      dgemm_kernel<128, 128, 2, 4><<<grid, 256, smem_big, st>>>(p); count_launch();
    }
    SLB_CUDA_CHECK(cudaGetLastError());
  }
}

namespace {
__global__ void dscale_kernel(int64_t M, int64_t N, double beta, double* C, int64_t ldc, int64_t sC) {
  double* c = C + blockIdx.z * sC;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < M * N;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % M, j = idx / M;
    c[j * ldc + i] = beta == 0.0 ? 0.0 : beta * c[j * ldc + i];
  }
}
}  // namespace

void dscale_batched(cudaStream_t st, int64_t M, int64_t N, double beta, double* C, int64_t ldc,
                    int64_t sC, int64_t batch) {
  if (M <= 0 || N <= 0 || batch <= 0 || beta == 1.0) return;
  const int64_t blocks = std::min<int64_t>(cdiv(M * N, 256), 4096);
  dscale_kernel<<<dim3((unsigned)blocks, 1, (unsigned)batch), 256, 0, st>>>(M, N, beta, C, ldc, sC); count_launch();
  SLB_CUDA_CHECK(cudaGetLastError());
}

}  // namespace slb
