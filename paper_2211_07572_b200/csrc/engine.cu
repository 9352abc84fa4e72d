// Engine orchestration and the C ABI (include/slablu_gpu.h).
//
// factorize (proj/include/slablu/driver.hpp:115-167):
//   stage one  = coupling/level extraction from the CSR, the level-by-level
//                block band LU of every slab (band_lu.cu, all slabs batched),
//                the Schur sweep (schur.cu) and T assembly;
//   stage two  = sweeping block LU of the reduced block tridiagonal system
//                (stage_two.hpp:131-150) with dense LU on the device
//                (dense.cu); each S_j is kept in LU form (DenseLU,
//                dense.hpp:31-61) and applied by the chained getrs.
// solve (driver.hpp:171-179): reduce_rhs -> sweep solve -> recover_interiors,
// all on the device.
#include <algorithm>
#include <array>
#include <memory>
#include <atomic>
#include <chrono>
#include <climits>
#include <cstring>
#include <map>
#include <cstdlib>
#include <fstream>
#include <mutex>
#include <vector>

#include <cuda.h>  // driver types for the green-context partition (entry points resolved at run time)

#include "common.cuh"
#include "host.h"
#include "kernels.h"

namespace slb {
std::atomic<long long> g_kernel_count{0};



namespace {

// ---------------------------------------------------------------------------
// Exact-size caching device allocator (repeated factorizations of the same
// problem reuse their buffers instead of paying cudaMalloc/cudaFree).
//
// Reuse is stream-ordered: a block released while the thread is inside a StreamScope records
// an event on that stream.  The same stream may take the block back at once (its later work is
// ordered after the earlier user's); any other stream takes it only once the event has
// completed.  Blocks released outside a scope (after a synchronize) carry no event.
thread_local cudaStream_t t_scope_stream = nullptr;
struct StreamScope {
  cudaStream_t prev;
  explicit StreamScope(cudaStream_t s) : prev(t_scope_stream) { t_scope_stream = s; }
  ~StreamScope() { t_scope_stream = prev; }
};
// Sets the current device for the lifetime of the guard and restores the caller's.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) {
      cudaGetLastError();
      prev = -1;
    }
    if (prev != dev) SLB_CUDA_CHECK(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

struct DevPool {
  struct Block {
    void* p;
    cudaStream_t stream;  // stream of the last user (nullptr: no pending work)
    cudaEvent_t ev;       // completes when that work is done (nullptr: nothing pending)
  };
  std::mutex mu;
  std::multimap<std::pair<int, size_t>, Block> free_blocks;
  size_t cached_bytes(int dev) {
    std::lock_guard<std::mutex> g(mu);
    size_t s = 0;
    for (auto& kv : free_blocks)
      if (kv.first.first == dev) s += kv.first.second;
    return s;
  }
  void* get(int dev, size_t bytes) {
    if (bytes == 0) return nullptr;
    DeviceGuard dg(dev);
    {
      std::lock_guard<std::mutex> g(mu);
      auto range = free_blocks.equal_range({dev, bytes});
      auto pick = free_blocks.end();
      for (auto it = range.first; it != range.second; ++it) {
        const Block& b = it->second;
        if (!b.ev || (t_scope_stream && b.stream == t_scope_stream)) {
          pick = it;
          break;
        }
        const cudaError_t q = cudaEventQuery(b.ev);
        if (q == cudaSuccess) {
          pick = it;
          break;
        }
        if (q != cudaErrorNotReady) cudaGetLastError();
      }
      if (pick != free_blocks.end()) {
        void* p = pick->second.p;
        if (pick->second.ev) cudaEventDestroy(pick->second.ev);
        free_blocks.erase(pick);
        return p;
      }
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      trim(dev);
      e = cudaMalloc(&p, bytes);
      if (e != cudaSuccess) {
        cudaGetLastError();
        throw HostError(SLABLU_ERR_OOM, "device memory exhausted (" + std::to_string(bytes >> 20) + " MiB)");
      }
    }
    return p;
  }
  void put(int dev, size_t bytes, void* p) {
    if (!p) return;
    Block b{p, nullptr, nullptr};
    if (t_scope_stream) {
      DeviceGuard dg(dev);
      if (cudaEventCreateWithFlags(&b.ev, cudaEventDisableTiming) == cudaSuccess &&
          cudaEventRecord(b.ev, t_scope_stream) == cudaSuccess) {
        b.stream = t_scope_stream;
      } else {
        cudaGetLastError();
        if (b.ev) cudaEventDestroy(b.ev);
        b.ev = nullptr;
        cudaStreamSynchronize(t_scope_stream);  // cannot order the reuse: wait for the user
        cudaGetLastError();
      }
    }
    std::lock_guard<std::mutex> g(mu);
    free_blocks.insert({{dev, bytes}, b});
  }
  // Frees every cached block of dev (waiting for pending users first).
  void trim(int dev) {
    DeviceGuard dg(dev);
    std::lock_guard<std::mutex> g(mu);
    for (auto it = free_blocks.begin(); it != free_blocks.end();) {
      if (it->first.first == dev) {
        if (it->second.ev) {
          cudaEventSynchronize(it->second.ev);
          cudaEventDestroy(it->second.ev);
        }
        cudaFree(it->second.p);
        it = free_blocks.erase(it);
      } else {
        ++it;
      }
    }
    cudaGetLastError();
  }
};
DevPool& pool() {
  static DevPool* p = new DevPool;  // never destroyed (process exit frees device memory)
  return *p;
}

template <class T>
struct DBuf {
  int dev = 0;
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  void alloc(int d, size_t count) {
    release();
    dev = d;
    n = count;
    p = static_cast<T*>(pool().get(d, count * sizeof(T)));
  }
  void release() {
    if (p) pool().put(dev, n * sizeof(T), p);
    p = nullptr;
    n = 0;
  }
  size_t bytes() const { return n * sizeof(T); }
  ~DBuf() { release(); }
};

// ---------------------------------------------------------------------------
// f on the interfaces j in [jlo, jhi) (zero elsewhere: a shard owns only those)
__global__ void gather_ifc_kernel(const double* f, int64_t ldf, int64_t nrhs, int nifc, const int64_t* off,
                                  int64_t n2, double* out, int64_t K, int jlo, int jhi) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= K * nrhs) return;
  const int64_t c = idx / K, r = idx % K, j = r / n2, q = r % n2;
  out[idx] = (j >= jlo && j < jhi) ? f[c * ldf + off[j] + q] : 0.0;
}
__global__ void scatter_ifc_kernel(const double* u_ifc, int64_t K, int64_t nrhs, const int64_t* off, int64_t n2,
                                   double* u, int64_t ldu, int jlo, int jhi) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= K * nrhs) return;
  const int64_t c = idx / K, r = idx % K, j = r / n2, q = r % n2;
  if (j >= jlo && j < jhi) u[c * ldu + off[j] + q] = u_ifc[idx];
}
// red_j = (f_j - contrib[strip j][R]) - contrib[strip j+1][L]  (stage_one.hpp:423-432 order);
// strips are the shard's, global strip g at local index g - sbase
__global__ void combine_reduce_kernel(double* red, int64_t K, int64_t nrhs, int64_t n2, int nstrips,
                                      const StripDesc* strips, const double* contrib, int sbase) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= K * nrhs) return;
  const int64_t c = idx / K, r = idx % K, j = r / n2, q = r % n2;
  double v = red[idx];
  const int64_t a = j - sbase, b = j + 1 - sbase;  // local strips left / right of interface j
  if (a >= 0 && a < nstrips && strips[a].right == j) v -= contrib[((int64_t)(a * 2 + 1) * nrhs + c) * n2 + q];
  if (b >= 0 && b < nstrips && strips[b].left == j) v -= contrib[((int64_t)(b * 2 + 0) * nrhs + c) * n2 + q];
  red[idx] = v;
}
// y[:, c] += x[:, c] for an n x nrhs block (lds, ldd)
__global__ void add2d_kernel(const double* x, int64_t ldx, double* y, int64_t ldy, int64_t rows, int64_t cols,
                             double alpha) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < rows * cols;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx % rows, c = idx / rows;
    y[c * ldy + r] += alpha * x[c * ldx + r];
  }
}
// r = f - A u (CSR, one thread per row and column), then u stays; used for refinement.
__global__ void residual_kernel(const int32_t* rp, const int32_t* ci, const double* v, int64_t n, int64_t nrhs,
                                const double* f, const double* u, double* r) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * nrhs) return;
  const int64_t row = idx % n, c = idx / n;
  const double* uc = u + c * n;
  double acc = 0.0;
  for (int32_t p = rp[row]; p < rp[row + 1]; p++) acc = fma(v[p], uc[ci[p]], acc);
  r[idx] = f[idx] - acc;
}
__global__ void axpy_kernel(int64_t count, const double* x, double* y) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < count) y[idx] += x[idx];
}
__global__ void copy2d_kernel(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows, int64_t cols) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < rows * cols;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx % rows, c = idx / rows;
    dst[c * ldd + r] = src[c * lds + r];
  }
}

void add2d(cudaStream_t st, const double* x, int64_t ldx, double* y, int64_t ldy, int64_t rows, int64_t cols,
           double alpha = 1.0) {
  if (rows <= 0 || cols <= 0) return;
  add2d_kernel<<<(unsigned)std::min<int64_t>(cdiv(rows * cols, 256), 8192), 256, 0, st>>>(x, ldx, y, ldy, rows, cols,
                                                                                     alpha); count_launch();
  SLB_CUDA_CHECK(cudaGetLastError());
}

void copy2d(cudaStream_t st, const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows, int64_t cols) {
  if (rows <= 0 || cols <= 0) return;
  copy2d_kernel<<<(unsigned)std::min<int64_t>(cdiv(rows * cols, 256), 8192), 256, 0, st>>>(src, lds, dst, ldd, rows, cols); count_launch();
  SLB_CUDA_CHECK(cudaGetLastError());
}

// A stream confined to a green context of `conv_sms` SMs (driver API, resolved through
// cudaGetDriverEntryPoint so the library carries no libcuda link dependency).  The band-LU
// chain is latency-bound on one CTA per strip; the LU -> GEMM-form conversion that runs
// beside it is throughput work.  Confining the conversion to a partition leaves the chain
// SMs that are always free, instead of making its CTAs wait for SMs the conversion holds.
// Returns nullptr when green contexts are unavailable (caller falls back to a priority stream).
cudaStream_t green_partition_stream(int dev, int conv_sms) {
  static std::mutex mu;
  static std::map<int, cudaStream_t> made;
  std::lock_guard<std::mutex> lk(mu);
  auto it = made.find(dev);
  if (it != made.end()) return it->second;
  made[dev] = nullptr;
  if (getenv("SLB_NO_GREEN")) return nullptr;
  // under a profiler (ncu/nsys inject through these variables) a green context ends the
  // profiled process; the priority-stream fallback runs the same kernels
  if (getenv("CUDA_INJECTION64_PATH") || getenv("NV_COMPUTE_PROFILER_PERFWORKS_DIR") ||
      getenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE"))
    return nullptr;
  using FnDeviceGet = CUresult (*)(CUdevice*, int);
  using FnGetRes = CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType);
  using FnSplit = CUresult (*)(CUdevResource*, unsigned int*, const CUdevResource*, CUdevResource*, unsigned int,
                               unsigned int);
  using FnDesc = CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned int);
  using FnGreen = CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned int);
  using FnStream = CUresult (*)(CUstream*, CUgreenCtx, unsigned int, int);
  FnDeviceGet deviceGet = nullptr;
  FnGetRes getRes = nullptr;
  FnSplit split = nullptr;
  FnDesc genDesc = nullptr;
  FnGreen greenCreate = nullptr;
  FnStream streamCreate = nullptr;
  auto get = [](const char* name, void** fn) {
    cudaDriverEntryPointQueryResult q;
    return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
           q == cudaDriverEntryPointSuccess && *fn;
  };
  if (!get("cuDeviceGet", (void**)&deviceGet) || !get("cuDeviceGetDevResource", (void**)&getRes) ||
      !get("cuDevSmResourceSplitByCount", (void**)&split) || !get("cuDevResourceGenerateDesc", (void**)&genDesc) ||
      !get("cuGreenCtxCreate", (void**)&greenCreate) || !get("cuGreenCtxStreamCreate", (void**)&streamCreate)) {
    cudaGetLastError();
    return nullptr;
  }
  CUdevice cu;
  CUdevResource all, part, rest;
  unsigned int ngroups = 1;
  CUdevResourceDesc desc;
  CUgreenCtx g;
  CUstream cs;
  if (deviceGet(&cu, dev) != CUDA_SUCCESS || getRes(cu, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) return nullptr;
  if (conv_sms <= 0 || (unsigned)conv_sms >= all.sm.smCount) return nullptr;
  if (split(&part, &ngroups, &all, &rest, 0, (unsigned)conv_sms) != CUDA_SUCCESS || ngroups != 1) return nullptr;
  if ((int)part.sm.smCount > conv_sms + 8) return nullptr;  // partition granularity ate the chain's SMs
  if (genDesc(&desc, &part, 1) != CUDA_SUCCESS) return nullptr;
  if (greenCreate(&g, desc, cu, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) return nullptr;
  if (streamCreate(&cs, g, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS) return nullptr;
  made[dev] = (cudaStream_t)cs;
  if (getenv("SLB_GREEN_VERBOSE"))
    fprintf(stderr, "[slablu] conversion partition: %u of %u SMs\n", part.sm.smCount, all.sm.smCount);
  return made[dev];
}

constexpr int64_t kMaxIfc = 8192;  // stage-two block dimension limit (dgetrf panel cluster: 16 CTAs x 256 threads x 2 rows, dense.cu)

int sm_count(int dev) {
  int v = 0;
  SLB_CUDA_CHECK(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
  return v;
}

}  // namespace


}  // namespace slb

using namespace slb;

struct slablu_gpu_fact {
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t n1 = 0, n2 = 0, N = 0, b = 0;
  bool single = false;
  int S = 0, K = 0, Wp = 0;
  // multi-GPU shard (nranks > 1): global strips [s0, s1) are local (F->S of them, local index
  // s - s0), interfaces [j0, j1) are owned; K and every interface-indexed array stay global
  int rank = 0, nranks = 1, Sg = 0, s0 = 0, s1 = 0, j0 = 0, j1 = 0;
  bool sharded = false, swept = false;
  bool stage2_only = false;  // slablu_gpu_sweep_build: a block-tridiagonal system only
  // partitioned stage two (SPIKE-style): the rank's interior chain [ia, ib) and the
  // spike ends on its separators: sh_a = super_{j0} (A_I^{-1} E_L)_first, sh_b = super_{j0}
  // (A_I^{-1} E_R)_first, sh_c = sub_{ib-1} (A_I^{-1} E_L)_last, sh_d = sub_{ib-1} (A_I^{-1} E_R)_last,
  // sh_yl = (A_I^{-1} E_L)_last, sh_xhat = S^_r^{-1} sh_b (all n2 x n2)
  int ia = 0, ib = 0;
  bool has_left = false, has_right = false, eliminated = false;
  DBuf<double> sh_a, sh_b, sh_c, sh_d, sh_yl, sh_xhat;
  // shard solve state between its phases
  DBuf<double> sh_f, sh_red, sh_red0, sh_uifc, sh_v;
  int64_t sh_nrhs = 0;
  int sh_phase = 0;  // 0 idle, 1 local done, 2 forward done
  std::vector<StripDesc> strips_h;
  std::vector<int64_t> ifc_off_h;
  std::vector<int32_t> sym_h;
  DBuf<StripDesc> strips;
  DBuf<int64_t> ifc_off;
  DBuf<double> fac;
  DBuf<int32_t> perm;
  DBuf<double> cpl;
  DBuf<int32_t> sym;
  DBuf<uint8_t> u13;
  DBuf<uint8_t> lnd;    // Lsub off-diagonal flags per (strip, level)
  DBuf<double> dsub;    // diag(Lsub_{l+1}) per (strip, level)
  DBuf<double> exc;     // exceptional Fbot rows per (strip, level): 8 x Wp
  DBuf<int32_t> excpos; // their positions: 8 per (strip, level)
  DBuf<double> hcol;    // x_{l+2} columns of H per (strip, level): 8 x Wp
  DBuf<int32_t> hidx;   // their column indices
  DBuf<double> T;       // [diag k | super k-1 | sub k-1] blocks, n2 x n2; diag holds LU(S_j) (ipivT)
  DBuf<int32_t> ipivT;  // pivots of LU(S_j), n2 per interface
  DBuf<int32_t> permT;  // the same interchanges as a row permutation (getrs_chain)
  DBuf<double> dinvT;   // inverses of the 64x64 diagonal blocks of L_j, U_j (getrs_chain)
  DBuf<double> Xup;     // block upper factor X_j = S_j^{-1} super_j (n2 x n2 per interface j < K-1)
  DBuf<double> Tkeep;   // optional copy of the reduced blocks
  DBuf<DevStatus> status;
  DBuf<DevStatus> sstatus;   // solve-time status (getrs_chain timeouts)
  DBuf<int32_t> a_rp, a_ci;  // the original operator (iterative refinement)
  DBuf<double> a_v;
  int refine = 0;
  int64_t sF = 0, sP = 0, sCPL = 0;
  double t1 = 0, t2 = 0, t_chain = 0, t_schur = 0, t_asm = 0, t_hbs = 0;
  int compression = 1;       // resolved: 1 dense, 2 hbs (driver.hpp:125-130)
  int64_t hbs_max_rank = 0;
  mutable double t_solve = 0, t_solve_strips = 0;
  int64_t storage1 = 0, storage2 = 0;
  int64_t launches_factor = 0;
  mutable int64_t launches_solve = 0;
  mutable std::mutex solve_mu;
  double* Tdiag() const { return T.p; }
  double* Tsup() const { return T.p + (size_t)K * n2 * n2; }
  double* Tsub() const { return T.p + (size_t)(2 * K - 1) * n2 * n2; }
  cudaStream_t stream2 = nullptr;  // stage two: the right half of X_j / S_{j+1} beside the LU
  ~slablu_gpu_fact() {
    if (stream || stream2) cudaSetDevice(device);
    if (stream2) {
      cudaStreamSynchronize(stream2);
      cudaStreamDestroy(stream2);
    }
    if (stream) {
      cudaStreamSynchronize(stream);
      cudaStreamDestroy(stream);
    }
  }
};

namespace {

void throw_status(const DevStatus& st) {
  if (st.flags & ERR_OUT_OF_BAND) throw HostError(SLABLU_ERR_GENERIC, "BandedMatrix::at: index outside band");
  if (st.flags & ERR_PAST_INTERFACE)
    throw HostError(SLABLU_ERR_GENERIC, "factor_one_interior: interior couples past its adjacent interfaces");
  if (st.flags & ERR_COUPLING_LEVEL)
    throw HostError(SLABLU_ERR_UNSUPPORTED, "interior/interface coupling outside the five-point level structure");
  if (st.flags & ERR_IFC_STRUCTURE)
    throw HostError(SLABLU_ERR_UNSUPPORTED, "interface row couples outside its adjacent strips/interfaces");
}

int64_t cfg_device(const slablu_gpu_config* c) { return c ? c->device : 0; }

// Factorize with the CSR already on the device.
// Contiguous strip split for rank r of G and the interfaces it owns (those whose right strip
// is local; the last rank also owns a trailing interface).  Shared by the engine and
// slablu_gpu_shard_plan so that hosts and engine agree.
void shard_ranges(int Sg, int K, int rank, int nranks, int* s0, int* s1, int* j0, int* j1) {
  *s0 = (int)((int64_t)rank * Sg / nranks);
  *s1 = (int)((int64_t)(rank + 1) * Sg / nranks);
  *j0 = rank == 0 ? 0 : *s0 - 1;
  *j1 = rank == nranks - 1 ? K : *s1 - 1;
}

// Stage two (stage_two.hpp:131-150) on F->T: S_0 = T_00, S_j = T_jj - sub_{j-1} S_{j-1}^{-1} super_{j-1}.
// S_j stays in LU form (as DenseLU in the reference): X = S_{j-1}^{-1} super_{j-1} by getrs, the
// solve applies S_j^{-1} by the chained getrs (stage_two.hpp:138-147, 176-186).  Singular S_j raise
// ERR_SINGULAR with the block index in F->status (checked by the caller).
void stage_two_alloc(slablu_gpu_fact* F) {
  const int dev = F->device, K = F->K;
  const int64_t n2 = F->n2, bs = n2 * n2;
  const int64_t dinv_sz = cdiv(n2, 64) * 2 * 64 * 64;
  F->ipivT.alloc(dev, (size_t)std::max(K, 1) * n2);
  F->permT.alloc(dev, (size_t)std::max(K, 1) * n2);
  F->dinvT.alloc(dev, (size_t)std::max(K, 1) * dinv_sz);
  // The block LU T = L~ U~ keeps, besides LU(S_j), U~'s off-diagonal blocks X_j = S_j^{-1} super_j:
  // the recurrence computes them anyway (stage_two.hpp:138-140), and the backward sweep of the
  // solve is then u_j -= X_j u_{j+1}, one GEMV instead of a GEMV plus a triangular-solve chain.
  F->Xup.alloc(dev, (size_t)std::max(K - 1, 1) * bs);
}

// LU form of S_j in place (Tdiag[j]) plus the chained-getrs data of the solve
void factor_S(slablu_gpu_fact* F, int j) {
  const int64_t n2 = F->n2, bs = n2 * n2, dinv_sz = cdiv(n2, 64) * 2 * 64 * 64;
  double* Sj = F->Tdiag() + j * bs;
  dgetrf(F->stream, n2, Sj, F->ipivT.p + (size_t)j * n2, nullptr, F->status.p, j);
  getrs_prepare(F->stream, n2, Sj, F->ipivT.p + (size_t)j * n2, F->permT.p + (size_t)j * n2,
                F->dinvT.p + (size_t)j * dinv_sz);
}

// The sweep over the interfaces [ia, ib) started fresh at ia: S_ia = T_{ia ia},
// X_{j-1} = S_{j-1}^{-1} super_{j-1}, S_j = T_jj - sub_{j-1} X_{j-1}.
//
// Overlap: the LU of S_j factors its left part (columns [0, h), h = n2 / 5) first; the right part
// of X_{j-1} and of S_j (getrs + GEMM on columns [h, n2)) is computed meanwhile on a second
// stream, and the LU waits for it only when it reaches those columns (dgetrf_split).  SLB_STAGE2_SERIAL=1 disables it.
void stage_two_range(slablu_gpu_fact* F, int ia, int ib) {
  cudaStream_t st = F->stream;
  const int64_t n2 = F->n2, bs = n2 * n2, dinv_sz = cdiv(n2, 64) * 2 * 64 * 64;
  static const bool serial = getenv("SLB_STAGE2_SERIAL") != nullptr;
  const bool overlap = !serial && n2 >= 512;
  cudaEvent_t ev_in = nullptr, ev_right = nullptr;
  if (overlap) {
    if (!F->stream2) {
      int least = 0, greatest = 0;
      SLB_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
      SLB_CUDA_CHECK(cudaStreamCreateWithPriority(&F->stream2, cudaStreamNonBlocking, least));
    }
    SLB_CUDA_CHECK(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
    SLB_CUDA_CHECK(cudaEventCreateWithFlags(&ev_right, cudaEventDisableTiming));
  }
  // split column of the overlap (SLB_S2_SPLIT: fraction of n2).  A narrow left part starts the
  // LU early and leaves most of the getrs / GEMM to run beside it: cfg3 stage two 0.679 s at
  // 0.5, 0.671 at 0.3, 0.650 at 0.2, 0.658 at 0.16, 0.678 at 0.1
  static const double split = [] {
    const char* e = getenv("SLB_S2_SPLIT");
    const double v = e ? atof(e) : 0.2;
    return v > 0.05 && v < 0.95 ? v : 0.2;
  }();
  const int64_t h = std::min(n2, round_up((int64_t)(split * (double)n2), 64));
  for (int j = ia; j < ib; j++) {
    if (j > ia) {
      double* X = F->Xup.p + (size_t)(j - 1) * bs;
      const double* LUp = F->Tdiag() + (j - 1) * bs;
      const int32_t* ip = F->ipivT.p + (size_t)(j - 1) * n2;
      double* Sj = F->Tdiag() + j * bs;
      const double* sub = F->Tsub() + (j - 1) * bs;
      SLB_CUDA_CHECK(cudaMemcpyAsync(X, F->Tsup() + (j - 1) * bs, bs * sizeof(double), cudaMemcpyDeviceToDevice, st));
      if (overlap) {
        SLB_CUDA_CHECK(cudaEventRecord(ev_in, st));
        SLB_CUDA_CHECK(cudaStreamWaitEvent(F->stream2, ev_in, 0));
        {
          StreamScope s2(F->stream2);
          dgetrs(F->stream2, n2, n2 - h, LUp, ip, X + h * n2, n2, nullptr);
          dgemm_batched(F->stream2, n2, n2 - h, n2, -1.0, sub, n2, 0, X + h * n2, n2, 0, 1.0, Sj + h * n2, n2, 0, 1);
        }
        SLB_CUDA_CHECK(cudaEventRecord(ev_right, F->stream2));
        dgetrs(st, n2, h, LUp, ip, X, n2, nullptr);
        dgemm_batched(st, n2, h, n2, -1.0, sub, n2, 0, X, n2, 0, 1.0, Sj, n2, 0, 1);
        dgetrf_split(st, n2, Sj, F->ipivT.p + (size_t)j * n2, F->status.p, j, h, ev_right);
        getrs_prepare(st, n2, Sj, F->ipivT.p + (size_t)j * n2, F->permT.p + (size_t)j * n2,
                      F->dinvT.p + (size_t)j * dinv_sz);
        continue;
      }
      dgetrs(st, n2, n2, LUp, ip, X, n2, nullptr);
      dgemm_batched(st, n2, n2, n2, -1.0, sub, n2, 0, X, n2, 0, 1.0, Sj, n2, 0, 1);
    }
    factor_S(F, j);
  }
  if (ev_in) cudaEventDestroy(ev_in);
  if (ev_right) cudaEventDestroy(ev_right);
}

void stage_two_build(slablu_gpu_fact* F) {
  stage_two_alloc(F);
  stage_two_range(F, 0, F->K);
}

// build_reduced in hbs mode (stage_one.hpp:357-411): every reduced block compressed with the
// adaptive randomized HBS scheme and densified in place, seeds mix_seed(seed, ordinal) with the
// reference's ordinals (diag j: 3j, super j: 3j+1, sub j: 3j+2), leaf and rank range derived
// as stage_one.hpp:364-370.
void hbs_reduce(slablu_gpu_fact* F, const slablu_gpu_config& c) {
  const int64_t n2 = F->n2, K = F->K, bs = n2 * n2;
  HbsOptions o;
  o.tol = c.hbs_tol > 0 ? c.hbs_tol : 1e-11;
  o.trunc_rel = c.hbs_trunc_rel > 0 ? c.hbs_trunc_rel : 1e-13;
  const int64_t leaf_cfg = c.hbs_leaf_size > 0 ? c.hbs_leaf_size : 64;
  const int64_t leaf = std::min(leaf_cfg, n2);
  int64_t r_start = std::max<int64_t>(2, (leaf - 10 + 1) / 2);
  int64_t r_max = std::max<int64_t>(2 * F->b + 8, r_start);
  r_max = std::min(r_max, n2);
  r_start = std::min(r_start, r_max);
  o.leaf = (int)leaf;
  o.r_start = r_start;
  o.r_max = r_max;
  std::vector<double*> blocks;
  std::vector<uint64_t> seeds;
  std::vector<std::pair<int64_t, int64_t>> jk;
  for (int64_t j = 0; j < K; j++) {
    blocks.push_back(F->Tdiag() + j * bs);
    seeds.push_back(mix_seed(c.seed, 3 * j));
    jk.push_back({j, j});
  }
  for (int64_t j = 0; j + 1 < K; j++) {
    blocks.push_back(F->Tsup() + j * bs);
    seeds.push_back(mix_seed(c.seed, 3 * j + 1));
    jk.push_back({j, j + 1});
    blocks.push_back(F->Tsub() + j * bs);
    seeds.push_back(mix_seed(c.seed, 3 * j + 2));
    jk.push_back({j + 1, j});
  }
  std::vector<HbsStats> stats(blocks.size());
  {
    // the compression works in stream-ordered allocations sized by the free memory: blocks the
    // exact-size pool keeps from earlier factorizations would shrink its batches to one block
    size_t fr = 0, tot = 0;
    SLB_CUDA_CHECK(cudaMemGetInfo(&fr, &tot));
    const HbsFootprint fp = hbs_footprint(n2, o);
    const double want = fp.densify + fp.per_block * (double)blocks.size();
    if (0.6 * (double)fr < want && pool().cached_bytes(F->device) > 0) pool().trim(F->device);
  }
  cudaEvent_t h0, h1;
  SLB_CUDA_CHECK(cudaEventCreate(&h0));
  SLB_CUDA_CHECK(cudaEventCreate(&h1));
  SLB_CUDA_CHECK(cudaEventRecord(h0, F->stream));
  try {
    hbs_compress_blocks(F->stream, n2, (int)blocks.size(), blocks.data(), seeds.data(), o, stats.data());
  } catch (const HostError& e) {
    cudaEventDestroy(h0);
    cudaEventDestroy(h1);
    if (e.code != SLABLU_ERR_COMPRESSION || e.index < 0) throw;
    const auto& p = jk[(size_t)e.index];
    HostError w(e.code, "build_reduced: block (" + std::to_string(p.first) + ", " + std::to_string(p.second) +
                            "): " + e.what(), -1);
    w.residual = e.residual;
    throw w;
  }
  SLB_CUDA_CHECK(cudaEventRecord(h1, F->stream));
  SLB_CUDA_CHECK(cudaEventSynchronize(h1));
  float ms = 0;
  SLB_CUDA_CHECK(cudaEventElapsedTime(&ms, h0, h1));
  F->t_hbs = ms * 1e-3;
  cudaEventDestroy(h0);
  cudaEventDestroy(h1);
  F->hbs_max_rank = 0;
  for (const HbsStats& st : stats) F->hbs_max_rank = std::max(F->hbs_max_rank, st.final_rank);
}

slablu_gpu_fact* factorize_impl(int64_t n1, int64_t n2, int64_t nnz, const int32_t* rp, const int32_t* ci,
                                const double* v, const slablu_gpu_config* cfg, int rank = 0, int nranks = 1,
                                bool sharded = false) {
  if (n1 * n2 == 0) throw HostError(SLABLU_ERR_CONFIG, "factorize: empty system");
  slablu_gpu_config c{};
  c.c = 0.6;
  if (cfg) c = *cfg;
  if (c.compression < 0 || c.compression > 2) throw HostError(SLABLU_ERR_CONFIG, "factorize: unknown compression choice");
  const int64_t launches0 = slb::g_kernel_count.load();
  auto F = std::make_unique<slablu_gpu_fact>();
  F->device = c.device;
  DeviceGuard dg(c.device);
  {
    // the level chain is latency-bound: its stream gets the greatest priority so that its CTAs
    // are scheduled ahead of the conversion kernels running beside it (which use the least)
    int least = 0, greatest = 0;
    SLB_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    SLB_CUDA_CHECK(cudaStreamCreateWithPriority(&F->stream, cudaStreamNonBlocking, greatest));
  }
  cudaStream_t st = F->stream;
  StreamScope scope(st);
  F->n1 = n1;
  F->n2 = n2;
  F->N = n1 * n2;
  F->b = c.b > 0 ? c.b : choose_b(n1, n2, 0, c.c);
  const int dev = c.device;
  // driver.hpp:125-130: automatic compresses once the interfaces are long enough
  const bool use_hbs = c.compression == 2 || (c.compression == 0 && n2 >= 512 && F->b >= 16 && !sharded);
  if (use_hbs && sharded)
    throw HostError(SLABLU_ERR_UNSUPPORTED, "shard: hbs compression needs whole reduced blocks (use dense)");
  F->compression = use_hbs ? 2 : 1;

  // geometry (driver.hpp:134-139: degenerate whole-grid path)
  std::vector<GridStrip> ints;
  std::vector<GridStrip> ifcs;
  if (F->b > n1 - 2 || n1 < 3) {
    F->single = true;
    ints.push_back({0, n1});
  } else {
    Partition p = partition(n1, n2, F->b);
    ints = p.interiors;
    ifcs = p.interfaces;
  }
  F->Sg = (int)ints.size();
  F->K = (int)ifcs.size();
  F->rank = rank;
  F->nranks = nranks;
  F->sharded = sharded;
  if (sharded) {
    if (F->single) throw HostError(SLABLU_ERR_CONFIG, "shard: the degenerate single-slab path does not shard");
    if (F->Sg < nranks)
      throw HostError(SLABLU_ERR_CONFIG, "shard: " + std::to_string(F->Sg) + " strips cannot cover " +
                                             std::to_string(nranks) + " ranks");
  }
  shard_ranges(F->Sg, F->K, rank, nranks, &F->s0, &F->s1, &F->j0, &F->j1);
  ints = std::vector<GridStrip>(ints.begin() + F->s0, ints.begin() + F->s1);
  F->S = (int)ints.size();
  int64_t wmax = 0;
  for (auto& s : ints) wmax = std::max(wmax, s.width);
  F->Wp = (int)round_up(wmax, 8);
  if (F->Wp > 160)
    throw HostError(SLABLU_ERR_UNSUPPORTED, "factorize: slab width " + std::to_string(wmax) + " exceeds the engine's 160-column envelope");
  if (!F->single && n2 > kMaxIfc)
    throw HostError(SLABLU_ERR_UNSUPPORTED, "factorize: interface length n2 = " + std::to_string(n2) +
                                                " exceeds the engine's " + std::to_string(kMaxIfc) +
                                                "-row stage-two envelope");
  const int Wp = F->Wp, S = F->S, K = F->K;
  for (int s = 0; s < S; s++) {
    StripDesc d;
    d.col0 = (int32_t)ints[s].first_col;
    d.w = (int32_t)ints[s].width;
    const int gs = F->s0 + s;  // global strip index
    d.left = gs > 0 ? gs - 1 : -1;
    d.right = gs < K ? gs : -1;
    d.left_off = d.left >= 0 ? ifcs[d.left].first_col * n2 : -1;
    d.right_off = d.right >= 0 ? ifcs[d.right].first_col * n2 : -1;
    F->strips_h.push_back(d);
  }
  for (auto& f : ifcs) F->ifc_off_h.push_back(f.first_col * n2);

  cudaEvent_t e0, e1, e2, ec, es;
  SLB_CUDA_CHECK(cudaEventCreate(&e0));
  SLB_CUDA_CHECK(cudaEventCreate(&e1));
  SLB_CUDA_CHECK(cudaEventCreate(&e2));
  SLB_CUDA_CHECK(cudaEventCreate(&ec));
  SLB_CUDA_CHECK(cudaEventCreate(&es));
  SLB_CUDA_CHECK(cudaEventRecord(e0, st));

  F->strips.alloc(dev, S);
  SLB_CUDA_CHECK(cudaMemcpyAsync(F->strips.p, F->strips_h.data(), S * sizeof(StripDesc), cudaMemcpyHostToDevice, st));
  if (K > 0) {
    F->ifc_off.alloc(dev, K);
    SLB_CUDA_CHECK(cudaMemcpyAsync(F->ifc_off.p, F->ifc_off_h.data(), K * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  }
  F->status.alloc(dev, 1);
  F->sstatus.alloc(dev, 1);
  static const DevStatus st0{0, INT_MAX, INT_MAX, INT_MAX};
  SLB_CUDA_CHECK(cudaMemcpyAsync(F->status.p, &st0, sizeof(DevStatus), cudaMemcpyHostToDevice, st));
  SLB_CUDA_CHECK(cudaMemcpyAsync(F->sstatus.p, &st0, sizeof(DevStatus), cudaMemcpyHostToDevice, st));
  CsrDev A{rp, ci, v, F->N};
  F->refine = std::max(0, c.refine);
  if (F->refine > 0) {
    F->a_rp.alloc(dev, F->N + 1);
    F->a_ci.alloc(dev, nnz);
    F->a_v.alloc(dev, nnz);
    SLB_CUDA_CHECK(cudaMemcpyAsync(F->a_rp.p, rp, (F->N + 1) * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    SLB_CUDA_CHECK(cudaMemcpyAsync(F->a_ci.p, ci, nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    SLB_CUDA_CHECK(cudaMemcpyAsync(F->a_v.p, v, nnz * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }

  // ---- stage one: couplings + level chain ---------------------------------------
  const int64_t lvl = 4LL * Wp * Wp;
  F->sF = n2 * lvl;
  F->sP = n2 * 2 * Wp;
  F->sCPL = 4 * n2 * Wp;
  F->fac.alloc(dev, (size_t)S * F->sF);
  F->perm.alloc(dev, (size_t)S * F->sP);
  F->cpl.alloc(dev, (size_t)S * F->sCPL);
  F->sym.alloc(dev, S);
  F->u13.alloc(dev, (size_t)S * n2);
  F->lnd.alloc(dev, (size_t)2 * S * n2);  // planes: Lsub / Usup not diagonal
  F->dsub.alloc(dev, (size_t)S * n2 * Wp);
  F->exc.alloc(dev, (size_t)S * n2 * 8 * Wp);
  F->excpos.alloc(dev, (size_t)S * n2 * 8);
  F->hcol.alloc(dev, (size_t)S * n2 * 8 * Wp);
  F->hidx.alloc(dev, (size_t)S * n2 * 8);
  SLB_CUDA_CHECK(cudaMemsetAsync(F->lnd.p, 0, F->lnd.bytes(), st));
  SLB_CUDA_CHECK(cudaMemsetAsync(F->dsub.p, 0, F->dsub.bytes(), st));
  {
    std::vector<int32_t> ones(S, 1);
    SLB_CUDA_CHECK(cudaMemcpyAsync(F->sym.p, ones.data(), S * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  }
  extract_couplings(st, A, F->strips.p, S, n2, Wp, F->cpl.p, F->sCPL, F->sym.p, F->status.p);

  const int64_t LCH = std::min<int64_t>(n2, 64);
  const int64_t sNX = LCH * 3 * Wp * Wp;
  DBuf<double> nx, sv;
  nx.alloc(dev, (size_t)S * sNX);
  sv.alloc(dev, (size_t)2 * S * 2 * Wp * Wp);
  const int64_t sSV = 2LL * Wp * Wp;
  double* svb[2] = {sv.p, sv.p + (size_t)S * sSV};
  extract_levels(st, A, F->strips.p, S, n2, Wp, 0, LCH, nx.p, sNX, F->status.p, F->dsub.p, F->lnd.p);
  init_sv(st, S, Wp, nx.p, sNX, svb[0], sSV);
  // LU-form -> GEMM-form conversion runs behind the chain on a low-priority
  // stream, one chunk of CCH levels at a time (idle SMs during the chain).
  // levels per conversion chunk (SLB_CONV_CHUNK, measurement): cfg3 chain 0.835 / 0.794 / 0.781 /
  // 0.787 / 0.812 s at 64 / 96 / 128 / 256 / 512
  static const int64_t cch_env = getenv("SLB_CONV_CHUNK") ? atoi(getenv("SLB_CONV_CHUNK")) : 128;
  const int64_t CCH = std::min<int64_t>(n2, std::max<int64_t>(64, cch_env));
  // conversion stream: a green-context partition that leaves the chain (one CTA per strip)
  // SMs of its own (SLB_NO_GREEN=1 disables; SLB_GREEN_SMS sets the partition), else a
  // least-priority stream.  cfg3: chain phase 0.981 -> 0.959 s with 120 of 148 SMs for the
  // conversion; smaller partitions no longer hide the conversion behind the chain.
  cudaStream_t cst = nullptr;
  bool cst_owned = false;
  // the partition pays only when the chain is long and the conversion large (cfg3-sized)
  if (S * n2 >= 16384 && n2 >= 1024) {
    const char* e = getenv("SLB_GREEN_SMS");
    const int want = e ? atoi(e) : sm_count(dev) - (int)round_up(S + 4, 8);
    cst = green_partition_stream(dev, want);
  }
  if (!cst) {
    int lo = 0, hi = 0;
    SLB_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    SLB_CUDA_CHECK(cudaStreamCreateWithPriority(&cst, cudaStreamNonBlocking, lo));
    cst_owned = true;
  }
  DBuf<double> cwork;
  cwork.alloc(dev, (size_t)CCH * 4 * Wp * Wp * S);
  cudaEvent_t chunk_ev;
  SLB_CUDA_CHECK(cudaEventCreateWithFlags(&chunk_ev, cudaEventDisableTiming));
  static const bool defer_conv = getenv("SLB_CONV_DEFER") != nullptr;  // measurement: no overlap
  auto convert_chunk = [&](int64_t c0, int64_t c1) {
    SLB_CUDA_CHECK(cudaEventRecord(chunk_ev, st));
    SLB_CUDA_CHECK(cudaStreamWaitEvent(cst, chunk_ev, 0));
    for (int s = 0; s < S; s++) {
      convert_levels(cst, Wp, F->fac.p + s * F->sF + c0 * lvl, lvl, c1 - c0, cwork.p + (size_t)s * CCH * 4 * Wp * Wp,
                     F->perm.p + s * F->sP + c0 * 2 * Wp, F->exc.p + ((size_t)s * n2 + c0) * 8 * Wp,
                     F->excpos.p + ((size_t)s * n2 + c0) * 8, F->hcol.p + ((size_t)s * n2 + c0) * 8 * Wp,
                     F->hidx.p + ((size_t)s * n2 + c0) * 8);
    }
  };
  int cur = 0;
  int64_t conv_done = 0;  // levels [0, conv_done) handed to the conversion stream
  for (int64_t l = 0; l < n2; l++) {
    const int64_t nxt = l + 1;
    const bool has_next = nxt < n2;
    // chunks of CCH levels; 64-level chunks over the last 2 CCH levels so that little
    // conversion is left once the chain ends
    const int64_t cch = (n2 - l <= 2 * CCH) ? std::min<int64_t>(CCH, 64) : CCH;
    if (!defer_conv && l - conv_done >= cch) {
      convert_chunk(conv_done, l);
      conv_done = l;
    }
    if (has_next && nxt % LCH == 0) {
      extract_levels(st, A, F->strips.p, S, n2, Wp, nxt, std::min(LCH, n2 - nxt), nx.p, sNX, F->status.p,
                     F->dsub.p, F->lnd.p);
    }
    LevelArgs la;
    la.Wp = Wp;
    la.nstrips = S;
    la.has_next = has_next;
    la.sv_in = svb[cur];
    la.sSV = sSV;
    la.nx = has_next ? nx.p + (nxt % LCH) * 3 * Wp * Wp : nullptr;
    la.sNX = sNX;
    la.sv_out = svb[1 - cur];
    la.slot = F->fac.p + l * lvl;
    la.sF = F->sF;
    la.perm = F->perm.p + l * 2 * Wp;
    la.sP = F->sP;
    la.u13 = F->u13.p + l;
    la.sU13 = n2;
    la.lnd = F->lnd.p + (has_next ? l + 1 : l);
    la.status = F->status.p;
    la.level = (int32_t)l;
    level_lu(st, la);
    if (has_next) {
      level_update(st, la);
    }
    cur = 1 - cur;
  }
  cudaEvent_t chain_end = nullptr;
  if (defer_conv) {
    SLB_CUDA_CHECK(cudaEventCreate(&chain_end));
    SLB_CUDA_CHECK(cudaEventRecord(chain_end, st));
    for (int64_t c0 = 0; c0 + CCH < n2; c0 += CCH) convert_chunk(c0, c0 + CCH);
  }
  if (!defer_conv) convert_chunk(conv_done, n2);
  else convert_chunk(((n2 - 1) / CCH) * CCH, n2);
  SLB_CUDA_CHECK(cudaEventRecord(chunk_ev, cst));
  SLB_CUDA_CHECK(cudaStreamWaitEvent(st, chunk_ev, 0));
  SLB_CUDA_CHECK(cudaEventDestroy(chunk_ev));
  if (cst_owned) SLB_CUDA_CHECK(cudaStreamDestroy(cst));
  nx.release();
  sv.release();
  SLB_CUDA_CHECK(cudaEventRecord(ec, st));
  if (chain_end) {
    SLB_CUDA_CHECK(cudaEventSynchronize(ec));
    float a = 0, b2 = 0;
    SLB_CUDA_CHECK(cudaEventElapsedTime(&a, e0, chain_end));
    SLB_CUDA_CHECK(cudaEventElapsedTime(&b2, chain_end, ec));
    fprintf(stderr, "[slablu] chain alone %.1f ms, conversion after it %.1f ms\n", a, b2);
    cudaEventDestroy(chain_end);
  }
  {
    DevStatus hs;
    SLB_CUDA_CHECK(cudaMemcpyAsync(&hs, F->status.p, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
    SLB_CUDA_CHECK(cudaStreamSynchronize(st));
    throw_status(hs);
    if (hs.flags & ERR_SINGULAR) {
      // single slab: the natural index (ix * n2 + iy) of the first zero pivot, as BandedLU reports
      // dgbtrf's info - 1 (banded.hpp:103-109); else the global strip index (stage_one.hpp:234-237)
      if (F->single) {
        const int64_t lvl_ = hs.singular_pos / Wp, col_ = hs.singular_pos % Wp;
        throw HostError(SLABLU_ERR_SINGULAR, "BandedLU: exactly singular pivot", col_ * n2 + lvl_);
      }
      throw HostError(SLABLU_ERR_SINGULAR, "factor_one_interior: singular slab interior",
                      (int64_t)hs.singular_strip + F->s0);
    }
    if (getenv("SLB_U13_STATS")) {
      std::vector<uint8_t> h((size_t)S * n2);
      SLB_CUDA_CHECK(cudaMemcpy(h.data(), F->u13.p, h.size(), cudaMemcpyDeviceToHost));
      int64_t ones = 0, pairs = 0, hist[16] = {0};
      for (int s = 0; s < S; s++)
        for (int64_t l = 0; l < n2; l++) {
          ones += h[s * n2 + l] & 1;
          pairs += (h[s * n2 + l] & 3) != 0 ? 1 : 0;
          hist[h[s * n2 + l] >> 2]++;
        }
      fprintf(stderr, "[slablu] rows pivoted up per level:");
      for (int i = 0; i < 16; i++) fprintf(stderr, " %d:%lld", i, (long long)hist[i]);
      fprintf(stderr, "\n");
      fprintf(stderr, "[slablu] U13 != 0 on %lld of %lld levels; full forward operator needed on %lld\n", (long long)ones,
              (long long)(S * n2), (long long)pairs);
    }
    F->sym_h.resize(S);
    SLB_CUDA_CHECK(cudaMemcpy(F->sym_h.data(), F->sym.p, S * sizeof(int32_t), cudaMemcpyDeviceToHost));
  }

  if (!F->single) {
    // ---- Schur sweep ----------------------------------------------------------------
    std::vector<int32_t> tasks;
    std::vector<std::array<int64_t, 4>> order;  // (-work, q0, strip, side)
    for (int s = 0; s < S; s++)
      for (int side = 0; side < 2; side++) {
        if ((side == 0 ? F->strips_h[s].left : F->strips_h[s].right) < 0) continue;
        for (int64_t q0 = 0; q0 < n2; q0 += kSweepChunk) {
          const int64_t l0 = q0 > 0 ? q0 - 1 : 0;
          const int64_t work = (n2 - l0) + (F->sym_h[s] ? n2 - q0 : n2);
          order.push_back({-work, q0, s, side});
        }
      }
    std::sort(order.begin(), order.end());
    for (auto& o : order) {
      tasks.push_back((int32_t)o[2]);
      tasks.push_back((int32_t)o[3]);
      tasks.push_back((int32_t)o[1]);
    }
    const int ntasks = (int)order.size();
    DBuf<int32_t> dtasks, counter;
    dtasks.alloc(dev, tasks.size());
    counter.alloc(dev, 1);
    SLB_CUDA_CHECK(cudaMemcpyAsync(dtasks.p, tasks.data(), tasks.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    SLB_CUDA_CHECK(cudaMemsetAsync(counter.p, 0, sizeof(int32_t), st));
    const int64_t sG = 4 * n2 * n2;
    DBuf<double> gbuf, ybuf;
    gbuf.alloc(dev, (size_t)S * sG);
    SLB_CUDA_CHECK(cudaMemsetAsync(gbuf.p, 0, gbuf.bytes(), st));
    const int64_t sY = n2 * Wp * kSweepChunk;
    int nslots = std::min(sm_count(dev), ntasks);
    {
      size_t fr = 0, tot = 0;
      SLB_CUDA_CHECK(cudaMemGetInfo(&fr, &tot));
      fr += pool().cached_bytes(dev);  // cached blocks are reusable (trimmed on demand)
      const size_t reserve = (size_t)(3 * K) * n2 * n2 * sizeof(double) + (size_t)(4LL << 30);
      const size_t per = (size_t)sY * sizeof(double);
      if (fr > reserve) nslots = (int)std::max<int64_t>(1, std::min<int64_t>(nslots, (fr - reserve) / per));
      else nslots = 1;
    }
    ybuf.alloc(dev, (size_t)nslots * sY);
    SchurArgs sa{};
    sa.Wp = Wp;
    sa.n2 = n2;
    sa.nstrips = S;
    sa.strips = F->strips.p;
    sa.fac = F->fac.p;
    sa.sF = F->sF;
    sa.perm = F->perm.p;
    sa.sP = F->sP;
    sa.cpl = F->cpl.p;
    sa.sCPL = F->sCPL;
    sa.sym = F->sym.p;
    sa.u13 = F->u13.p;
    sa.dsub = F->dsub.p;
    sa.fsc = getenv("SLB_NO_FSC") ? 0 : 1;  // forward shortcut (SLB_NO_FSC=1 disables, for A/B runs)
    sa.exc = F->exc.p;
    sa.excpos = F->excpos.p;
    sa.bsc = getenv("SLB_NO_BSC") ? 0 : 1;  // backward shortcut (SLB_NO_BSC=1 disables, for A/B runs)
    sa.hcol = F->hcol.p;
    sa.hidx = F->hidx.p;
    sa.chunk = kSweepChunk;
    sa.gbuf = gbuf.p;
    sa.sG = sG;
    sa.ybuf = ybuf.p;
    sa.sY = sY;
    sa.task_counter = counter.p;
    sa.ntasks = ntasks;
    sa.tasks = dtasks.p;
    sa.mode = SWEEP_SCHUR;
    sweep(st, sa, nslots);
    SLB_CUDA_CHECK(cudaEventRecord(es, st));
    ybuf.release();
    // ---- T assembly --------------------------------------------------------------------
    F->T.alloc(dev, (size_t)(3 * K - 2) * n2 * n2);
    TRanges tr;
    tr.sbase = F->s0;
    tr.nstrips_global = F->Sg;
    tr.dlo = std::max(0, F->s0 - 1);  // diag blocks touching a local strip
    tr.dhi = std::min(K, F->s1);
    tr.olo = F->j0;  // owned: direct operator terms
    tr.ohi = F->j1;
    tr.ulo = std::max(0, F->s0 - 1);  // super/sub j come from strip j+1
    tr.uhi = std::min(K - 1, F->s1 - 1);
    assemble_T(st, n2, K, S, F->strips.p, F->sym.p, gbuf.p, sG, F->Tdiag(), F->Tsup(), F->Tsub(), A,
               F->ifc_off.p, F->status.p, tr);
    check_finite(st, F->T.p, (int64_t)(3 * K - 2) * n2 * n2, F->status.p);
    if (F->compression == 2 && K > 0) hbs_reduce(F.get(), c);
    if (c.keep_T) {
      F->Tkeep.alloc(dev, F->T.n);
      SLB_CUDA_CHECK(cudaMemcpyAsync(F->Tkeep.p, F->T.p, F->T.bytes(), cudaMemcpyDeviceToDevice, st));
    }
    gbuf.release();
    SLB_CUDA_CHECK(cudaEventRecord(e1, st));

    // ---- stage two: sweeping block LU (stage_two.hpp:131-150) --------------------------
    if (!sharded) stage_two_build(F.get());  // sharded: slablu_gpu_shard_sweep
  } else {
    SLB_CUDA_CHECK(cudaEventRecord(es, st));
    SLB_CUDA_CHECK(cudaEventRecord(e1, st));
  }
  SLB_CUDA_CHECK(cudaEventRecord(e2, st));
  SLB_CUDA_CHECK(cudaEventSynchronize(e2));
  {
    DevStatus hs;
    SLB_CUDA_CHECK(cudaMemcpy(&hs, F->status.p, sizeof(DevStatus), cudaMemcpyDeviceToHost));
    throw_status(hs);
    if (hs.flags & ERR_NONFINITE) throw HostError(SLABLU_ERR_GENERIC, "BlockTridiagonal: non-finite block entry");
    if (hs.flags & ERR_SINGULAR)
      throw HostError(SLABLU_ERR_SINGULAR, "sweep_build: singular Schur complement block", hs.singular_block);
  }
  float ms1 = 0, ms2 = 0, msc = 0, mss = 0, msa = 0;
  SLB_CUDA_CHECK(cudaEventElapsedTime(&ms1, e0, e1));
  SLB_CUDA_CHECK(cudaEventElapsedTime(&ms2, e1, e2));
  SLB_CUDA_CHECK(cudaEventElapsedTime(&msc, e0, ec));
  SLB_CUDA_CHECK(cudaEventElapsedTime(&mss, ec, es));
  SLB_CUDA_CHECK(cudaEventElapsedTime(&msa, es, e1));
  F->t_chain = msc * 1e-3;
  F->t_schur = mss * 1e-3;
  F->t_asm = msa * 1e-3;
  for (cudaEvent_t ev : {e0, e1, e2, ec, es}) cudaEventDestroy(ev);
  F->t1 = ms1 * 1e-3;
  F->t2 = ms2 * 1e-3;
  // reference-equivalent storage (driver.hpp:153-159; stage_two.hpp:191-198)
  for (auto& s : F->strips_h) {
    const int64_t w = s.w;
    if (F->single) {
      F->storage1 += (3 * n2 + 1) * F->N;  // BandedLU(n, n2, n2) in the reference
    } else {
      F->storage1 += (3 * w + 1) * w * n2 + (s.left >= 0 ? 2 * n2 : 0) + (s.right >= 0 ? 2 * n2 : 0);
    }
  }
  if (!F->single) F->storage2 = (int64_t)(K + 2 * (K - 1)) * n2 * n2;
  F->launches_factor = slb::g_kernel_count.load() - launches0;
  return F.release();
}

// Raises the solve-time device status (bounded waits of getrs_chain that expired) and re-arms it.
void check_solve_status(const slablu_gpu_fact* F) {
  DevStatus hs;
  SLB_CUDA_CHECK(cudaMemcpyAsync(&hs, F->sstatus.p, sizeof(DevStatus), cudaMemcpyDeviceToHost, F->stream));
  SLB_CUDA_CHECK(cudaStreamSynchronize(F->stream));
  if (hs.flags) {
    static const DevStatus st0{0, INT_MAX, INT_MAX, INT_MAX};
    SLB_CUDA_CHECK(cudaMemcpyAsync(F->sstatus.p, &st0, sizeof(DevStatus), cudaMemcpyHostToDevice, F->stream));
    SLB_CUDA_CHECK(cudaStreamSynchronize(F->stream));
    throw HostError(SLABLU_ERR_CUDA, "solve: stage-two block chain timed out (a published block never arrived)");
  }
}

// Slab sweeps of the solve for the factorization's (local) strips: reduce (contributions
// to_X A_ii^{-1} f_i) or recover (A_ii^{-1}(f_i - couplings u)).  nrhs <= 8: cluster sweeps
// (solve.cu); more columns: the 64-column persistent sweep kernel (schur.cu).
struct StripSweeper {
  const slablu_gpu_fact* F;
  cudaStream_t st;
  int CH = 8, ntasks = 0, nslots = 0;
  bool clustered = false, v2 = false;
  DBuf<int32_t> dtasks, counter;
  DBuf<double> ybuf;
  SchurArgs sa{};
  StripSweeper(const slablu_gpu_fact* F_, const double* fp, int64_t nrhs) : F(F_), st(F_->stream) {
    const int dev = F->device;
    const int64_t n2 = F->n2;
    // 8-column tasks on the cluster kernel for any nrhs (each task streams its strip's operators
    // once per 8 columns but keeps every SM busy); the 64-column sweep kernel (one CTA per
    // strip and chunk) only if the cluster kernel does not fit or SLB_SOLVE_WIDE=1 (A/B runs)
    static const bool wide = getenv("SLB_SOLVE_WIDE") != nullptr;
    static const bool force_v1_ch = getenv("SLB_SOLVE_V1") != nullptr;
    CH = (nrhs <= 8 || (!wide && !force_v1_ch && strip_solve2_fits(F->Wp, n2, std::min(4, F->Wp / 8)))) ? 8
                                                                                                       : kSweepChunk;
    const int64_t nch = cdiv(nrhs, CH);
    std::vector<int32_t> tasks;
    for (int s = 0; s < F->S; s++)
      for (int64_t cch = 0; cch < nch; cch++) {
        tasks.push_back(s);
        tasks.push_back(0);
        tasks.push_back((int32_t)(cch * CH));
      }
    ntasks = (int)(tasks.size() / 3);
    dtasks.alloc(dev, tasks.size());
    counter.alloc(dev, 1);
    SLB_CUDA_CHECK(cudaMemcpyAsync(dtasks.p, tasks.data(), tasks.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    // cluster sweeps for small nrhs: version 2 (TMA tensor slices + st.async exchange, solve2.cu)
    // unless SLB_SOLVE_V1=1 selects the round-1 kernel (solve.cu)
    static const bool force_v1 = getenv("SLB_SOLVE_V1") != nullptr;
    v2 = CH == 8 && !force_v1 && strip_solve2_fits(F->Wp, n2, std::min(4, F->Wp / 8));
    clustered = CH == 8 && (v2 || strip_solve_fits(F->Wp, n2));
    nslots = clustered ? ntasks : std::min(sm_count(dev), ntasks);
    const int64_t sY = n2 * F->Wp * CH;
    ybuf.alloc(dev, (size_t)nslots * sY);
    sa.chunk = CH;
    sa.u13 = F->u13.p;
    sa.dsub = F->dsub.p;
    sa.fsc = getenv("SLB_NO_FSC") ? 0 : getenv("SLB_SOLVE_NOTMA") ? 2 : 1;  // forward shortcut (A/B runs)
    sa.exc = F->exc.p;
    sa.excpos = F->excpos.p;
    sa.bsc = getenv("SLB_NO_BSC") ? 0 : 1;  // backward shortcut (SLB_NO_BSC=1 disables, for A/B runs)
    sa.hcol = F->hcol.p;
    sa.hidx = F->hidx.p;
    sa.Wp = F->Wp;
    sa.n2 = n2;
    sa.nstrips = F->S;
    sa.strips = F->strips.p;
    sa.fac = F->fac.p;
    sa.sF = F->sF;
    sa.perm = F->perm.p;
    sa.sP = F->sP;
    sa.cpl = F->cpl.p;
    sa.sCPL = F->sCPL;
    sa.sym = F->sym.p;
    sa.ybuf = ybuf.p;
    sa.sY = sY;
    sa.task_counter = counter.p;
    sa.ntasks = ntasks;
    sa.tasks = dtasks.p;
    sa.N = F->N;
    sa.K = (int64_t)F->K * n2;
    sa.nrhs = nrhs;
    sa.f = fp;
  }
  void run(SweepMode mode, const double* u_ifc, double* out) {
    SLB_CUDA_CHECK(cudaMemsetAsync(counter.p, 0, sizeof(int32_t), st));
    sa.mode = mode;
    sa.u_ifc = u_ifc;
    sa.out = out;
    if (v2) {
      strip_solve2(st, sa, ntasks);  // rhs pack + cluster sweep (+ contributions in reduce mode)
    } else if (clustered) {
      strip_solve(st, sa, ntasks);  // rhs pack + cluster sweep
    } else {
      sweep(st, sa, nslots);
    }
  }
};

// reduce_rhs (stage_one.hpp:415-433): red (K n2 x nrhs, ld K n2) = f on the interfaces [jlo, jhi)
// minus the adjacent local strips' terms to_X A_ii^{-1} f_i.  fp: N x nrhs, ld N (device).
void reduce_phase(const slablu_gpu_fact* F, StripSweeper& sw, const double* fp, int64_t nrhs, double* red, int jlo,
                  int jhi) {
  cudaStream_t st = F->stream;
  const int64_t n2 = F->n2, N = F->N, Kn = (int64_t)F->K * n2;
  DBuf<double> contrib;
  contrib.alloc(F->device, (size_t)F->S * 2 * nrhs * n2);
  const unsigned gb = (unsigned)cdiv(Kn * nrhs, 256);
  gather_ifc_kernel<<<gb, 256, 0, st>>>(fp, N, nrhs, F->K, F->ifc_off.p, n2, red, Kn, jlo, jhi); count_launch();
  sw.run(SWEEP_REDUCE, nullptr, contrib.p);
  combine_reduce_kernel<<<gb, 256, 0, st>>>(red, Kn, nrhs, n2, F->S, F->strips.p, contrib.p, F->s0); count_launch();
  SLB_CUDA_CHECK(cudaGetLastError());
}

// Sweep solve over the interfaces [jlo, jhi) (stage_two.hpp:170-188) with the LU factors of S_j:
// forward u_j = S_j^{-1}(red_j - sub_{j-1} u_{j-1}), backward u_j -= S_j^{-1} super_j u_{j+1}.
// red and uifc are K n2 x nrhs (ld K n2); red is consumed (overwritten).
struct SweepSolver {
  const slablu_gpu_fact* F;
  int64_t nrhs;
  DBuf<double> yz, tmp, part;
  int epoch = 0;
  SweepSolver(const slablu_gpu_fact* F_, int64_t nrhs_) : F(F_), nrhs(nrhs_) {
    const int64_t n2 = F->n2;
    yz.alloc(F->device, (size_t)getrs_chain_scratch(n2, nrhs));
    tmp.alloc(F->device, (size_t)n2 * nrhs);
    part.alloc(F->device, (size_t)8 * n2 * nrhs);
    getrs_chain_init(F->stream, n2, nrhs, yz.p);
  }
  int64_t dinv_sz() const { return cdiv(F->n2, 64) * 2 * 64 * 64; }
  // out = beta out + alpha S_j^{-1} v
  void apply_Sinv(int j, const double* v, int64_t ldv, double* out, int64_t ldo, double alpha, double beta) {
    getrs_chain(F->stream, F->n2, nrhs, F->Tdiag() + (size_t)j * F->n2 * F->n2, F->dinvT.p + (size_t)j * dinv_sz(),
                F->permT.p + (size_t)j * F->n2, v, ldv, out, ldo, alpha, beta, yz.p, ++epoch, F->sstatus.p);
  }
  void forward(double* red, double* uifc, int jlo, int jhi) {
    const int64_t n2 = F->n2, Kn = (int64_t)F->K * n2, bs = n2 * n2;
    for (int j = jlo; j < jhi; j++) {
      double* rj = red + j * n2;
      if (j > jlo)
        dgemv_batched_rhs(F->stream, n2, n2, nrhs, -1.0, F->Tsub() + (j - 1) * bs, n2, uifc + (j - 1) * n2, Kn, 1.0,
                          rj, Kn, part.p);
      apply_Sinv(j, rj, Kn, uifc + j * n2, Kn, 1.0, 0.0);
    }
  }
  // backward u_j -= S_j^{-1} super_j u_{j+1} = X_j u_{j+1} (stage_two.hpp:181-187 with the block upper
  // factor kept by stage_two_build)
  // open_end: [jlo, jhi) is a chain of its own (u_{jhi} is not part of it: no X_{jhi-1} term)
  void backward(double* uifc, int jlo, int jhi, bool open_end = false) {
    const int64_t n2 = F->n2, Kn = (int64_t)F->K * n2, bs = n2 * n2;
    for (int j = jhi - 1; j >= jlo; j--) {
      if (j + 1 >= F->K || (open_end && j == jhi - 1)) continue;
      dgemv_batched_rhs(F->stream, n2, n2, nrhs, -1.0, F->Xup.p + (size_t)j * bs, n2, uifc + (j + 1) * n2, Kn, 1.0,
                        uifc + j * n2, Kn, part.p);
    }
  }
};

// recover_interiors (stage_one.hpp:438-462) on the local strips, then the owned interface
// values [jlo, jhi) copied in: up is N x nrhs (ld N).
void recover_phase(const slablu_gpu_fact* F, StripSweeper& sw, const double* uifc, int64_t nrhs, double* up, int jlo,
                   int jhi) {
  cudaStream_t st = F->stream;
  const int64_t n2 = F->n2, N = F->N, Kn = (int64_t)F->K * n2;
  sw.run(SWEEP_RECOVER, uifc, up);
  if (Kn > 0) {
    const unsigned gb = (unsigned)cdiv(Kn * nrhs, 256);
    scatter_ifc_kernel<<<gb, 256, 0, st>>>(uifc, Kn, nrhs, F->ifc_off.p, n2, up, N, jlo, jhi); count_launch();
  }
  SLB_CUDA_CHECK(cudaGetLastError());
}

void solve_once(const slablu_gpu_fact* F, const double* d_f, int64_t ldf, int64_t nrhs, double* d_u, int64_t ldu) {
  const int64_t launches0 = slb::g_kernel_count.load();
  cudaStream_t st = F->stream;
  const int dev = F->device;
  const int64_t n2 = F->n2, N = F->N, Kn = (int64_t)F->K * n2;
  // compact f (ld N)
  DBuf<double> f;
  const double* fp = d_f;
  if (ldf != N) {
    f.alloc(dev, (size_t)N * nrhs);
    copy2d(st, d_f, ldf, f.p, N, N, nrhs);
    fp = f.p;
  }
  DBuf<double> u;
  double* up = d_u;
  if (ldu != N) {
    u.alloc(dev, (size_t)N * nrhs);
    up = u.p;
  }
  cudaEvent_t s0, s1, s2, s3, s4;
  for (cudaEvent_t* ev : {&s0, &s1, &s2, &s3, &s4}) SLB_CUDA_CHECK(cudaEventCreate(ev));
  SLB_CUDA_CHECK(cudaEventRecord(s0, st));
  SLB_CUDA_CHECK(cudaEventRecord(s1, st));
  SLB_CUDA_CHECK(cudaEventRecord(s2, st));
  SLB_CUDA_CHECK(cudaEventRecord(s3, st));
  StripSweeper sw(F, fp, nrhs);
  if (F->single) {
    sw.run(SWEEP_RECOVER, nullptr, up);
  } else {
    DBuf<double> red, uifc;
    red.alloc(dev, (size_t)Kn * nrhs);
    uifc.alloc(dev, (size_t)Kn * nrhs);
    reduce_phase(F, sw, fp, nrhs, red.p, 0, F->K);
    SLB_CUDA_CHECK(cudaEventRecord(s1, st));
    SweepSolver ss(F, nrhs);
    ss.forward(red.p, uifc.p, 0, F->K);
    ss.backward(uifc.p, 0, F->K);
    SLB_CUDA_CHECK(cudaEventRecord(s2, st));
    recover_phase(F, sw, uifc.p, nrhs, up, 0, F->K);
    SLB_CUDA_CHECK(cudaEventRecord(s3, st));
  }
  if (up != d_u) copy2d(st, up, N, d_u, ldu, N, nrhs);
  SLB_CUDA_CHECK(cudaEventRecord(s4, st));
  SLB_CUDA_CHECK(cudaStreamSynchronize(st));
  float a = 0, b = 0, c = 0;
  SLB_CUDA_CHECK(cudaEventElapsedTime(&a, s0, s4));
  SLB_CUDA_CHECK(cudaEventElapsedTime(&b, s0, s1));
  SLB_CUDA_CHECK(cudaEventElapsedTime(&c, s2, s3));
  F->t_solve = a * 1e-3;
  F->t_solve_strips = F->single ? a * 1e-3 : (b + c) * 1e-3;
  for (cudaEvent_t ev : {s0, s1, s2, s3, s4}) cudaEventDestroy(ev);
  F->launches_solve = slb::g_kernel_count.load() - launches0;
}

void require_shard(const slablu_gpu_fact* F, const char* who) {
  if (!F->sharded) throw HostError(SLABLU_ERR_CONFIG, std::string(who) + ": not a sharded factorization");
}

// ---------------------------------------------------------------------------
// Partitioned stage two over the ranks.  Rank r owns the
// interfaces [j0, j1): for r > 0 the first, j0, is its separator s_r; the others form its interior
// chain [ia, ib) (ia = j0 + 1, or 0 on rank 0; ib = j1).  Every rank eliminates its interior on its
// own (shard_eliminate, no communication), leaving a block-tridiagonal system on the G - 1
// separators whose blocks are, with E_L = [sub_{j0}; 0 ..] and E_R = [.. 0; super_{ib-1}]:
//   D^_r = T_{s_r s_r} - super_{j0} (A_I^{-1} E_L)_first - sub_{ib'-1} (A_I'^{-1} E_R)_last   (I' of r-1)
//   U^_r = -super_{j0} (A_I^{-1} E_R)_first,   L^_r = -sub_{ib-1} (A_I^{-1} E_L)_last
// (direct couplings super_{j0} / sub_{j0} when the interior is empty).  The separator sweep is a
// pipeline with ONE n2 x n2 message per rank boundary (shard_sweep):
//   S^_r = T_{j0 j0}[own terms] - a_r + M_in,  X^_r = S^_r^{-1} b_r,
//   M_out = T_{j1 j1}[own strip term] - d_r - c_r X^_r          (c X^ = L^ S^^{-1} U^).
// The solve: every rank reduces its right-hand side and solves its interior (shard_solve_local);
// the separator values go forward and back through the pipeline with one n2 x nrhs message per
// boundary and direction; every rank then re-solves its interior with the separator couplings
// moved to the right-hand side and recovers its slab interiors.

void shard_eliminate_impl(slablu_gpu_fact* F) {
  require_shard(F, "shard_eliminate");
  DeviceGuard dg(F->device);
  cudaStream_t st = F->stream;
  StreamScope scope(st);
  const int dev = F->device;
  const int64_t n2 = F->n2, bs = n2 * n2;
  const int64_t l0 = slb::g_kernel_count.load();
  cudaEvent_t e0, e1;
  SLB_CUDA_CHECK(cudaEventCreate(&e0));
  SLB_CUDA_CHECK(cudaEventCreate(&e1));
  SLB_CUDA_CHECK(cudaEventRecord(e0, st));
  F->has_left = F->rank > 0;
  F->has_right = F->rank < F->nranks - 1;
  F->ia = F->has_left ? F->j0 + 1 : 0;
  F->ib = F->j1;
  const int ia = F->ia, ib = F->ib, m = ib - ia, j0 = F->j0;
  stage_two_alloc(F);
  stage_two_range(F, ia, ib);  // the interior chain: LU(S_j), X_j for j in [ia, ib - 1)
  for (DBuf<double>* b : {&F->sh_a, &F->sh_b, &F->sh_c, &F->sh_d, &F->sh_yl, &F->sh_xhat}) {
    b->alloc(dev, bs);
    SLB_CUDA_CHECK(cudaMemsetAsync(b->p, 0, b->bytes(), st));
  }
  auto gemm = [&](double* C, const double* A, const double* B, double alpha, double beta) {
    dgemm_batched(st, n2, n2, n2, alpha, A, n2, 0, B, n2, 0, beta, C, n2, 0, 1);
  };
  auto getrs = [&](int j, double* B) {  // B = S_j^{-1} B
    dgetrs(st, n2, n2, F->Tdiag() + (size_t)j * bs, F->ipivT.p + (size_t)j * n2, B, n2, nullptr);
  };
  auto copy = [&](double* dst, const double* src) {
    SLB_CUDA_CHECK(cudaMemcpyAsync(dst, src, bs * sizeof(double), cudaMemcpyDeviceToDevice, st));
  };
  if (m == 0) {  // adjacent separators couple directly: U^ = super_{j0}, L^ = sub_{j0}
    if (F->has_left && F->has_right) {
      add2d(st, F->Tsup() + (size_t)j0 * bs, n2, F->sh_b.p, n2, n2, n2, -1.0);
      add2d(st, F->Tsub() + (size_t)j0 * bs, n2, F->sh_c.p, n2, n2, n2, -1.0);
    }
  } else {
    DBuf<double> Y, t0;
    t0.alloc(dev, bs);
    if (F->has_left) {
      // A_I^{-1} E_L: forward y_ia = S_ia^{-1} sub_{j0}, y_j = -S_j^{-1} sub_{j-1} y_{j-1};
      // backward x_j = y_j - X_j x_{j+1} (all m blocks kept: the first and the last are needed)
      Y.alloc(dev, (size_t)m * bs);
      copy(Y.p, F->Tsub() + (size_t)j0 * bs);
      getrs(ia, Y.p);
      for (int j = ia + 1; j < ib; j++) {
        double* y = Y.p + (size_t)(j - ia) * bs;
        gemm(y, F->Tsub() + (size_t)(j - 1) * bs, y - bs, -1.0, 0.0);
        getrs(j, y);
      }
      for (int j = ib - 2; j >= ia; j--) {
        double* y = Y.p + (size_t)(j - ia) * bs;
        gemm(y, F->Xup.p + (size_t)j * bs, y + bs, -1.0, 1.0);
      }
      gemm(F->sh_a.p, F->Tsup() + (size_t)j0 * bs, Y.p, 1.0, 0.0);
      if (F->has_right) {
        copy(F->sh_yl.p, Y.p + (size_t)(m - 1) * bs);
        gemm(F->sh_c.p, F->Tsub() + (size_t)(ib - 1) * bs, F->sh_yl.p, 1.0, 0.0);
      }
      Y.release();
    }
    if (F->has_right) {
      // A_I^{-1} E_R: x_{ib-1} = S_{ib-1}^{-1} super_{ib-1}, x_j = -X_j x_{j+1}
      copy(t0.p, F->Tsup() + (size_t)(ib - 1) * bs);
      getrs(ib - 1, t0.p);
      gemm(F->sh_d.p, F->Tsub() + (size_t)(ib - 1) * bs, t0.p, 1.0, 0.0);
      if (F->has_left) {
        DBuf<double> t1;
        t1.alloc(dev, bs);
        double* cur = t0.p;
        double* nxt = t1.p;
        for (int j = ib - 2; j >= ia; j--) {
          gemm(nxt, F->Xup.p + (size_t)j * bs, cur, -1.0, 0.0);
          std::swap(cur, nxt);
        }
        gemm(F->sh_b.p, F->Tsup() + (size_t)j0 * bs, cur, 1.0, 0.0);
      }
    }
  }
  SLB_CUDA_CHECK(cudaEventRecord(e1, st));
  SLB_CUDA_CHECK(cudaEventSynchronize(e1));
  {
    DevStatus hs;
    SLB_CUDA_CHECK(cudaMemcpy(&hs, F->status.p, sizeof(DevStatus), cudaMemcpyDeviceToHost));
    if (hs.flags & ERR_SINGULAR)
      throw HostError(SLABLU_ERR_SINGULAR, "sweep_build: singular Schur complement block", hs.singular_block);
  }
  float ms = 0;
  SLB_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  F->t2 = ms * 1e-3;
  F->launches_factor += slb::g_kernel_count.load() - l0;
  F->eliminated = true;
}

// One step of the separator sweep (rank order): M_in from r - 1, M_out to r + 1 (n2 x n2, ld n2).
void shard_sweep_impl(slablu_gpu_fact* F, const double* d_in, double* d_out) {
  require_shard(F, "shard_sweep");
  if (!F->eliminated) throw HostError(SLABLU_ERR_CONFIG, "shard_sweep: call slablu_gpu_shard_eliminate first");
  if (F->has_left && !d_in) throw HostError(SLABLU_ERR_CONFIG, "shard_sweep: rank > 0 needs the message of rank - 1");
  if (F->has_right && !d_out)
    throw HostError(SLABLU_ERR_CONFIG, "shard_sweep: rank < nranks - 1 needs an output message buffer");
  DeviceGuard dg(F->device);
  cudaStream_t st = F->stream;
  StreamScope scope(st);
  const int64_t n2 = F->n2, bs = n2 * n2;
  const int j0 = F->j0, j1 = F->j1;
  const int64_t l0 = slb::g_kernel_count.load();
  cudaEvent_t e0, e1;
  SLB_CUDA_CHECK(cudaEventCreate(&e0));
  SLB_CUDA_CHECK(cudaEventCreate(&e1));
  SLB_CUDA_CHECK(cudaEventRecord(e0, st));
  if (F->has_left) {  // S^_r = T_{j0 j0} - a_r + M_in, in place; X^_r = S^_r^{-1} b_r
    double* Sh = F->Tdiag() + (size_t)j0 * bs;
    add2d(st, F->sh_a.p, n2, Sh, n2, n2, n2, -1.0);
    add2d(st, d_in, n2, Sh, n2, n2, n2, 1.0);
    factor_S(F, j0);
    if (F->has_right) {
      SLB_CUDA_CHECK(cudaMemcpyAsync(F->sh_xhat.p, F->sh_b.p, bs * sizeof(double), cudaMemcpyDeviceToDevice, st));
      dgetrs(st, n2, n2, Sh, F->ipivT.p + (size_t)j0 * n2, F->sh_xhat.p, n2, nullptr);
    }
  }
  if (F->has_right) {  // M_out = T_{j1 j1}[own strip term] - d_r - c_r X^_r
    SLB_CUDA_CHECK(cudaMemcpyAsync(d_out, F->Tdiag() + (size_t)j1 * bs, bs * sizeof(double), cudaMemcpyDeviceToDevice, st));
    add2d(st, F->sh_d.p, n2, d_out, n2, n2, n2, -1.0);
    if (F->has_left) dgemm_batched(st, n2, n2, n2, -1.0, F->sh_c.p, n2, 0, F->sh_xhat.p, n2, 0, 1.0, d_out, n2, 0, 1);
  }
  SLB_CUDA_CHECK(cudaEventRecord(e1, st));
  SLB_CUDA_CHECK(cudaEventSynchronize(e1));
  {
    DevStatus hs;
    SLB_CUDA_CHECK(cudaMemcpy(&hs, F->status.p, sizeof(DevStatus), cudaMemcpyDeviceToHost));
    if (hs.flags & ERR_SINGULAR)
      throw HostError(SLABLU_ERR_SINGULAR, "sweep_build: singular Schur complement block", hs.singular_block);
  }
  float ms = 0;
  SLB_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  F->t2 += ms * 1e-3;
  F->launches_factor += slb::g_kernel_count.load() - l0;
  F->swept = true;
}

// Solve, local phase: reduce_rhs on the local strips (stage_one.hpp:415-433) and the interior
// chain solve z = A_I^{-1} red_I (no communication).
void shard_solve_local_impl(slablu_gpu_fact* F, const double* d_f, int64_t ldf, int64_t nrhs) {
  require_shard(F, "shard_solve_local");
  if (!F->swept) throw HostError(SLABLU_ERR_CONFIG, "shard_solve_local: factor with shard_eliminate + shard_sweep first");
  DeviceGuard dg(F->device);
  cudaStream_t st = F->stream;
  StreamScope scope(st);
  const int dev = F->device;
  const int64_t n2 = F->n2, N = F->N, Kn = (int64_t)F->K * n2;
  F->sh_nrhs = nrhs;
  F->sh_f.alloc(dev, (size_t)N * nrhs);
  copy2d(st, d_f, ldf, F->sh_f.p, N, N, nrhs);
  F->sh_red.alloc(dev, (size_t)std::max<int64_t>(Kn, 1) * nrhs);
  F->sh_red0.alloc(dev, (size_t)std::max<int64_t>(Kn, 1) * nrhs);
  F->sh_uifc.alloc(dev, (size_t)std::max<int64_t>(Kn, 1) * nrhs);
  F->sh_v.alloc(dev, (size_t)n2 * nrhs);
  SLB_CUDA_CHECK(cudaMemsetAsync(F->sh_uifc.p, 0, F->sh_uifc.bytes(), st));
  SLB_CUDA_CHECK(cudaMemsetAsync(F->sh_v.p, 0, F->sh_v.bytes(), st));
  {
    StripSweeper sw(F, F->sh_f.p, nrhs);
    reduce_phase(F, sw, F->sh_f.p, nrhs, F->sh_red.p, F->j0, F->j1);
  }
  copy2d(st, F->sh_red.p, Kn, F->sh_red0.p, Kn, Kn, nrhs);
  if (F->ib > F->ia) {  // z = A_I^{-1} red_I into uifc[ia, ib)
    SweepSolver ss(F, nrhs);
    ss.forward(F->sh_red.p, F->sh_uifc.p, F->ia, F->ib);
    ss.backward(F->sh_uifc.p, F->ia, F->ib, true);
  }
  SLB_CUDA_CHECK(cudaStreamSynchronize(st));
  F->sh_phase = 1;
}

// Separator forward step (rank order): q_in from r - 1, q_out to r + 1 (n2 x nrhs, ld n2):
//   v_r = S^_r^{-1} (red[j0] - super_{j0} z_ia + q_in),
//   q_out = red[j1] - sub_{ib-1} (z_{ib-1} - (A_I^{-1} E_L)_last v_r)     (L^ v folded in).
void shard_solve_fwd_impl(slablu_gpu_fact* F, const double* d_in, double* d_out) {
  require_shard(F, "shard_solve_forward");
  if (F->sh_phase != 1) throw HostError(SLABLU_ERR_CONFIG, "shard_solve_forward: call slablu_gpu_shard_solve_local first");
  if (F->has_left && !d_in) throw HostError(SLABLU_ERR_CONFIG, "shard_solve_forward: rank > 0 needs the message of rank - 1");
  if (F->has_right && !d_out)
    throw HostError(SLABLU_ERR_CONFIG, "shard_solve_forward: rank < nranks - 1 needs an output message buffer");
  DeviceGuard dg(F->device);
  cudaStream_t st = F->stream;
  StreamScope scope(st);
  const int dev = F->device;
  const int64_t n2 = F->n2, Kn = (int64_t)F->K * n2, bs = n2 * n2, nrhs = F->sh_nrhs;
  const int j0 = F->j0, j1 = F->j1, ia = F->ia, ib = F->ib;
  const bool interior = ib > ia;
  DBuf<double> part, t;
  part.alloc(dev, (size_t)8 * n2 * nrhs);
  t.alloc(dev, (size_t)n2 * nrhs);
  const double* red0 = F->sh_red0.p;
  const double* z = F->sh_uifc.p;
  if (F->has_left) {
    copy2d(st, red0 + (size_t)j0 * n2, Kn, t.p, n2, n2, nrhs);
    if (interior)
      dgemv_batched_rhs(st, n2, n2, nrhs, -1.0, F->Tsup() + (size_t)j0 * bs, n2, z + (size_t)ia * n2, Kn, 1.0, t.p, n2,
                        part.p);
    add2d(st, d_in, n2, t.p, n2, n2, nrhs, 1.0);
    SweepSolver ss(F, nrhs);
    ss.apply_Sinv(j0, t.p, n2, F->sh_v.p, n2, 1.0, 0.0);
  }
  if (F->has_right) {
    copy2d(st, red0 + (size_t)j1 * n2, Kn, d_out, n2, n2, nrhs);
    if (interior) {
      copy2d(st, z + (size_t)(ib - 1) * n2, Kn, t.p, n2, n2, nrhs);
      if (F->has_left)
        dgemv_batched_rhs(st, n2, n2, nrhs, -1.0, F->sh_yl.p, n2, F->sh_v.p, n2, 1.0, t.p, n2, part.p);
      dgemv_batched_rhs(st, n2, n2, nrhs, -1.0, F->Tsub() + (size_t)(ib - 1) * bs, n2, t.p, n2, 1.0, d_out, n2,
                        part.p);
    } else if (F->has_left) {  // adjacent separators: q = red[j1] - sub_{j0} v
      dgemv_batched_rhs(st, n2, n2, nrhs, -1.0, F->Tsub() + (size_t)j0 * bs, n2, F->sh_v.p, n2, 1.0, d_out, n2,
                        part.p);
    }
  }
  SLB_CUDA_CHECK(cudaGetLastError());
  SLB_CUDA_CHECK(cudaStreamSynchronize(st));
  F->sh_phase = 2;
}

// Separator backward step (reverse rank order) and the local finish: u_{s_r} = v_r + X^_r u_{s_{r+1}}
// (d_in = u_{s_{r+1}} from r + 1, d_out = u_{s_r} to r - 1), then the interior re-solved with the
// separator couplings on the right-hand side, recover_interiors (stage_one.hpp:438-462) on the local
// strips.  d_u (ld N) receives the shard's unknowns; every other entry is left untouched.
void shard_solve_bwd_impl(slablu_gpu_fact* F, const double* d_in, double* d_out, double* d_u, int64_t ldu) {
  require_shard(F, "shard_solve_backward");
  if (F->sh_phase != 2) throw HostError(SLABLU_ERR_CONFIG, "shard_solve_backward: call slablu_gpu_shard_solve_forward first");
  if (ldu != F->N) throw HostError(SLABLU_ERR_CONFIG, "shard_solve_backward: ldu must equal n1*n2");
  if (F->has_right && !d_in)
    throw HostError(SLABLU_ERR_CONFIG, "shard_solve_backward: rank < nranks - 1 needs u of interface j_end");
  if (F->has_left && !d_out) throw HostError(SLABLU_ERR_CONFIG, "shard_solve_backward: rank > 0 needs an output buffer");
  DeviceGuard dg(F->device);
  cudaStream_t st = F->stream;
  StreamScope scope(st);
  const int dev = F->device;
  const int64_t n2 = F->n2, Kn = (int64_t)F->K * n2, bs = n2 * n2, nrhs = F->sh_nrhs;
  const int j0 = F->j0, j1 = F->j1, ia = F->ia, ib = F->ib;
  double* uifc = F->sh_uifc.p;
  double* red = F->sh_red.p;
  DBuf<double> part;
  part.alloc(dev, (size_t)8 * n2 * nrhs);
  if (F->has_right) copy2d(st, d_in, n2, uifc + (size_t)j1 * n2, Kn, n2, nrhs);
  if (F->has_left) {
    copy2d(st, F->sh_v.p, n2, uifc + (size_t)j0 * n2, Kn, n2, nrhs);
    if (F->has_right)
      dgemv_batched_rhs(st, n2, n2, nrhs, 1.0, F->sh_xhat.p, n2, d_in, n2, 1.0, uifc + (size_t)j0 * n2, Kn, part.p);
    copy2d(st, uifc + (size_t)j0 * n2, Kn, d_out, n2, n2, nrhs);
  }
  if (ib > ia) {  // u_I = A_I^{-1} (red_I - E_L u_{s_r} - E_R u_{s_{r+1}})
    copy2d(st, F->sh_red0.p, Kn, red, Kn, Kn, nrhs);
    if (F->has_left)
      dgemv_batched_rhs(st, n2, n2, nrhs, -1.0, F->Tsub() + (size_t)j0 * bs, n2, uifc + (size_t)j0 * n2, Kn, 1.0,
                        red + (size_t)ia * n2, Kn, part.p);
    if (F->has_right)
      dgemv_batched_rhs(st, n2, n2, nrhs, -1.0, F->Tsup() + (size_t)(ib - 1) * bs, n2, uifc + (size_t)j1 * n2, Kn, 1.0,
                        red + (size_t)(ib - 1) * n2, Kn, part.p);
    SweepSolver ss(F, nrhs);
    ss.forward(red, uifc, ia, ib);
    ss.backward(uifc, ia, ib, true);
  }
  {
    StripSweeper sw(F, F->sh_f.p, nrhs);
    recover_phase(F, sw, uifc, nrhs, d_u, j0, j1);
  }
  SLB_CUDA_CHECK(cudaStreamSynchronize(st));
  check_solve_status(F);
  for (DBuf<double>* b : {&F->sh_f, &F->sh_red, &F->sh_red0, &F->sh_uifc, &F->sh_v}) b->release();
  F->sh_nrhs = 0;
  F->sh_phase = 0;
}

void solve_impl(const slablu_gpu_fact* F, const double* d_f, int64_t ldf, int64_t nrhs, double* d_u, int64_t ldu) {
  if (F->stage2_only)
    throw HostError(SLABLU_ERR_CONFIG, "solve: a sweep_build handle holds stage two only, use slablu_gpu_sweep_solve");
  if (F->sharded)
    throw HostError(SLABLU_ERR_CONFIG, "solve: sharded factorization, use slablu_gpu_shard_solve_forward/backward");
  std::lock_guard<std::mutex> guard(F->solve_mu);
  DeviceGuard dg(F->device);
  cudaStream_t st = F->stream;
  StreamScope scope(st);
  const int dev = F->device;
  const int64_t N = F->N;
  cudaEvent_t e0, e1;
  SLB_CUDA_CHECK(cudaEventCreate(&e0));
  SLB_CUDA_CHECK(cudaEventCreate(&e1));
  SLB_CUDA_CHECK(cudaEventRecord(e0, st));
  const int64_t l0 = slb::g_kernel_count.load();
  if (F->refine == 0 || !F->a_rp.p) {
    solve_once(F, d_f, ldf, nrhs, d_u, ldu);
  } else {
    DBuf<double> f, u, r, du;
    f.alloc(dev, (size_t)N * nrhs);
    u.alloc(dev, (size_t)N * nrhs);
    r.alloc(dev, (size_t)N * nrhs);
    du.alloc(dev, (size_t)N * nrhs);
    copy2d(st, d_f, ldf, f.p, N, N, nrhs);
    solve_once(F, f.p, N, nrhs, u.p, N);
    double t_strips = F->t_solve_strips;
    const unsigned gb = (unsigned)cdiv(N * nrhs, 256);
    for (int it = 0; it < F->refine; it++) {
      residual_kernel<<<gb, 256, 0, st>>>(F->a_rp.p, F->a_ci.p, F->a_v.p, N, nrhs, f.p, u.p, r.p); count_launch();
      SLB_CUDA_CHECK(cudaGetLastError());
      solve_once(F, r.p, N, nrhs, du.p, N);
      t_strips += F->t_solve_strips;
      axpy_kernel<<<gb, 256, 0, st>>>(N * nrhs, du.p, u.p); count_launch();
      SLB_CUDA_CHECK(cudaGetLastError());
    }
    copy2d(st, u.p, N, d_u, ldu, N, nrhs);
    F->t_solve_strips = t_strips;
  }
  SLB_CUDA_CHECK(cudaEventRecord(e1, st));
  SLB_CUDA_CHECK(cudaEventSynchronize(e1));
  float ms = 0;
  SLB_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
  F->t_solve = ms * 1e-3;
  F->launches_solve = slb::g_kernel_count.load() - l0;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  check_solve_status(F);
}

slablu_gpu_status status_from(const HostError& e) { return make_status(e.code, e.what(), e.index, e.residual); }
slablu_gpu_status status_from(const CudaFailure& e) {
  const int code = e.err == cudaErrorMemoryAllocation ? SLABLU_ERR_OOM : SLABLU_ERR_CUDA;
  return make_status(code, std::string("CUDA error: ") + cudaGetErrorString(e.err) + " at " + e.file + ":" +
                               std::to_string(e.line) + " (" + e.expr + ")", -1);
}

#define ABI_TRY(...)                                   \
  try {                                                \
    __VA_ARGS__;                                       \
    return make_status(SLABLU_OK, "", -1);             \
  } catch (const HostError& e) {                       \
    return status_from(e);                             \
  } catch (const CudaFailure& e) {                     \
    return status_from(e);                             \
  } catch (const std::bad_alloc&) {                    \
    return make_status(SLABLU_ERR_OOM, "host allocation failed", -1); \
  }

void require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw HostError(SLABLU_ERR_CUDA, "no CUDA device available (the engine has no CPU fallback)");
  }
}

}  // namespace

extern "C" {

int slablu_gpu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

slablu_gpu_status slablu_gpu_factorize(int64_t n1, int64_t n2, const int32_t* row_ptr, const int32_t* col_idx,
                                       const double* val, const slablu_gpu_config* config, slablu_gpu_fact** out) {
  ABI_TRY({
    require_device();
    *out = nullptr;
    const int dev = (int)cfg_device(config);
    SLB_CUDA_CHECK(cudaSetDevice(dev));
    const int64_t n = n1 * n2;
    if (n == 0) throw HostError(SLABLU_ERR_CONFIG, "factorize: empty system");
    const int64_t nnz = row_ptr[n];
    DBuf<int32_t> rp, ci;
    DBuf<double> v;
    rp.alloc(dev, n + 1);
    ci.alloc(dev, nnz);
    v.alloc(dev, nnz);
    SLB_CUDA_CHECK(cudaMemcpy(rp.p, row_ptr, (n + 1) * sizeof(int32_t), cudaMemcpyHostToDevice));
    SLB_CUDA_CHECK(cudaMemcpy(ci.p, col_idx, nnz * sizeof(int32_t), cudaMemcpyHostToDevice));
    SLB_CUDA_CHECK(cudaMemcpy(v.p, val, nnz * sizeof(double), cudaMemcpyHostToDevice));
    *out = factorize_impl(n1, n2, nnz, rp.p, ci.p, v.p, config);
  })
}

slablu_gpu_status slablu_gpu_factorize_device(int64_t n1, int64_t n2, int64_t nnz, const int32_t* d_row_ptr,
                                              const int32_t* d_col_idx, const double* d_val,
                                              const slablu_gpu_config* config, slablu_gpu_fact** out) {
  ABI_TRY({
    require_device();
    *out = nullptr;
    *out = factorize_impl(n1, n2, nnz, d_row_ptr, d_col_idx, d_val, config);
  })
}

slablu_gpu_status slablu_gpu_shard_plan(int64_t n1, int64_t n2, int64_t b, int rank, int nranks,
                                        slablu_gpu_shard_t* out) {
  ABI_TRY({
    if (nranks < 1 || rank < 0 || rank >= nranks) throw HostError(SLABLU_ERR_CONFIG, "shard_plan: bad rank/nranks");
    if (b > n1 - 2 || n1 < 3) throw HostError(SLABLU_ERR_CONFIG, "shard_plan: the single-slab path does not shard");
    Partition p = partition(n1, n2, b);
    const int Sg = (int)p.interiors.size(), K = (int)p.interfaces.size();
    if (Sg < nranks) throw HostError(SLABLU_ERR_CONFIG, "shard_plan: fewer strips than ranks");
    int s0, s1, j0, j1;
    shard_ranges(Sg, K, rank, nranks, &s0, &s1, &j0, &j1);
    *out = slablu_gpu_shard_t{rank, nranks, s0, s1, j0, j1, Sg, K};
  })
}

slablu_gpu_status slablu_gpu_shard_factorize_device(int64_t n1, int64_t n2, int64_t nnz, const int32_t* d_row_ptr,
                                                    const int32_t* d_col_idx, const double* d_val,
                                                    const slablu_gpu_config* config, int rank, int nranks,
                                                    slablu_gpu_fact** out) {
  ABI_TRY({
    require_device();
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks) throw HostError(SLABLU_ERR_CONFIG, "shard_factorize: bad rank/nranks");
    slablu_gpu_config c{};
    c.c = 0.6;
    if (config) c = *config;
    // refine > 0 keeps a copy of the CSR for slablu_gpu_residual (host-driven refinement)
    *out = factorize_impl(n1, n2, nnz, d_row_ptr, d_col_idx, d_val, &c, rank, nranks, true);
  })
}

slablu_gpu_status slablu_gpu_residual(const slablu_gpu_fact* fact, const double* d_f, int64_t ldf, int64_t nrhs,
                                     const double* d_u, int64_t ldu, double* d_r) {
  ABI_TRY({
    if (!fact) throw HostError(SLABLU_ERR_GENERIC, "residual: null factorization");
    if (!fact->a_rp.p) throw HostError(SLABLU_ERR_CONFIG, "residual: factorize with config.refine > 0 to keep the operator");
    if (ldf != fact->N || ldu != fact->N || nrhs < 1) throw HostError(SLABLU_ERR_GENERIC, "residual: ld must equal n1*n2");
    DeviceGuard dg(fact->device);
    const int64_t N = fact->N;
    residual_kernel<<<(unsigned)cdiv(N * nrhs, 256), 256, 0, fact->stream>>>(fact->a_rp.p, fact->a_ci.p, fact->a_v.p, N,
                                                                         nrhs, d_f, d_u, d_r); count_launch();
    SLB_CUDA_CHECK(cudaGetLastError());
    SLB_CUDA_CHECK(cudaStreamSynchronize(fact->stream));
  })
}

slablu_gpu_status slablu_gpu_shard_eliminate(slablu_gpu_fact* fact) {
  ABI_TRY({
    if (!fact) throw HostError(SLABLU_ERR_GENERIC, "shard_eliminate: null factorization");
    shard_eliminate_impl(fact);
  })
}

slablu_gpu_status slablu_gpu_shard_solve_local(slablu_gpu_fact* fact, const double* d_f, int64_t ldf, int64_t nrhs) {
  ABI_TRY({
    if (!fact) throw HostError(SLABLU_ERR_GENERIC, "shard_solve_local: null factorization");
    if (nrhs < 1 || ldf < fact->N) throw HostError(SLABLU_ERR_GENERIC, "shard_solve_local: bad rhs shape");
    shard_solve_local_impl(fact, d_f, ldf, nrhs);
  })
}

slablu_gpu_status slablu_gpu_shard_sweep(slablu_gpu_fact* fact, const double* d_in, double* d_out) {
  ABI_TRY({
    if (!fact) throw HostError(SLABLU_ERR_GENERIC, "shard_sweep: null factorization");
    shard_sweep_impl(fact, d_in, d_out);
  })
}

slablu_gpu_status slablu_gpu_shard_solve_forward(slablu_gpu_fact* fact, const double* d_in, double* d_out) {
  ABI_TRY({
    if (!fact) throw HostError(SLABLU_ERR_GENERIC, "shard_solve_forward: null factorization");
    shard_solve_fwd_impl(fact, d_in, d_out);
  })
}

slablu_gpu_status slablu_gpu_shard_solve_backward(slablu_gpu_fact* fact, const double* d_in, double* d_out,
                                                  double* d_u, int64_t ldu) {
  ABI_TRY({
    if (!fact) throw HostError(SLABLU_ERR_GENERIC, "shard_solve_backward: null factorization");
    shard_solve_bwd_impl(fact, d_in, d_out, d_u, ldu);
  })
}

slablu_gpu_status slablu_gpu_solve(const slablu_gpu_fact* fact, const double* f, int64_t ldf, int64_t nrhs,
                                   double* u, int64_t ldu) {
  ABI_TRY({
    if (!fact) throw HostError(SLABLU_ERR_GENERIC, "solve: null factorization");
    if (nrhs < 0 || ldf < fact->N || ldu < fact->N)
      throw HostError(SLABLU_ERR_GENERIC, "solve: rhs length must equal the grid size");
    if (nrhs == 0) return make_status(SLABLU_OK, "", -1);
    DeviceGuard dg(fact->device);
    const int64_t N = fact->N;
    DBuf<double> df, du;
    df.alloc(fact->device, (size_t)N * nrhs);
    du.alloc(fact->device, (size_t)N * nrhs);
    SLB_CUDA_CHECK(cudaMemcpy2DAsync(df.p, N * sizeof(double), f, ldf * sizeof(double), N * sizeof(double), nrhs,
                                     cudaMemcpyHostToDevice, fact->stream));
    solve_impl(fact, df.p, N, nrhs, du.p, N);
    SLB_CUDA_CHECK(cudaMemcpy2DAsync(u, ldu * sizeof(double), du.p, N * sizeof(double), N * sizeof(double), nrhs,
                                     cudaMemcpyDeviceToHost, fact->stream));
    SLB_CUDA_CHECK(cudaStreamSynchronize(fact->stream));
  })
}

slablu_gpu_status slablu_gpu_solve_device(const slablu_gpu_fact* fact, const double* d_f, int64_t ldf, int64_t nrhs,
                                          double* d_u, int64_t ldu) {
  ABI_TRY({
    if (!fact) throw HostError(SLABLU_ERR_GENERIC, "solve: null factorization");
    if (nrhs < 0 || ldf < fact->N || ldu < fact->N)
      throw HostError(SLABLU_ERR_GENERIC, "solve: rhs length must equal the grid size");
    if (nrhs == 0) return make_status(SLABLU_OK, "", -1);
    solve_impl(fact, d_f, ldf, nrhs, d_u, ldu);
  })
}

slablu_gpu_status slablu_gpu_stats(const slablu_gpu_fact* F, slablu_gpu_stats_t* o) {
  ABI_TRY({
    if (!F) throw HostError(SLABLU_ERR_GENERIC, "stats: null factorization");
    o->n1 = F->n1;
    o->n2 = F->n2;
    o->b = F->b;
    o->interfaces = F->K;
    o->strips = F->S;
    o->padded_width = F->Wp;
    o->single_slab = F->single ? 1 : 0;
    o->symmetric_strips = 0;
    for (int v : F->sym_h) o->symmetric_strips += v ? 1 : 0;
    o->t_stage1 = F->t1;
    o->t_stage2 = F->t2;
    o->storage_stage1 = F->storage1;
    o->storage_stage2 = F->storage2;
    o->device_bytes = (int64_t)(F->fac.bytes() + F->perm.bytes() + F->cpl.bytes() + F->T.bytes() + F->Tkeep.bytes() +
                                F->Xup.bytes());
    o->gpu_launches = F->launches_factor;
    o->solve_launches = F->launches_solve;
    o->t_chain = F->t_chain;
    o->t_schur = F->t_schur;
    o->t_assemble = F->t_asm;
    o->compression = F->compression;
    o->hbs_max_rank = F->hbs_max_rank;
    o->t_hbs = F->t_hbs;
    o->t_solve_last = F->t_solve;
    o->t_solve_strips = F->t_solve_strips;
  })
}

slablu_gpu_status slablu_gpu_set_refine(slablu_gpu_fact* F, int refine) {
  ABI_TRY({
    if (!F) throw HostError(SLABLU_ERR_GENERIC, "set_refine: null factorization");
    if (refine < 0) throw HostError(SLABLU_ERR_CONFIG, "set_refine: refine must be nonnegative");
    if (refine > 0 && !F->a_rp.p)
      throw HostError(SLABLU_ERR_CONFIG, "set_refine: factorize with config.refine > 0 to keep the operator");
    std::lock_guard<std::mutex> guard(F->solve_mu);
    F->refine = refine;
  })
}

slablu_gpu_status slablu_gpu_T_block(const slablu_gpu_fact* F, int which, int64_t j, double* out) {
  ABI_TRY({
    if (!F || !F->Tkeep.p) throw HostError(SLABLU_ERR_GENERIC, "T_block: factorization was not built with keep_T");
    const int64_t nb = which == 0 ? F->K : F->K - 1;
    if (j < 0 || j >= nb || which < 0 || which > 2) throw HostError(SLABLU_ERR_GENERIC, "T_block: index out of range");
    const int64_t base = which == 0 ? j : which == 1 ? F->K + j : 2 * F->K - 1 + j;
    DeviceGuard dg(F->device);
    SLB_CUDA_CHECK(cudaMemcpy(out, F->Tkeep.p + base * F->n2 * F->n2, F->n2 * F->n2 * sizeof(double),
                              cudaMemcpyDeviceToHost));
  })
}

slablu_gpu_status slablu_gpu_reduce_rhs(const slablu_gpu_fact* F, const double* f, int64_t nrhs, double* out) {
  ABI_TRY({
    if (!F || F->single || F->stage2_only) throw HostError(SLABLU_ERR_GENERIC, "reduce_rhs: no partition");
    if (F->sharded) throw HostError(SLABLU_ERR_CONFIG, "reduce_rhs: sharded factorization");
    if (nrhs < 1) throw HostError(SLABLU_ERR_GENERIC, "reduce_rhs: nrhs must be positive");
    std::lock_guard<std::mutex> guard(F->solve_mu);
    DeviceGuard dg(F->device);
    StreamScope scope(F->stream);
    const int64_t N = F->N, Kn = (int64_t)F->K * F->n2;
    DBuf<double> df, red;
    df.alloc(F->device, (size_t)N * nrhs);
    red.alloc(F->device, (size_t)Kn * nrhs);
    SLB_CUDA_CHECK(cudaMemcpyAsync(df.p, f, N * nrhs * sizeof(double), cudaMemcpyHostToDevice, F->stream));
    StripSweeper sw(F, df.p, nrhs);  // the solve's own dispatch (cluster sweeps for nrhs <= 8)
    reduce_phase(F, sw, df.p, nrhs, red.p, 0, F->K);
    SLB_CUDA_CHECK(cudaMemcpyAsync(out, red.p, Kn * nrhs * sizeof(double), cudaMemcpyDeviceToHost, F->stream));
    SLB_CUDA_CHECK(cudaStreamSynchronize(F->stream));
  })
}

slablu_gpu_status slablu_gpu_sweep_solve(const slablu_gpu_fact* F, const double* red, int64_t nrhs, double* u_ifc) {
  ABI_TRY({
    if (!F || F->single) throw HostError(SLABLU_ERR_GENERIC, "sweep_solve: no partition");
    if (F->sharded) throw HostError(SLABLU_ERR_CONFIG, "sweep_solve: sharded factorization");
    if (nrhs < 1) throw HostError(SLABLU_ERR_GENERIC, "sweep_solve: nrhs must be positive");
    std::lock_guard<std::mutex> guard(F->solve_mu);
    DeviceGuard dg(F->device);
    StreamScope scope(F->stream);
    const int64_t Kn = (int64_t)F->K * F->n2;
    DBuf<double> r, u;
    r.alloc(F->device, (size_t)Kn * nrhs);
    u.alloc(F->device, (size_t)Kn * nrhs);
    SLB_CUDA_CHECK(cudaMemcpyAsync(r.p, red, Kn * nrhs * sizeof(double), cudaMemcpyHostToDevice, F->stream));
    SweepSolver ss(F, nrhs);
    ss.forward(r.p, u.p, 0, F->K);
    ss.backward(u.p, 0, F->K);
    SLB_CUDA_CHECK(cudaMemcpyAsync(u_ifc, u.p, Kn * nrhs * sizeof(double), cudaMemcpyDeviceToHost, F->stream));
    SLB_CUDA_CHECK(cudaStreamSynchronize(F->stream));
    check_solve_status(F);
  })
}

// sweep_build (stage_two.hpp:131-150, validate :41-56) on a caller-supplied block-tridiagonal
// system: blocks = [diag 0..k-1 | super 0..k-2 | sub 0..k-2], each m x m column major (host).
slablu_gpu_status slablu_gpu_hbs_compress(int64_t n, const double* m, int64_t leaf_size, int64_t r_start,
                                          int64_t r_max, int adaptive, double tol, double trunc_rel,
                                          uint64_t seed, int device, double* out, slablu_gpu_hbs_stats* stats) {
  ABI_TRY({
    require_device();
    if (n < 1 || !m || !out) throw HostError(SLABLU_ERR_CONFIG, "hbs_compress: empty operator");
    if (leaf_size < 1 || leaf_size > n) throw HostError(SLABLU_ERR_CONFIG, "ClusterTree: need 1 <= leaf_size <= n");
    DeviceGuard dg(device);
    cudaStream_t st;
    SLB_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    StreamScope scope(st);
    HbsOptions o;
    o.tol = tol;
    o.trunc_rel = trunc_rel;
    o.leaf = (int)leaf_size;
    o.r_start = r_start;
    o.r_max = r_max;
    o.fixed_rank = adaptive == 0;
    HbsStats hs;
    double* d = nullptr;
    try {
      SLB_CUDA_CHECK(cudaMalloc(&d, (size_t)n * n * sizeof(double)));
      SLB_CUDA_CHECK(cudaMemcpyAsync(d, m, (size_t)n * n * sizeof(double), cudaMemcpyHostToDevice, st));
      hbs_compress_blocks(st, n, 1, &d, &seed, o, &hs);
      SLB_CUDA_CHECK(cudaMemcpyAsync(out, d, (size_t)n * n * sizeof(double), cudaMemcpyDeviceToHost, st));
      SLB_CUDA_CHECK(cudaStreamSynchronize(st));
    } catch (const HostError& e) {
      if (stats) {
        stats->residual_estimate = e.residual;
      }
      cudaFree(d);
      cudaStreamDestroy(st);
      HostError w(e.code, e.what(), -1);
      w.residual = e.residual;
      throw w;
    } catch (...) {
      cudaFree(d);
      cudaStreamDestroy(st);
      throw;
    }
    cudaFree(d);
    cudaStreamDestroy(st);
    if (stats) {
      stats->products_normal = hs.products_normal;
      stats->products_adjoint = hs.products_adjoint;
      stats->rounds = hs.rounds;
      stats->final_rank = hs.final_rank;
      stats->residual_estimate = hs.residual;
    }
  });
}

slablu_gpu_status slablu_gpu_sweep_build(int64_t m, int64_t k, const double* blocks, int device,
                                         slablu_gpu_fact** out) {
  ABI_TRY({
    require_device();
    *out = nullptr;
    if (k < 1) throw HostError(SLABLU_ERR_CONFIG, "BlockTridiagonal: no blocks");
    if (m < 1) throw HostError(SLABLU_ERR_CONFIG, "BlockTridiagonal: inconsistent block dimensions");
    if (m > kMaxIfc)
      throw HostError(SLABLU_ERR_UNSUPPORTED, "sweep_build: block dimension exceeds the engine's envelope");
    auto F = std::make_unique<slablu_gpu_fact>();
    F->device = device;
    DeviceGuard dg(device);
    SLB_CUDA_CHECK(cudaStreamCreateWithFlags(&F->stream, cudaStreamNonBlocking));
    cudaStream_t st = F->stream;
    StreamScope scope(st);
    F->stage2_only = true;
    F->n1 = k;
    F->n2 = m;
    F->N = k * m;
    F->K = (int)k;
    F->status.alloc(device, 1);
    F->sstatus.alloc(device, 1);
    static const DevStatus st0{0, INT_MAX, INT_MAX, INT_MAX};
    SLB_CUDA_CHECK(cudaMemcpyAsync(F->status.p, &st0, sizeof(DevStatus), cudaMemcpyHostToDevice, st));
    SLB_CUDA_CHECK(cudaMemcpyAsync(F->sstatus.p, &st0, sizeof(DevStatus), cudaMemcpyHostToDevice, st));
    const int64_t nb = 3 * k - 2;
    F->T.alloc(device, (size_t)nb * m * m);
    SLB_CUDA_CHECK(cudaMemcpyAsync(F->T.p, blocks, (size_t)nb * m * m * sizeof(double), cudaMemcpyHostToDevice, st));
    check_finite(st, F->T.p, nb * m * m, F->status.p);
    DevStatus hs;
    SLB_CUDA_CHECK(cudaMemcpyAsync(&hs, F->status.p, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
    SLB_CUDA_CHECK(cudaStreamSynchronize(st));
    if (hs.flags & ERR_NONFINITE) throw HostError(SLABLU_ERR_GENERIC, "BlockTridiagonal: non-finite block entry");
    cudaEvent_t e0, e1;
    SLB_CUDA_CHECK(cudaEventCreate(&e0));
    SLB_CUDA_CHECK(cudaEventCreate(&e1));
    SLB_CUDA_CHECK(cudaEventRecord(e0, st));
    const int64_t l0 = slb::g_kernel_count.load();
    stage_two_build(F.get());
    SLB_CUDA_CHECK(cudaEventRecord(e1, st));
    SLB_CUDA_CHECK(cudaEventSynchronize(e1));
    float ms = 0;
    SLB_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    F->t2 = ms * 1e-3;
    F->launches_factor = slb::g_kernel_count.load() - l0;
    F->storage2 = (k + 2 * (k - 1)) * m * m;
    SLB_CUDA_CHECK(cudaMemcpy(&hs, F->status.p, sizeof(DevStatus), cudaMemcpyDeviceToHost));
    if (hs.flags & ERR_SINGULAR)
      throw HostError(SLABLU_ERR_SINGULAR, "sweep_build: singular Schur complement block", hs.singular_block);
    *out = F.release();
  })
}

slablu_gpu_status slablu_gpu_recover(const slablu_gpu_fact* F, const double* f, const double* u_ifc, int64_t nrhs,
                                     double* u) {
  ABI_TRY({
    if (!F || F->single || F->stage2_only) throw HostError(SLABLU_ERR_GENERIC, "recover: no partition");
    if (F->sharded) throw HostError(SLABLU_ERR_CONFIG, "recover: sharded factorization");
    if (nrhs < 1) throw HostError(SLABLU_ERR_GENERIC, "recover: nrhs must be positive");
    std::lock_guard<std::mutex> guard(F->solve_mu);
    DeviceGuard dg(F->device);
    StreamScope scope(F->stream);
    const int64_t N = F->N, Kn = (int64_t)F->K * F->n2;
    DBuf<double> df, du, dui;
    df.alloc(F->device, (size_t)N * nrhs);
    du.alloc(F->device, (size_t)N * nrhs);
    dui.alloc(F->device, (size_t)Kn * nrhs);
    SLB_CUDA_CHECK(cudaMemcpyAsync(df.p, f, N * nrhs * sizeof(double), cudaMemcpyHostToDevice, F->stream));
    SLB_CUDA_CHECK(cudaMemcpyAsync(dui.p, u_ifc, Kn * nrhs * sizeof(double), cudaMemcpyHostToDevice, F->stream));
    StripSweeper sw(F, df.p, nrhs);
    recover_phase(F, sw, dui.p, nrhs, du.p, 0, F->K);
    SLB_CUDA_CHECK(cudaMemcpyAsync(u, du.p, N * nrhs * sizeof(double), cudaMemcpyDeviceToHost, F->stream));
    SLB_CUDA_CHECK(cudaStreamSynchronize(F->stream));
  })
}

// Micro-benchmark of the stage-two building blocks at block size n (device
// time, CUDA events): out[0] GEMM n^3, out[1] getrf, out[2] inverse via getrs(I).
int slablu_gpu_debug_dense_bench(int64_t n, int device, double* out) {
  try {
    SLB_CUDA_CHECK(cudaSetDevice(device));
    cudaStream_t st;
    SLB_CUDA_CHECK(cudaStreamCreate(&st));
    DBuf<double> A, B, C;
    DBuf<int32_t> ipiv;
    DBuf<DevStatus> status;
    A.alloc(device, n * n);
    B.alloc(device, n * n);
    C.alloc(device, n * n);
    ipiv.alloc(device, n);
    status.alloc(device, 1);
    DevStatus st0{0, INT_MAX, INT_MAX, INT_MAX};
    SLB_CUDA_CHECK(cudaMemcpy(status.p, &st0, sizeof(st0), cudaMemcpyHostToDevice));
    std::vector<double> h(n * n);
    uint64_t x = 88172645463325252ULL;
    for (auto& v : h) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      v = (double)(x >> 11) / 9007199254740992.0 - 0.5;
    }
    for (int64_t i = 0; i < n; i++) h[i * n + i] += 0.0;  // general (pivoting exercised)
    SLB_CUDA_CHECK(cudaMemcpy(A.p, h.data(), n * n * sizeof(double), cudaMemcpyHostToDevice));
    SLB_CUDA_CHECK(cudaMemcpy(B.p, h.data(), n * n * sizeof(double), cudaMemcpyHostToDevice));
    cudaEvent_t ev[4];
    for (auto& e0 : ev) SLB_CUDA_CHECK(cudaEventCreate(&e0));
    SLB_CUDA_CHECK(cudaEventRecord(ev[0], st));
    dgemm_batched(st, n, n, n, 1.0, A.p, n, 0, B.p, n, 0, 0.0, C.p, n, 0, 1);
    SLB_CUDA_CHECK(cudaEventRecord(ev[1], st));
    dgetrf(st, n, A.p, ipiv.p, nullptr, status.p, 0);
    SLB_CUDA_CHECK(cudaEventRecord(ev[2], st));
    dset_identity(st, B.p, n);
    dgetrs(st, n, n, A.p, ipiv.p, B.p, n, nullptr);
    SLB_CUDA_CHECK(cudaEventRecord(ev[3], st));
    SLB_CUDA_CHECK(cudaEventSynchronize(ev[3]));
    float ms;
    for (int i = 0; i < 3; i++) {
      SLB_CUDA_CHECK(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
      out[i] = ms * 1e-3;
    }
    for (auto& e0 : ev) cudaEventDestroy(e0);
    cudaStreamDestroy(st);
    return 0;
  } catch (const CudaFailure& f) {
    fprintf(stderr, "debug_dense_bench: %s at %s:%d (%s)\n", cudaGetErrorString(f.err), f.file, f.line, f.expr);
    return 1;
  } catch (...) {
    return 1;
  }
}

// Test hook for the stage-two solve kernel: LU-factor the n x n column-major a (host),
// then x = A^{-1} b (n x nrhs, host) through getrs_chain.
// t_out[0] = average device seconds per getrs over `reps` calls.
int slablu_gpu_debug_getrs(int64_t n, int64_t nrhs, const double* a, const double* b, double* x, int reps,
                           int device, double* t_out) {
  try {
    SLB_CUDA_CHECK(cudaSetDevice(device));
    cudaStream_t st;
    SLB_CUDA_CHECK(cudaStreamCreate(&st));
    const int64_t dinv_sz = cdiv(n, 64) * 2 * 64 * 64;
    DBuf<double> A, B, X, D, yz;
    DBuf<int32_t> ipiv, perm;
    DBuf<DevStatus> status;
    A.alloc(device, n * n);
    B.alloc(device, n * nrhs);
    X.alloc(device, n * nrhs);
    D.alloc(device, dinv_sz);
    yz.alloc(device, getrs_chain_scratch(n, nrhs));
    ipiv.alloc(device, n);
    perm.alloc(device, n);
    status.alloc(device, 1);
    DevStatus st0{0, INT_MAX, INT_MAX, INT_MAX};
    SLB_CUDA_CHECK(cudaMemcpy(status.p, &st0, sizeof(st0), cudaMemcpyHostToDevice));
    SLB_CUDA_CHECK(cudaMemcpy(A.p, a, n * n * sizeof(double), cudaMemcpyHostToDevice));
    SLB_CUDA_CHECK(cudaMemcpy(B.p, b, n * nrhs * sizeof(double), cudaMemcpyHostToDevice));
    getrs_chain_init(st, n, nrhs, yz.p);
    dgetrf(st, n, A.p, ipiv.p, nullptr, status.p, 0);
    getrs_prepare(st, n, A.p, ipiv.p, perm.p, D.p);
    cudaEvent_t e0, e1;
    SLB_CUDA_CHECK(cudaEventCreate(&e0));
    SLB_CUDA_CHECK(cudaEventCreate(&e1));
    int epoch = 0;
    reps = std::max(reps, 1);
    SLB_CUDA_CHECK(cudaEventRecord(e0, st));
    for (int r = 0; r < reps; r++) {
      getrs_chain(st, n, nrhs, A.p, D.p, perm.p, B.p, n, X.p, n, 1.0, 0.0, yz.p, ++epoch, status.p);
    }
    SLB_CUDA_CHECK(cudaEventRecord(e1, st));
    SLB_CUDA_CHECK(cudaEventSynchronize(e1));
    float ms;
    SLB_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
    if (t_out) t_out[0] = ms * 1e-3 / reps;
    SLB_CUDA_CHECK(cudaMemcpy(x, X.p, n * nrhs * sizeof(double), cudaMemcpyDeviceToHost));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(st);
    return 0;
  } catch (const CudaFailure& f) {
    fprintf(stderr, "debug_getrs: %s at %s:%d (%s)\n", cudaGetErrorString(f.err), f.file, f.line, f.expr);
    return 1;
  } catch (...) {
    return 1;
  }
}

void slablu_gpu_destroy(slablu_gpu_fact* fact) {
  if (!fact) return;
  try {
    delete fact;
  } catch (...) {
  }
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Factor caching (the reference serializes each factor object in a versioned
// binary layout: stage_two.hpp:95-120, 200-232, dense.hpp:71-87, banded.hpp:133-163).
//   SLBGPU01  the whole GPU factorization (level operators, couplings, reduced blocks in LU form,
//             the block upper factor, optional operator copy), for factor-once-solve-many across
//             processes: named sections, each u64 name length, name, u64 bytes, raw bytes.
//   SLBSWP01  stage two in the reference's own SweepFactorization layout (k DenseLU blocks as
//             write_dense + int64 1-based pivots, then sub and super blocks), so a factorization
//             made on the GPU loads into the reference and vice versa.
namespace {

constexpr size_t kStage = 64u << 20;  // pinned staging bytes per copy step

struct Pinned {
  void* p = nullptr;
  explicit Pinned(size_t bytes) { SLB_CUDA_CHECK(cudaMallocHost(&p, bytes)); }
  ~Pinned() {
    if (p) cudaFreeHost(p);
  }
};

void write_u64(std::ostream& os, uint64_t v) { os.write(reinterpret_cast<const char*>(&v), sizeof(v)); }
uint64_t read_u64(std::istream& is) {
  uint64_t v = 0;
  is.read(reinterpret_cast<char*>(&v), sizeof(v));
  if (!is) throw HostError(SLABLU_ERR_GENERIC, "deserialize: truncated stream");
  return v;
}
void write_dev(std::ostream& os, const void* d, size_t bytes, Pinned& stage) {
  for (size_t o = 0; o < bytes; o += kStage) {
    const size_t n = std::min(kStage, bytes - o);
    SLB_CUDA_CHECK(cudaMemcpy(stage.p, static_cast<const char*>(d) + o, n, cudaMemcpyDeviceToHost));
    os.write(static_cast<const char*>(stage.p), (std::streamsize)n);
  }
}
void read_dev(std::istream& is, void* d, size_t bytes, Pinned& stage) {
  for (size_t o = 0; o < bytes; o += kStage) {
    const size_t n = std::min(kStage, bytes - o);
    is.read(static_cast<char*>(stage.p), (std::streamsize)n);
    if (!is) throw HostError(SLABLU_ERR_GENERIC, "deserialize: truncated stream");
    SLB_CUDA_CHECK(cudaMemcpy(static_cast<char*>(d) + o, stage.p, n, cudaMemcpyHostToDevice));
  }
}
void write_section(std::ostream& os, const char* name, const void* data, size_t bytes, bool device, Pinned& stage) {
  const size_t ln = strlen(name);
  write_u64(os, ln);
  os.write(name, (std::streamsize)ln);
  write_u64(os, bytes);
  if (device) write_dev(os, data, bytes, stage);
  else os.write(static_cast<const char*>(data), (std::streamsize)bytes);
}
// reads the next section, which must be `name`; returns its byte count (payload left unread)
uint64_t open_section(std::istream& is, const char* name) {
  const uint64_t ln = read_u64(is);
  if (ln > 64) throw HostError(SLABLU_ERR_GENERIC, "deserialize: corrupt section header");
  std::string got(ln, '\0');
  is.read(&got[0], (std::streamsize)ln);
  if (!is || got != name) throw HostError(SLABLU_ERR_GENERIC, std::string("deserialize: expected section ") + name);
  return read_u64(is);
}
template <class T>
void read_section_dev(std::istream& is, const char* name, DBuf<T>& buf, int dev, Pinned& stage) {
  const uint64_t bytes = open_section(is, name);
  if (bytes % sizeof(T)) throw HostError(SLABLU_ERR_GENERIC, "deserialize: section size");
  buf.release();
  if (bytes) {
    buf.alloc(dev, bytes / sizeof(T));
    read_dev(is, buf.p, bytes, stage);
  }
}
template <class T>
void read_section_host(std::istream& is, const char* name, std::vector<T>& v) {
  const uint64_t bytes = open_section(is, name);
  if (bytes % sizeof(T)) throw HostError(SLABLU_ERR_GENERIC, "deserialize: section size");
  v.resize(bytes / sizeof(T));
  is.read(reinterpret_cast<char*>(v.data()), (std::streamsize)bytes);
  if (!is) throw HostError(SLABLU_ERR_GENERIC, "deserialize: truncated stream");
}

const char kMagicGpu[9] = "SLBGPU01";
const char kMagicSwp[9] = "SLBSWP01";

void save_impl(const slablu_gpu_fact* F, const char* path) {
  if (F->sharded) throw HostError(SLABLU_ERR_CONFIG, "save: sharded factorizations are saved per rank (not supported)");
  std::lock_guard<std::mutex> guard(F->solve_mu);
  DeviceGuard dg(F->device);
  SLB_CUDA_CHECK(cudaStreamSynchronize(F->stream));
  std::ofstream os(path, std::ios::binary | std::ios::trunc);
  if (!os) throw HostError(SLABLU_ERR_GENERIC, std::string("save: cannot open ") + path);
  Pinned stage(kStage);
  os.write(kMagicGpu, 8);
  const int64_t hdr[12] = {F->n1, F->n2, F->b, F->S, F->K, F->Wp, F->single ? 1 : 0, F->stage2_only ? 1 : 0,
                           F->refine, F->storage1, F->storage2, F->sF};
  write_section(os, "header", hdr, sizeof(hdr), false, stage);
  const double times[5] = {F->t1, F->t2, F->t_chain, F->t_schur, F->t_asm};
  write_section(os, "times", times, sizeof(times), false, stage);
  write_section(os, "strips_h", F->strips_h.data(), F->strips_h.size() * sizeof(StripDesc), false, stage);
  write_section(os, "ifc_off_h", F->ifc_off_h.data(), F->ifc_off_h.size() * sizeof(int64_t), false, stage);
  write_section(os, "sym_h", F->sym_h.data(), F->sym_h.size() * sizeof(int32_t), false, stage);
#define SLB_SEC(buf) write_section(os, #buf, F->buf.p, F->buf.bytes(), true, stage)
  SLB_SEC(fac); SLB_SEC(perm); SLB_SEC(cpl); SLB_SEC(sym); SLB_SEC(u13); SLB_SEC(lnd); SLB_SEC(dsub); SLB_SEC(exc);
  SLB_SEC(excpos); SLB_SEC(hcol); SLB_SEC(hidx); SLB_SEC(T); SLB_SEC(ipivT); SLB_SEC(permT); SLB_SEC(dinvT);
  SLB_SEC(Xup); SLB_SEC(a_rp); SLB_SEC(a_ci); SLB_SEC(a_v);
#undef SLB_SEC
  os.flush();
  if (!os) throw HostError(SLABLU_ERR_GENERIC, std::string("save: write failed: ") + path);
}

slablu_gpu_fact* load_impl(const char* path, int device) {
  std::ifstream is(path, std::ios::binary);
  if (!is) throw HostError(SLABLU_ERR_GENERIC, std::string("load: cannot open ") + path);
  char magic[8];
  is.read(magic, 8);
  if (!is || memcmp(magic, kMagicGpu, 8) != 0)
    throw HostError(SLABLU_ERR_GENERIC, "load: bad magic or version (expected SLBGPU01)");
  auto F = std::make_unique<slablu_gpu_fact>();
  F->device = device;
  DeviceGuard dg(device);
  int least = 0, greatest = 0;
  SLB_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  SLB_CUDA_CHECK(cudaStreamCreateWithPriority(&F->stream, cudaStreamNonBlocking, greatest));
  StreamScope scope(F->stream);
  std::vector<int64_t> hdr;
  read_section_host(is, "header", hdr);
  if (hdr.size() != 12) throw HostError(SLABLU_ERR_GENERIC, "load: bad header");
  F->n1 = hdr[0];
  F->n2 = hdr[1];
  F->N = F->n1 * F->n2;
  F->b = hdr[2];
  F->S = (int)hdr[3];
  F->Sg = F->S;
  F->s1 = F->S;
  F->K = (int)hdr[4];
  F->j1 = F->K;
  F->Wp = (int)hdr[5];
  F->single = hdr[6] != 0;
  F->stage2_only = hdr[7] != 0;
  F->refine = (int)hdr[8];
  F->storage1 = hdr[9];
  F->storage2 = hdr[10];
  F->sF = hdr[11];
  F->sP = F->n2 * 2 * F->Wp;
  F->sCPL = 4 * F->n2 * F->Wp;
  std::vector<double> times;
  read_section_host(is, "times", times);
  if (times.size() == 5) {
    F->t1 = times[0];
    F->t2 = times[1];
    F->t_chain = times[2];
    F->t_schur = times[3];
    F->t_asm = times[4];
  }
  read_section_host(is, "strips_h", F->strips_h);
  read_section_host(is, "ifc_off_h", F->ifc_off_h);
  read_section_host(is, "sym_h", F->sym_h);
  if ((int)F->strips_h.size() != F->S || (int)F->ifc_off_h.size() != F->K)
    throw HostError(SLABLU_ERR_GENERIC, "load: inconsistent geometry");
  Pinned stage(kStage);
#define SLB_SEC(buf) read_section_dev(is, #buf, F->buf, device, stage)
  SLB_SEC(fac); SLB_SEC(perm); SLB_SEC(cpl); SLB_SEC(sym); SLB_SEC(u13); SLB_SEC(lnd); SLB_SEC(dsub); SLB_SEC(exc);
  SLB_SEC(excpos); SLB_SEC(hcol); SLB_SEC(hidx); SLB_SEC(T); SLB_SEC(ipivT); SLB_SEC(permT); SLB_SEC(dinvT);
  SLB_SEC(Xup); SLB_SEC(a_rp); SLB_SEC(a_ci); SLB_SEC(a_v);
#undef SLB_SEC
  if (F->S > 0) {
    F->strips.alloc(device, F->S);
    SLB_CUDA_CHECK(cudaMemcpy(F->strips.p, F->strips_h.data(), F->S * sizeof(StripDesc), cudaMemcpyHostToDevice));
  }
  if (F->K > 0) {
    F->ifc_off.alloc(device, F->K);
    SLB_CUDA_CHECK(cudaMemcpy(F->ifc_off.p, F->ifc_off_h.data(), F->K * sizeof(int64_t), cudaMemcpyHostToDevice));
  }
  static const DevStatus st0{0, INT_MAX, INT_MAX, INT_MAX};
  F->status.alloc(device, 1);
  F->sstatus.alloc(device, 1);
  SLB_CUDA_CHECK(cudaMemcpy(F->status.p, &st0, sizeof(st0), cudaMemcpyHostToDevice));
  SLB_CUDA_CHECK(cudaMemcpy(F->sstatus.p, &st0, sizeof(st0), cudaMemcpyHostToDevice));
  return F.release();
}

// stage two in the reference's SweepFactorization layout (stage_two.hpp:200-207, dense.hpp:71-76)
void export_sweep_impl(const slablu_gpu_fact* F, const char* path) {
  if (F->single || F->sharded || F->K < 1) throw HostError(SLABLU_ERR_CONFIG, "export_sweep: no stage two");
  std::lock_guard<std::mutex> guard(F->solve_mu);
  DeviceGuard dg(F->device);
  SLB_CUDA_CHECK(cudaStreamSynchronize(F->stream));
  std::ofstream os(path, std::ios::binary | std::ios::trunc);
  if (!os) throw HostError(SLABLU_ERR_GENERIC, std::string("export_sweep: cannot open ") + path);
  Pinned stage(kStage);
  const int64_t n2 = F->n2, bs = n2 * n2;
  os.write(kMagicSwp, 8);
  write_u64(os, (uint64_t)F->K);
  std::vector<int32_t> piv32(n2);
  std::vector<int64_t> piv64(n2);
  for (int j = 0; j < F->K; j++) {  // DenseLU: write_dense(lu), then int64 1-based pivots
    write_u64(os, (uint64_t)n2);
    write_u64(os, (uint64_t)n2);
    write_dev(os, F->Tdiag() + j * bs, bs * sizeof(double), stage);
    SLB_CUDA_CHECK(cudaMemcpy(piv32.data(), F->ipivT.p + (size_t)j * n2, n2 * sizeof(int32_t), cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < n2; i++) piv64[i] = (int64_t)piv32[i] + 1;
    os.write(reinterpret_cast<const char*>(piv64.data()), (std::streamsize)(n2 * sizeof(int64_t)));
  }
  for (int which = 0; which < 2; which++)  // sub blocks, then super blocks
    for (int j = 0; j + 1 < F->K; j++) {
      write_u64(os, (uint64_t)n2);
      write_u64(os, (uint64_t)n2);
      write_dev(os, (which == 0 ? F->Tsub() : F->Tsup()) + j * bs, bs * sizeof(double), stage);
    }
  os.flush();
  if (!os) throw HostError(SLABLU_ERR_GENERIC, std::string("export_sweep: write failed: ") + path);
}

// SLBSWP01 -> a stage-two-only handle (slablu_gpu_sweep_solve); the solve-side data (row
// permutation, diagonal-block inverses, X_j = S_j^{-1} super_j) is rebuilt from the LU factors
slablu_gpu_fact* import_sweep_impl(const char* path, int device) {
  std::ifstream is(path, std::ios::binary);
  if (!is) throw HostError(SLABLU_ERR_GENERIC, std::string("import_sweep: cannot open ") + path);
  char magic[8];
  is.read(magic, 8);
  if (!is || memcmp(magic, kMagicSwp, 8) != 0)
    throw HostError(SLABLU_ERR_GENERIC, "SweepFactorization::deserialize: bad magic or version");
  const int64_t k = (int64_t)read_u64(is);
  if (k < 1 || k > (1 << 20)) throw HostError(SLABLU_ERR_GENERIC, "import_sweep: bad block count");
  auto F = std::make_unique<slablu_gpu_fact>();
  F->device = device;
  DeviceGuard dg(device);
  SLB_CUDA_CHECK(cudaStreamCreateWithFlags(&F->stream, cudaStreamNonBlocking));
  StreamScope scope(F->stream);
  Pinned stage(kStage);
  int64_t m = -1;
  auto dense_header = [&]() {
    const int64_t r = (int64_t)read_u64(is), c = (int64_t)read_u64(is);
    if (r != c || (m >= 0 && r != m) || r < 1 || r > kMaxIfc)
      throw HostError(SLABLU_ERR_GENERIC, "import_sweep: blocks must be square, equal-sized, <= 4096");
    m = r;
  };
  std::vector<std::vector<int64_t>> pivs;
  for (int64_t j = 0; j < k; j++) {
    dense_header();
    if (j == 0) {
      F->K = (int)k;
      F->n1 = k;
      F->n2 = m;
      F->N = k * m;
      F->T.alloc(device, (size_t)(3 * k - 2) * m * m);
      F->ipivT.alloc(device, (size_t)k * m);
    }
    read_dev(is, F->Tdiag() + j * m * m, (size_t)m * m * sizeof(double), stage);
    std::vector<int64_t> p64(m);
    is.read(reinterpret_cast<char*>(p64.data()), (std::streamsize)(m * sizeof(int64_t)));
    if (!is) throw HostError(SLABLU_ERR_GENERIC, "DenseLU::deserialize: truncated stream");
    std::vector<int32_t> p32(m);
    for (int64_t i = 0; i < m; i++) {
      if (p64[i] < 1 || p64[i] > m) throw HostError(SLABLU_ERR_GENERIC, "import_sweep: pivot out of range");
      p32[i] = (int32_t)(p64[i] - 1);
    }
    SLB_CUDA_CHECK(cudaMemcpy(F->ipivT.p + (size_t)j * m, p32.data(), m * sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  for (int which = 0; which < 2; which++)
    for (int64_t j = 0; j + 1 < k; j++) {
      dense_header();
      read_dev(is, (which == 0 ? F->Tsub() : F->Tsup()) + j * m * m, (size_t)m * m * sizeof(double), stage);
    }
  F->stage2_only = true;
  F->status.alloc(device, 1);
  F->sstatus.alloc(device, 1);
  static const DevStatus st0{0, INT_MAX, INT_MAX, INT_MAX};
  SLB_CUDA_CHECK(cudaMemcpy(F->status.p, &st0, sizeof(st0), cudaMemcpyHostToDevice));
  SLB_CUDA_CHECK(cudaMemcpy(F->sstatus.p, &st0, sizeof(st0), cudaMemcpyHostToDevice));
  const int64_t dinv_sz = cdiv(m, 64) * 2 * 64 * 64, bs = m * m;
  F->permT.alloc(device, (size_t)k * m);
  F->dinvT.alloc(device, (size_t)k * dinv_sz);
  F->Xup.alloc(device, (size_t)std::max<int64_t>(k - 1, 1) * bs);
  for (int64_t j = 0; j < k; j++)
    getrs_prepare(F->stream, m, F->Tdiag() + j * bs, F->ipivT.p + j * m, F->permT.p + j * m, F->dinvT.p + j * dinv_sz);
  for (int64_t j = 0; j + 1 < k; j++) {
    double* X = F->Xup.p + j * bs;
    SLB_CUDA_CHECK(cudaMemcpyAsync(X, F->Tsup() + j * bs, bs * sizeof(double), cudaMemcpyDeviceToDevice, F->stream));
    dgetrs(F->stream, m, m, F->Tdiag() + j * bs, F->ipivT.p + j * m, X, m, nullptr);
  }
  SLB_CUDA_CHECK(cudaStreamSynchronize(F->stream));
  F->storage2 = (k + 2 * (k - 1)) * m * m;
  return F.release();
}

}  // namespace

extern "C" {

slablu_gpu_status slablu_gpu_save(const slablu_gpu_fact* fact, const char* path) {
  ABI_TRY({
    if (!fact || !path) throw HostError(SLABLU_ERR_GENERIC, "save: null argument");
    save_impl(fact, path);
  })
}
slablu_gpu_status slablu_gpu_load(const char* path, int device, slablu_gpu_fact** out) {
  ABI_TRY({
    require_device();
    *out = nullptr;
    if (!path) throw HostError(SLABLU_ERR_GENERIC, "load: null path");
    *out = load_impl(path, device);
  })
}
slablu_gpu_status slablu_gpu_export_sweep(const slablu_gpu_fact* fact, const char* path) {
  ABI_TRY({
    if (!fact || !path) throw HostError(SLABLU_ERR_GENERIC, "export_sweep: null argument");
    export_sweep_impl(fact, path);
  })
}
slablu_gpu_status slablu_gpu_import_sweep(const char* path, int device, slablu_gpu_fact** out) {
  ABI_TRY({
    require_device();
    *out = nullptr;
    if (!path) throw HostError(SLABLU_ERR_GENERIC, "import_sweep: null path");
    *out = import_sweep_impl(path, device);
  })
}

}  // extern "C"
